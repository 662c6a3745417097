set -x
python -m paper_1203_2739_b200.build > /dev/null
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
cd scripts
timeout 300 python ab.py c4 panel,rowtile
timeout 300 python ab.py c2 panel,rowtile
timeout 300 python ab.py c4 panel
