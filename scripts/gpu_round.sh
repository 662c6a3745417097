python -m paper_1203_2739_b200.build > /dev/null
cd scripts
timeout 600 python c5_drift.py c5 10 2>&1 | tail -10
