set -x
python -m paper_1203_2739_b200.build > /dev/null
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
cd scripts
for w in c5 c4 c2; do timeout 300 python ab.py $w rowtile; done
timeout 300 python c3_split.py 2>&1 | grep -E "fused|single"
