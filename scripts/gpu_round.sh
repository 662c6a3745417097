python -m paper_1203_2739_b200.build > /dev/null
for c in c4 c5; do
timeout 600 python bench.py --workload $c --no-e2e --no-cpu-baseline --no-parity --no-reorder-ref --no-cusparse 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$c', j['spmv_ms'], j['roofline']['frac'], j['roofline_gather'])"
done
