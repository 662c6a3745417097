set -x
mkdir -p gpurun_out
python -m paper_1203_2739_b200.build > /dev/null
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/r60_pytest.log 2>&1; tail -2 gpurun_out/r60_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r60_bench.json 2> gpurun_out/r60_bench.err; tail -1 gpurun_out/r60_bench.err; cat gpurun_out/r60_bench.json
for w in c4 c3 c2 c1; do timeout 300 python bench.py --workload $w > gpurun_out/r60_bench_$w.json 2> gpurun_out/r60_bench_$w.err; python -c "import json;d=json.load(open('gpurun_out/r60_bench_$w.json'));print('$w', d['value'], d['spmv_ms'], d['roofline']['frac'], d['parity']['failures'], d['e2e']['value'], d.get('reordering',{}).get('speedup'), d.get('warm_l2_spmv_ms'))"; done
