set -x
mkdir -p gpurun_out
python -m paper_1203_2739_b200.build > /dev/null
for w in c4 c3 c2 c1; do timeout 300 python bench.py --workload $w --no-e2e > gpurun_out/r53_bench_$w.json 2> gpurun_out/r53_bench_$w.err; python -c "import json;d=json.load(open('gpurun_out/r53_bench_$w.json'));print('$w', d['value'], d['spmv_ms'], d['roofline']['frac'], d['config'].get('kernel'), d['parity']['failures'])"; done
cd scripts && timeout 300 python c3_split.py > ../gpurun_out/r53_c3_split.json 2>&1; cat ../gpurun_out/r53_c3_split.json
