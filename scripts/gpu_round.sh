set -x
python -m paper_1203_2739_b200.build > /dev/null
timeout 900 python bench.py --no-cpu-baseline --no-reorder-ref > gpurun_out/r58_c5.json 2>gpurun_out/r58_c5.err; tail -2 gpurun_out/r58_c5.err; python -c "import json;d=json.load(open('gpurun_out/r58_c5.json'));print('c5', d['spmv_ms'], d['roofline']['frac'], d['e2e'])"
timeout 600 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/r58_c3.json 2>gpurun_out/r58_c3.err; tail -2 gpurun_out/r58_c3.err; python -c "import json;d=json.load(open('gpurun_out/r58_c3.json'));print('c3', d['spmv_ms'], d['e2e'])"
