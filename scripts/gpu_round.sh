set -x
python -m paper_1203_2739_b200.build > /dev/null
timeout 600 python bench.py --workload c2 --no-e2e --no-cpu-baseline > gpurun_out/r57_c2.json 2>gpurun_out/r57_c2.err; tail -2 gpurun_out/r57_c2.err; python -c "import json;d=json.load(open('gpurun_out/r57_c2.json'));print('c2', d['spmv_ms'], d.get('warm_l2_spmv_ms'), d.get('reordering'))"
timeout 900 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r57_c5.json 2>gpurun_out/r57_c5.err; tail -2 gpurun_out/r57_c5.err; python -c "import json;d=json.load(open('gpurun_out/r57_c5.json'));print('c5', d['spmv_ms'], d['roofline']['frac'], d.get('reordering'))"
