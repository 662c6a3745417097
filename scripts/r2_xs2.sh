set -u
R=${R:-r2u}
mkdir -p gpurun_out
python -m paper_1203_2739_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_xstaged.py -q -rf --timeout 300 --timeout-method=thread > gpurun_out/${R}_xs.log 2>&1; echo "xs tests rc=$? $(tail -1 gpurun_out/${R}_xs.log)"
timeout 600 python bench.py --workload c2 > gpurun_out/${R}_bench_c2.json 2> gpurun_out/${R}_bench_c2.err; echo "bench c2 rc=$?"
timeout 600 python scripts/ab_kernels.py c2 rowtile xstaged panel > gpurun_out/${R}_abk.txt 2>&1; echo "abk rc=$?"
