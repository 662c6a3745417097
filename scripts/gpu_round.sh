set -x
mkdir -p gpurun_out
python -m paper_1203_2739_b200.build > /dev/null
timeout 300 python -m pytest tests/test_gpu_xstage.py -q -x > gpurun_out/r25_pytest_xs.log 2>&1; tail -15 gpurun_out/r25_pytest_xs.log
cd scripts
KERNELS=panel,rowtile timeout 300 python xs_probe.py > ../gpurun_out/r25_probe.json 2>&1; cat ../gpurun_out/r25_probe.json
cd ..
timeout 400 python -m pytest tests -m gpu -q -x > gpurun_out/r25_pytest.log 2>&1; tail -5 gpurun_out/r25_pytest.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-gather-peak > gpurun_out/r25_bench.json 2> gpurun_out/r25_bench.err; tail -3 gpurun_out/r25_bench.err; cat gpurun_out/r25_bench.json
