set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r23_smoke.log 2>&1; tail -3 gpurun_out/r23_smoke.log
timeout 300 python -m pytest tests/test_gpu_xstage.py -q -x > gpurun_out/r23_pytest_xs.log 2>&1; tail -5 gpurun_out/r23_pytest_xs.log
timeout 400 python -m pytest tests -m gpu -q -x > gpurun_out/r23_pytest.log 2>&1; tail -5 gpurun_out/r23_pytest.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-gather-peak > gpurun_out/r23_bench.json 2> gpurun_out/r23_bench.err; tail -3 gpurun_out/r23_bench.err; cat gpurun_out/r23_bench.json
