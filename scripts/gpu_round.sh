set -x
mkdir -p gpurun_out
free -g | head -2; nproc
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r22_smoke.log 2>&1; tail -3 gpurun_out/r22_smoke.log
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/r22_pytest.log 2>&1
tail -30 gpurun_out/r22_pytest.log
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r22_bench.json 2> gpurun_out/r22_bench.err; tail -3 gpurun_out/r22_bench.err; cat gpurun_out/r22_bench.json
