set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/r1_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1_smoke.log 2>&1
timeout 300 python bench.py --workload c2 --steps 20 --warmup 3 --cpu-seconds 3 > gpurun_out/r1_bench_c2.log 2>&1
timeout 300 python bench.py --workload c4 --steps 50 --warmup 3 --cpu-seconds 3 > gpurun_out/r1_bench_c4.log 2>&1
timeout 900 python bench.py --workload c5 --steps 20 --warmup 3 --cpu-seconds 5 > gpurun_out/r1_bench_c5.log 2>&1
tail -3 gpurun_out/r1_*.log
