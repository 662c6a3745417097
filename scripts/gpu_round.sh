set -x
mkdir -p gpurun_out
python -m paper_1203_2739_b200.build > /dev/null
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/r48_pytest.log 2>&1; tail -2 gpurun_out/r48_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r48_bench.json 2> gpurun_out/r48_bench.err; tail -2 gpurun_out/r48_bench.err; cat gpurun_out/r48_bench.json
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-gather-peak"
$CMD > gpurun_out/r48_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r48_launches.csv $CMD > gpurun_out/r48_ncu_launch.log 2>&1; tail -1 gpurun_out/r48_ncu_launch.log
