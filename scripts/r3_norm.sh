# Owner-map runs in the x-update (a9): GPU tests of the power glue, C5/C4 bench
# lines, and the C5 launch list (per-kernel durations: normalize before/after).
set -u
R=${R:-r03n}
mkdir -p gpurun_out
python -m paper_1203_2739_b200.build > /dev/null
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -k "power or owner or original or edge" --timeout 900 > gpurun_out/${R}_pytest.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/${R}_pytest.log)"
for c in c5 c4; do
  timeout 900 python bench.py --workload $c > gpurun_out/${R}_bench_$c.json 2> gpurun_out/${R}_bench_$c.err
  echo "bench $c rc=$?"
done
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-gather-peak --no-reorder-ref --no-cusparse"
timeout 600 $B --workload c5 > gpurun_out/${R}_plain_c5.json 2>&1; echo "plain c5 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${R}_launches_c5.csv $B --workload c5 > gpurun_out/${R}_ncu_launch.log 2>&1; echo "launch list c5 rc=$?"
timeout 600 $B --workload c4 > gpurun_out/${R}_plain_c4.json 2>&1; echo "plain c4 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${R}_launches_c4.csv $B --workload c4 > gpurun_out/${R}_ncu_launch4.log 2>&1; echo "launch list c4 rc=$?"
