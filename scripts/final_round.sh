# Round-end evidence: tests, smoke, the five bench lines, the C5 launch list
# and full ncu captures of the C5 and C4 SpMxV kernels (each ncu run wraps a
# command that has just exited 0 without ncu).
set -u
R=${R:-r99}
mkdir -p gpurun_out
python -m paper_1203_2739_b200.build > /dev/null
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/${R}_pytest.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/${R}_pytest.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo "smoke rc=$? $(tail -1 gpurun_out/${R}_smoke.log)"
for c in c1 c2 c3 c4 c5; do
  timeout 900 python bench.py --workload $c > gpurun_out/${R}_bench_$c.json 2> gpurun_out/${R}_bench_$c.err
  echo "bench $c rc=$?"
done
(cd scripts && timeout 600 python c3_split.py > ../gpurun_out/${R}_c3_split.json 2> ../gpurun_out/${R}_c3_split.err); echo "c3 split rc=$?"
(cd scripts && timeout 600 python c5_drift.py c5 10 > ../gpurun_out/${R}_c5_drift.jsonl 2> ../gpurun_out/${R}_c5_drift.err); echo "drift rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${R}_bench_ref.json 2> gpurun_out/${R}_bench_ref.err; echo "ref rc=$?"
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-gather-peak --no-reorder-ref --no-cusparse"
timeout 600 $B --workload c5 > gpurun_out/${R}_plain_c5.json 2>&1; echo "plain c5 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${R}_launches_c5.csv $B --workload c5 > gpurun_out/${R}_ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:spmv_panel_kernel -s 3 -c 1 -f -o gpurun_out/${R}_panel_c5 $B --workload c5 > gpurun_out/${R}_ncu_c5.log 2>&1; echo "full c5 rc=$?"
timeout 600 $B --workload c4 > gpurun_out/${R}_plain_c4.json 2>&1; echo "plain c4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_panel_kernel -s 3 -c 1 -f -o gpurun_out/${R}_panel_c4 $B --workload c4 > gpurun_out/${R}_ncu_c4.log 2>&1; echo "full c4 rc=$?"
