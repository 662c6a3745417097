# Round-2 round-end evidence on the final code: GPU tests, smoke, the five bench
# lines, C3 split, C5 power drift, the reference arm, then (each after its
# command exited 0 without ncu) the C5/C4 launch lists and full ncu captures of
# the C5/C4 panel kernels, the C5 x-update and the C2 row-tile kernel.
set -u
R=${R:-r02z}
mkdir -p gpurun_out
python -m paper_1203_2739_b200.build > /dev/null
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 900 --timeout-method=thread > gpurun_out/${R}_pytest.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/${R}_pytest.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo "smoke rc=$? $(tail -1 gpurun_out/${R}_smoke.log)"
for c in c5 c4 c3 c2 c1; do
  timeout 900 python bench.py --workload $c > gpurun_out/${R}_bench_$c.json 2> gpurun_out/${R}_bench_$c.err
  echo "bench $c rc=$?"
done
(cd scripts && timeout 600 python c3_split.py > ../gpurun_out/${R}_c3_split.json 2> ../gpurun_out/${R}_c3_split.err); echo "c3 split rc=$?"
(cd scripts && timeout 600 python c5_drift.py c5 10 > ../gpurun_out/${R}_c5_drift.jsonl 2> ../gpurun_out/${R}_c5_drift.err); echo "drift rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${R}_bench_ref.json 2> gpurun_out/${R}_bench_ref.err; echo "ref rc=$?"
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-gather-peak --no-reorder-ref --no-cusparse --no-sbfs"
for c in c5 c4; do
  timeout 600 $B --workload $c > gpurun_out/${R}_plain_$c.json 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${R}_launches_$c.csv $B --workload $c > gpurun_out/${R}_ncu_launch_$c.log 2>&1; echo "launch list $c rc=$?"
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:spmv_panel_kernel -s 3 -c 1 -f -o gpurun_out/${R}_panel_$c $B --workload $c > gpurun_out/${R}_ncu_$c.log 2>&1; echo "full $c rc=$?"
done
timeout 900 ncu --set full --clock-control none -k regex:normalize -s 2 -c 1 -f -o gpurun_out/${R}_norm_c5 $B --workload c5 > gpurun_out/${R}_ncu_norm.log 2>&1; echo "full norm c5 rc=$?"
timeout 600 $B --workload c2 > gpurun_out/${R}_plain_c2.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_ -s 3 -c 1 -f -o gpurun_out/${R}_kernel_c2 $B --workload c2 > gpurun_out/${R}_ncu_c2.log 2>&1; echo "full c2 rc=$?"
