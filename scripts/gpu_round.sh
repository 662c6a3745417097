mkdir -p gpurun_out
python -m paper_1203_2739_b200.build > /dev/null
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-gather-peak --no-reorder-ref --no-cusparse"
for c in c2 c3; do
  timeout 600 $B --workload $c > gpurun_out/r87_plain_$c.json 2> gpurun_out/r87_plain_$c.err; echo "plain $c rc=$?"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_rowtile -s 3 -c 1 -f -o gpurun_out/r87_rowtile_c2 $B --workload c2 > gpurun_out/r87_ncu_c2.log 2>&1; echo "full c2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_panel -s 3 -c 1 -f -o gpurun_out/r87_panel_c3 $B --workload c3 > gpurun_out/r87_ncu_c3.log 2>&1; echo "full c3 rc=$?"
