# ncu evidence of the current code: C5 launch list, full captures of the C5 and C4 panel kernels
set -u
R=${R:-r2m}
mkdir -p gpurun_out
python -m paper_1203_2739_b200.build > /dev/null
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-gather-peak --no-reorder-ref --no-cusparse --no-sbfs"
timeout 600 $B --workload c5 > gpurun_out/${R}_plain_c5.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${R}_launches_c5.csv $B --workload c5 > gpurun_out/${R}_ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:spmv_panel_kernel -s 3 -c 1 -f -o gpurun_out/${R}_panel_c5 $B --workload c5 > gpurun_out/${R}_ncu_c5.log 2>&1; echo "full c5 rc=$?"
timeout 600 $B --workload c4 > gpurun_out/${R}_plain_c4.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_panel_kernel -s 3 -c 1 -f -o gpurun_out/${R}_panel_c4 $B --workload c4 > gpurun_out/${R}_ncu_c4.log 2>&1; echo "full c4 rc=$?"
