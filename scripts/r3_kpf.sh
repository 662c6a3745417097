# group-stream L2 prefetch distance (epochs) and a stronger y-bank colouring on C5: sustained bench SpMxV time and DRAM bytes per launch
set -u
B="python bench.py --workload c5 --steps 64 --warmup 5 --no-e2e --no-cpu-baseline --no-parity --no-gather-peak --no-reorder-ref --no-cusparse --no-sbfs"
for r in 1 2; do for v in NOPF KPF2 KPF3 KPF6 NS8; do
  cp ablib/lib$v.so paper_1203_2739_b200/libspmv_b200.so
  echo "$r $v $(timeout 600 $B 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["spmv_ms"], d["ms_per_step"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])')"
done; done
Q="python bench.py --workload c5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-gather-peak --no-reorder-ref --no-cusparse --no-sbfs"
for v in NOPF KPF2 KPF3 KPF6 NS8; do
  cp ablib/lib$v.so paper_1203_2739_b200/libspmv_b200.so
  timeout 600 $Q > /dev/null 2>&1 && timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:spmv_panel_kernel -s 3 -c 1 --csv $Q 2>/dev/null | grep -E "dram__bytes|gpu__time" | awk -F'","' -v v=$v '{print v, $(NF-2), $(NF-1), $NF}'
done
cp ablib/libNOPF.so paper_1203_2739_b200/libspmv_b200.so
