# Shared-memory carveout of the panel kernel (build-time hint SPMV_PN_CARVEOUT):
# what the driver picks (ncu launch metrics) and interleaved timings.
set -u
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-gather-peak --no-reorder-ref --no-cusparse --no-sbfs"
for v in BASE CV58 CV72 CV100; do
  cp ablib/lib$v.so paper_1203_2739_b200/libspmv_b200.so
  for c in c4 c5; do
    timeout 900 ncu --metrics launch__shared_mem_config_size,launch__shared_mem_per_block_dynamic,launch__shared_mem_per_block_static,launch__shared_mem_per_block_driver,gpu__time_duration.sum --clock-control none -k regex:spmv_panel -s 2 -c 1 --csv $B --workload $c 2>/dev/null | grep -E "launch__|gpu__time" | sed "s/^/$v $c /"
  done
done > gpurun_out/r03c_smem_config.csv
echo "config rc=$?"
AB="BASE CV58 CV72 CV100" CFGS="c4 c5" ROUNDS=2 bash scripts/ab_lib.sh > gpurun_out/r03c_ab.txt 2>&1; echo "ab rc=$?"
cp ablib/libBASE.so paper_1203_2739_b200/libspmv_b200.so
