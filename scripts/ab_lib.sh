# A/B of prebuilt library variants (ablib/lib<V>.so), interleaved rounds:
#   AB="W16 W24" CFGS="c4 c5" ROUNDS=2 bash scripts/ab_lib.sh
set -u
mkdir -p gpurun_out
B="python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-parity --no-gather-peak --no-reorder-ref --no-cusparse"
for r in $(seq 1 ${ROUNDS:-2}); do
  for c in ${CFGS:-c4 c5}; do
    for v in ${AB}; do
      cp ablib/lib$v.so paper_1203_2739_b200/libspmv_b200.so
      out=$(timeout 600 $B --workload $c 2>/dev/null | tail -1)
      echo "$r $c $v $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["spmv_ms"], d["roofline"]["frac"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])' 2>&1)"
    done
  done
done
