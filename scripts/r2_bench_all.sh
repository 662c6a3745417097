set -u
R=${R:-r2p}
mkdir -p gpurun_out
python -m paper_1203_2739_b200.build > /dev/null
for c in ${CFGS:-c5 c3 c1}; do
  timeout 900 python bench.py --workload $c > gpurun_out/${R}_bench_$c.json 2> gpurun_out/${R}_bench_$c.err
  echo "bench $c rc=$?"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${R}_bench_ref.json 2> gpurun_out/${R}_bench_ref.err; echo "ref rc=$?"
