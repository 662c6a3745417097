set -x
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/r14_bench_c5.json 2> gpurun_out/r14_bench_c5.err
tail -1 gpurun_out/r14_bench_c5.json
for w in c4 c3 c2; do timeout 300 python bench.py --workload $w > gpurun_out/r14_bench_$w.json 2> gpurun_out/r14_bench_$w.err; tail -1 gpurun_out/r14_bench_$w.json | cut -c1-400; done
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-gather-peak"
timeout 300 $B > gpurun_out/r14_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r14_launches_c5.csv $B > gpurun_out/r14_ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:spmv_rowtile -s 4 -c 1 -o gpurun_out/r14_full_c5 $B > gpurun_out/r14_ncu_full.log 2>&1
ls -la gpurun_out | tail -5
