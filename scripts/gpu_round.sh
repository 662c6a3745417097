set -x
mkdir -p gpurun_out
python -m paper_1203_2739_b200.build > /dev/null
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/r35_pytest.log 2>&1; tail -3 gpurun_out/r35_pytest.log
for w in c4 c3 c2 c1; do timeout 300 python bench.py --workload $w --no-e2e > gpurun_out/r35_bench_$w.json 2> gpurun_out/r35_bench_$w.err; tail -1 gpurun_out/r35_bench_$w.err; python -c "import json;d=json.load(open('gpurun_out/r35_bench_$w.json'));print('$w', d['value'], d['spmv_ms'], d['roofline']['frac'], d['parity'])"; done
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-gather-peak"
$CMD > gpurun_out/r35_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:rowtile -s 3 -c 1 -o gpurun_out/r35_rowtile_c5 $CMD > gpurun_out/r35_ncu.log 2>&1; tail -2 gpurun_out/r35_ncu.log
