set -x
mkdir -p gpurun_out
python -m paper_1203_2739_b200.build > /dev/null
cd scripts
timeout 300 python c3_split.py > ../gpurun_out/r37_c3.json 2>&1; cat ../gpurun_out/r37_c3.json
cd ..
CMD="python bench.py --workload c4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-gather-peak"
$CMD > gpurun_out/r37_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:rowtile -s 3 -c 1 -o gpurun_out/r37_rowtile_c4 $CMD > gpurun_out/r37_ncu.log 2>&1; tail -2 gpurun_out/r37_ncu.log
