set -x
mkdir -p gpurun_out
python -m paper_1203_2739_b200.build > /dev/null
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-gather-peak"
$CMD > gpurun_out/r49_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:panel -s 3 -c 1 -o gpurun_out/r49_panel_c5 $CMD > gpurun_out/r49_ncu.log 2>&1; tail -1 gpurun_out/r49_ncu.log
