set -x
mkdir -p gpurun_out
python -m paper_1203_2739_b200.build > /dev/null
cd scripts
for g in 0 1 2; do SPMV_RT_GMODE=$g K=64 KERNELS=rowtile timeout 300 python xs_probe.py 2>&1 | grep -E '"rowtile_ms"|Error' | sed "s/^/C5 gmode $g /"; done
