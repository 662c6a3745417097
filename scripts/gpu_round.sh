set -x
python -m paper_1203_2739_b200.build > /dev/null
cd scripts
run() { K=16 KERNELS=panel timeout 300 python xs_probe.py 2>&1 | grep -E '"panel_ms"|rror' | sed "s/^/K16 $1 /"; }
run b4; SPMV_LIB=/root/repo/ablib/pnb8.so run b8; run b4; SPMV_LIB=/root/repo/ablib/pnb8.so run b8
