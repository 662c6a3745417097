set -x
python -m paper_1203_2739_b200.build > /dev/null
cd scripts
run() { K=16 KERNELS=panel timeout 300 python xs_probe.py 2>&1 | grep -E '"panel_ms"|rror' | sed "s/^/K16 $1 /"; }
SPMV_LIB=/root/repo/ablib/nospread.so run nospread; run spread; SPMV_LIB=/root/repo/ablib/nospread.so run nospread; run spread
