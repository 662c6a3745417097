set -x
python -m paper_1203_2739_b200.build > /dev/null
timeout 400 python -m pytest tests/test_gpu_xstage.py -q -x 2>&1 | tail -1
cd scripts
run() { K=16 KERNELS=panel timeout 300 python xs_probe.py 2>&1 | grep -E '"panel_ms"|rror' | sed "s/^/K16 $1 /"; }
SPMV_LIB=/root/repo/ablib/prev.so run prev
run new
SPMV_PN_NOCOLOUR=1 run new_nocolour
SPMV_PN_SWEEPS=4 SPMV_PN_TRIES=6 run new_s4t6
