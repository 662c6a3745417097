set -x
python -m paper_1203_2739_b200.build > /dev/null
timeout 300 python -m pytest tests/test_gpu_xstage.py tests/test_gpu_parity.py -q -x 2>&1 | tail -1
cd scripts
run() { SPMV_PN_MODE=$1 SPMV_PN_ROWS=$2 K=$3 KERNELS=panel timeout 300 python xs_probe.py 2>&1 | grep -E '"panel_ms"|rror' | sed "s/^/K$3 mode $1 rows $2 /"; }
run 0 16384 16; run 19 16384 16
run 0 16384 64
