set -x
python -m paper_1203_2739_b200.build > /dev/null
SPMV_KERNEL=panel timeout 300 python -m pytest tests/test_gpu_xstage.py -q -x 2>&1 | tail -2
SPMV_PN_MODE=9 timeout 300 python -m pytest tests/test_gpu_xstage.py -q -x -k "panel and not c5_like" 2>&1 | tail -2
cd scripts
for m in 0 9; do SPMV_PN_MODE=$m SPMV_PN_ROWS=16384 K=4 KERNELS=panel,rowtile timeout 300 python xs_warmx.py | sed "s/^/K4 mode $m /"; done
SPMV_PN_MODE=0 K=64 KERNELS=panel timeout 300 python xs_probe.py | grep panel_ms | sed "s/^/C5 mode 0 /"
SPMV_PN_MODE=9 SPMV_PN_ROWS=16384 K=64 KERNELS=panel timeout 300 python xs_probe.py | grep panel_ms | sed "s/^/C5 mode 9 /"
