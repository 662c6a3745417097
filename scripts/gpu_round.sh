set -x
python -m paper_1203_2739_b200.build > /dev/null
SPMV_PN_MODE=23 timeout 300 python -m pytest tests/test_gpu_xstage.py tests/test_gpu_variants.py -q -x -k "panel" 2>&1 | tail -1
cd scripts
run() { SPMV_PN_MODE=$1 K=16 KERNELS=panel timeout 300 python xs_probe.py 2>&1 | grep -E '"panel_ms"|rror' | sed "s/^/K16 mode $1 /"; }
run 0; run 23; run 0; run 23
SPMV_PN_MODE=23 timeout 300 python ab.py c4 panel | sed "s/^/mode23 /"
timeout 300 python ab.py c4 panel | sed "s/^/mode0 /"
