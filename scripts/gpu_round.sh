set -x
python -m paper_1203_2739_b200.build > /dev/null
timeout 400 python -m pytest tests/test_gpu_xstage.py tests/test_gpu_parity.py -q -x 2>&1 | tail -1
cd scripts
run() { K=$1 KERNELS=panel timeout 300 python xs_probe.py 2>&1 | grep -E '"panel_ms"|create_s|rror' | tr '\n' ' ' | sed "s/^/K$1 $2 /"; echo; }
run 16 colour; SPMV_PN_NOCOLOUR=1 run 16 nocolour
run 64 colour
