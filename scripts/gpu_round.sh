set -x
python -m paper_1203_2739_b200.build > /dev/null
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
SPMV_KERNEL=panel timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "spmv_parity or edge" 2>&1 | tail -2
cd scripts
timeout 300 python ab.py c4 panel,rowtile
K=16 KERNELS=panel timeout 300 python xs_probe.py 2>&1 | grep -E '"panel_ms"'
