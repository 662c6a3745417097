python -m paper_1203_2739_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_xstage.py -q -x -k "persistent" 2>&1 | tail -3
cd scripts
ROUNDS=6 timeout 900 python ab_inter.py c4 "" "SPMV_PN_PERSIST=1" 2>&1 | tail -1
ROUNDS=8 timeout 1200 python ab_inter.py c5 "" "SPMV_PN_PERSIST=1" 2>&1 | tail -1
