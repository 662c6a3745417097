python -m paper_1203_2739_b200.build > /dev/null
cd scripts
ROUNDS=6 timeout 900 python ab_inter.py c4 "" "SPMV_PN_PERSIST=2" "SPMV_PN_PERSIST=2,SPMV_PN_ROWS=10000" "SPMV_PN_PERSIST=2,SPMV_PN_ROWS=8400" "SPMV_PN_PERSIST=2,SPMV_PN_ROWS=5600" 2>&1 | tail -1
ROUNDS=4 timeout 900 python ab_inter.py c3 "" "SPMV_PN_PERSIST=2" 2>&1 | tail -1
