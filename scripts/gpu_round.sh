python -m paper_1203_2739_b200.build > /dev/null
cd scripts
ROUNDS=8 timeout 900 python ab_inter.py c4 "" "SPMV_PN_ROWS=16800" "SPMV_PN_ROWS=8400" "SPMV_PN_ROWS=16800,SPMV_PN_GATHER_NA=1" 2>&1 | tail -1
