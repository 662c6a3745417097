python -m paper_1203_2739_b200.build > /dev/null
cd scripts
ROUNDS=8 timeout 1200 python ab_inter.py c5 "" "SPMV_PN_ROWS=13000" "SPMV_PN_ROWS=18000" "SPMV_PN_GATHER_NA=0" 2>&1 | tail -1
