python -m paper_1203_2739_b200.build > /dev/null
cd scripts
ROUNDS=8 timeout 900 python ab_inter.py c4 "" "SPMV_PN_RING=8" "SPMV_PN_RING=16" 2>&1 | tail -1
ROUNDS=8 timeout 900 python ab_inter.py c3 "" "SPMV_PN_RING=8" 2>&1 | tail -1
