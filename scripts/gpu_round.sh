python -m paper_1203_2739_b200.build > /dev/null
cd scripts
ROUNDS=6 timeout 900 python ab_inter.py c4 "" "SPMV_PN_GATHER_NA=1" "SPMV_PN_RING=12" "SPMV_PN_PF=6" 2>&1 | tail -1
ROUNDS=6 timeout 900 python ab_inter.py c3 "" "SPMV_PN_GATHER_NA=1" 2>&1 | tail -1
