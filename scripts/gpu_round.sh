python -m paper_1203_2739_b200.build > /dev/null
cd scripts
timeout 900 python ab_inter.py c5 "" "SPMV_PN_GATHER_NA=1" "SPMV_PN_ROWS=20480,SPMV_PN_GATHER_NA=1" "SPMV_PN_ROWS=24576,SPMV_PN_GATHER_NA=1" 2>&1 | tail -1
