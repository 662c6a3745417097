python -m paper_1203_2739_b200.build > /dev/null
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
cd scripts
ROUNDS=10 timeout 900 python ab_inter.py c5 "SPMV_PN_NOWAVES=1" "" 2>&1 | tail -1
