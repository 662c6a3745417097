python -m paper_1203_2739_b200.build > /dev/null
cd scripts
ROUNDS=6 timeout 900 python ab_inter.py c4 "LIB=$PWD/../ablib/prepersist.so" "" 2>&1 | tail -1
ROUNDS=8 timeout 1200 python ab_inter.py c5 "LIB=$PWD/../ablib/prepersist.so" "" 2>&1 | tail -1
