python -m paper_1203_2739_b200.build > /dev/null
cd scripts
ROUNDS=6 timeout 900 python ab_inter.py c2 "" "SPMV_TILE_NNZ=1700" "SPMV_TILE_NNZ=1400" "SPMV_TILE_NNZ=1024" "SPMV_TILE_NNZ=700" 2>&1 | tail -1
ROUNDS=6 timeout 900 python ab_inter.py c1 "" "SPMV_TILE_NNZ=1024" "SPMV_TILE_NNZ=512" "SPMV_TILE_NNZ=256" 2>&1 | tail -1
