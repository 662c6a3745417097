set -x
mkdir -p gpurun_out
python -m paper_1203_2739_b200.build > /dev/null
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/r39_pytest.log 2>&1; tail -3 gpurun_out/r39_pytest.log
cd scripts
timeout 300 python ab.py c4 rowtile,rowlin
SPMV_LONG_INLINE=1 timeout 300 python ab.py c4 rowtile
timeout 300 python c3_split.py 2>&1 | grep -E "fused|single"
