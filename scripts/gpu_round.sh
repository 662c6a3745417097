set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r16_pytest.log 2>&1
tail -15 gpurun_out/r16_pytest.log
cd scripts
for w in c5 c4 c2; do AB=1 timeout 600 python diag_c5.py $w > ../gpurun_out/r16_diag_$w.json 2>&1; grep -E "mode1_ms|spmv" ../gpurun_out/r16_diag_$w.json; done
