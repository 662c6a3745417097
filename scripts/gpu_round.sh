set -x
mkdir -p gpurun_out
python -m paper_1203_2739_b200.build > /dev/null
timeout 600 python -m pytest tests/test_gpu_variants.py -q -x > gpurun_out/r36_pytest.log 2>&1; tail -3 gpurun_out/r36_pytest.log
cd scripts
for w in c4 c5 c2; do timeout 300 python ab.py $w rowtile,rowlin; done
