set -x
mkdir -p gpurun_out
python -m paper_1203_2739_b200.build > /dev/null
timeout 600 python -m pytest tests -m gpu -q -x -k "split or smoke or power" > gpurun_out/r38_pytest.log 2>&1; tail -3 gpurun_out/r38_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
cd scripts
timeout 300 python c3_split.py 2>&1 | tail -12
SPMV_SPLIT_PARTMAJOR=1 timeout 300 python c3_split.py 2>&1 | grep fused
