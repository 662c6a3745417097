# the multi-GPU loopback tests alone, each under a timeout
set -u
R=${R:-r2c}
mkdir -p gpurun_out
python -m paper_1203_2739_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_ranks.py -q -rf --timeout 240 --timeout-method=thread > gpurun_out/${R}_ranks.log 2>&1; echo "ranks rc=$? $(tail -1 gpurun_out/${R}_ranks.log)"
timeout 600 python -m pytest tests/test_gpu_order.py -q -rf --timeout 240 --timeout-method=thread > gpurun_out/${R}_order.log 2>&1; echo "order rc=$? $(tail -1 gpurun_out/${R}_order.log)"
AB="W16 W24" CFGS="c4 c5" ROUNDS=2 bash scripts/ab_lib.sh > gpurun_out/${R}_ab.txt 2>&1; echo "ab done"
