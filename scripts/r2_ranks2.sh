set -u
R=${R:-r2g}
mkdir -p gpurun_out
python -m paper_1203_2739_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_ranks.py tests/test_gpu_parity.py -k "ranks or index16 or db or peer or edge" -q -rf --timeout 300 --timeout-method=thread > gpurun_out/${R}_ranks.log 2>&1; echo "ranks rc=$? $(tail -1 gpurun_out/${R}_ranks.log)"
