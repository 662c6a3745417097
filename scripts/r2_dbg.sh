set -u
R=${R:-r2l}
mkdir -p gpurun_out
python -m paper_1203_2739_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_panel.py -q -rf --timeout 300 --timeout-method=thread > gpurun_out/${R}_dbg.log 2>&1; echo "panel tests rc=$? $(tail -1 gpurun_out/${R}_dbg.log)"
