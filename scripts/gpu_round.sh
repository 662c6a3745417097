python -m paper_1203_2739_b200.build > /dev/null
timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_xstage.py tests/test_gpu_parity.py -q -x -k "panel or c5_like or split or edge" 2>&1 | tail -15
echo "memcheck rc=$?"
