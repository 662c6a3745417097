python -m paper_1203_2739_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_ranks.py -q -x 2>&1 | tail -15
