set -u
# tests on the DYN1 build (the default), then the A/B
python -m paper_1203_2739_b200.build > /dev/null
timeout 1200 python -m pytest tests/test_gpu_panel.py tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_ranks.py -q -x --timeout 300 --timeout-method=thread 2>&1 | tail -3
AB="DYN0 DYN1" CFGS="c4 c5" ROUNDS=2 bash scripts/ab_lib.sh
