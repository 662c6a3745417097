set -u
# correctness of the default build first (panel tests), then the A/B
python -m paper_1203_2739_b200.build > /dev/null
timeout 600 python -m pytest tests/test_gpu_panel.py tests/test_gpu_variants.py -q -x --timeout 300 --timeout-method=thread 2>&1 | tail -1
AB="I8V8G4 I16V8G4 I16V8G8 I8V4G4 I16V4G8" CFGS="c4 c5" ROUNDS=2 bash scripts/ab_lib.sh
