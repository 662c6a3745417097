set -u
mkdir -p gpurun_out
python -m paper_1203_2739_b200.build > /dev/null
timeout 300 python scripts/db_debug.py c3 8 2>&1 | tail -40
echo "== EAGER"
CUDA_MODULE_LOADING=EAGER timeout 300 python scripts/db_debug.py c3 8 2>&1 | tail -12
echo "== c3 4"
timeout 300 python scripts/db_debug.py c3 4 2>&1 | tail -12
