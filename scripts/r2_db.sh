set -u
mkdir -p gpurun_out
python -m paper_1203_2739_b200.build > /dev/null
for L in LAZY EAGER; do
  echo "== CUDA_MODULE_LOADING=$L"
  CUDA_MODULE_LOADING=$L timeout 300 python scripts/db_debug.py c3s 2 2>&1 | tail -30
done
CUDA_MODULE_LOADING=LAZY timeout 300 python scripts/db_debug.py c3 8 2>&1 | tail -30
