# GPU test suite without -x (all failures listed) + smoke
set -u
R=${R:-r2b}
mkdir -p gpurun_out
python -m paper_1203_2739_b200.build > /dev/null
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/${R}_pytest.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/${R}_pytest.log)"
