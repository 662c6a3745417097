set -u
R=${R:-r2j}
mkdir -p gpurun_out
python -m paper_1203_2739_b200.build > /dev/null
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 300 --timeout-method=thread > gpurun_out/${R}_pytest.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/${R}_pytest.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo "smoke rc=$? $(tail -1 gpurun_out/${R}_smoke.log)"
