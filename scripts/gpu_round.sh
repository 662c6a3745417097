set -x
python -m paper_1203_2739_b200.build > /dev/null
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/r42_pytest.log 2>&1; tail -2 gpurun_out/r42_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r42_bench.json 2> gpurun_out/r42_bench.err; tail -2 gpurun_out/r42_bench.err; cat gpurun_out/r42_bench.json
