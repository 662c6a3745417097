# Full GPU suite (per-test timeout), smoke, and the C5/C4/C2 bench lines
set -u
R=${R:-r2e}
mkdir -p gpurun_out
python -m paper_1203_2739_b200.build > /dev/null
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 300 --timeout-method=thread > gpurun_out/${R}_pytest.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/${R}_pytest.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo "smoke rc=$? $(tail -1 gpurun_out/${R}_smoke.log)"
for c in ${CFGS:-c2 c4 c5}; do
  timeout 900 python bench.py --workload $c > gpurun_out/${R}_bench_$c.json 2> gpurun_out/${R}_bench_$c.err
  echo "bench $c rc=$?"
done
