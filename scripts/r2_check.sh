# Round-2 first check: GPU tests, smoke, C5 and C4 bench lines on the restructured library
set -u
R=${R:-r2a}
mkdir -p gpurun_out
python -m paper_1203_2739_b200.build > /dev/null
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${R}_pytest.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/${R}_pytest.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo "smoke rc=$? $(tail -1 gpurun_out/${R}_smoke.log)"
for c in c5 c4; do
  timeout 900 python bench.py --workload $c > gpurun_out/${R}_bench_$c.json 2> gpurun_out/${R}_bench_$c.err
  echo "bench $c rc=$?"
done
