# Round-2 final evidence (no ncu; the captures are r2s3, scripts/r2_profile.sh):
# GPU tests, smoke, the five bench lines, the C3 split timing, the C5 power drift, the reference arm.
set -u
R=${R:-r2f}
mkdir -p gpurun_out
python -m paper_1203_2739_b200.build > /dev/null
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 300 --timeout-method=thread > gpurun_out/${R}_pytest.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/${R}_pytest.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo "smoke rc=$? $(tail -1 gpurun_out/${R}_smoke.log)"
for c in c5 c4 c3 c2 c1; do
  timeout 900 python bench.py --workload $c > gpurun_out/${R}_bench_$c.json 2> gpurun_out/${R}_bench_$c.err
  echo "bench $c rc=$?"
done
(cd scripts && timeout 600 python c3_split.py > ../gpurun_out/${R}_c3_split.json 2> ../gpurun_out/${R}_c3_split.err); echo "c3 split rc=$?"
(cd scripts && timeout 600 python c5_drift.py c5 10 > ../gpurun_out/${R}_c5_drift.jsonl 2> ../gpurun_out/${R}_c5_drift.err); echo "drift rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${R}_bench_ref.json 2> gpurun_out/${R}_bench_ref.err; echo "ref rc=$?"
