set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r20_smoke.log 2>&1; tail -3 gpurun_out/r20_smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r20_pytest.log 2>&1
tail -15 gpurun_out/r20_pytest.log
timeout 900 python bench.py > gpurun_out/r20_bench.json 2> gpurun_out/r20_bench.err; tail -3 gpurun_out/r20_bench.err; cat gpurun_out/r20_bench.json
cd scripts
for w in c5 c4; do AB=1 timeout 600 python diag_c5.py $w > ../gpurun_out/r20_diag_$w.json 2>&1; cat ../gpurun_out/r20_diag_$w.json | tail -20; done
