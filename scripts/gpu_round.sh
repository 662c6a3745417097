set -x
python -m paper_1203_2739_b200.build > /dev/null
timeout 300 python bench.py --workload c4 > gpurun_out/r63_c4.json 2>gpurun_out/r63_c4.err; python -c "import json;d=json.load(open('gpurun_out/r63_c4.json'));print('c4', d['value'], d['spmv_ms'], d['roofline']['frac'], d['parity'], d['config']['kernel'])"
cd scripts
for r in 8192 11000 16384 20000; do SPMV_PN_ROWS=$r timeout 300 python ab.py c4 panel | sed "s/^/rows $r /"; done
