set -u
run() { cp ablib/lib$1.so paper_1203_2739_b200/libspmv_b200.so; echo "== $1"; shift; timeout 900 python scripts/ab_opts.py "$@" 2>&1 | tail -4; }
cp ablib/libCW.so paper_1203_2739_b200/libspmv_b200.so
timeout 900 python -m pytest tests/test_gpu_panel.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for r in 1 2 3; do for v in PRO CW; do run $v c5 '{}'; done; done
for r in 1 2; do for v in PRO CW; do run $v c4 '{}'; done; done
cp ablib/libCW.so paper_1203_2739_b200/libspmv_b200.so
