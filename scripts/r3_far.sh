set -u
run() { cp ablib/lib$1.so paper_1203_2739_b200/libspmv_b200.so; echo "== $1"; shift; timeout 900 python scripts/ab_opts.py "$@" 2>&1 | tail -4; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_panel.py -x -q 2>&1 | tail -3
for r in 1 2; do
run ROT c4 '{}'
run FAR c4 '{}'
run ROT c3 '{}'
run FAR c3 '{}'
done
run ROT c5 '{}'
run FAR c5 '{}'
cp ablib/libFAR.so paper_1203_2739_b200/libspmv_b200.so
