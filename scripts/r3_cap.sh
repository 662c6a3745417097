set -u
run() { cp ablib/lib$1.so paper_1203_2739_b200/libspmv_b200.so; echo "== $1"; shift; timeout 600 python scripts/ab_opts.py "$@" 2>&1 | tail -6; }
for r in 1 2 3; do
run ROT c4 '{}'
run CAP100 c4 '{}'
done
cp ablib/libROT.so paper_1203_2739_b200/libspmv_b200.so
