set -u
run() { cp ablib/lib$1.so paper_1203_2739_b200/libspmv_b200.so; echo "== $1"; shift; timeout 900 python scripts/ab_opts.py "$@" 2>&1 | tail -4; }
for r in 1 2 3; do for v in PRO S8T8; do run $v c5 '{}'; done; done
for v in PRO S8T8; do run $v c4 '{}'; done
cp ablib/libPRO.so paper_1203_2739_b200/libspmv_b200.so
