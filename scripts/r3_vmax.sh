set -u
run() { cp ablib/lib$1.so paper_1203_2739_b200/libspmv_b200.so; shift; echo "== $1 ${LIBV}"; timeout 600 python scripts/ab_opts.py "$@" 2>&1 | tail -6; }
for r in 1 2; do
LIBV=ROT run ROT c4 '{}' '{"panel_rows": 8300}' '{"panel_rows": 9000}'
LIBV=V24 run V24 c4 '{}' '{"panel_rows": 8300}' '{"panel_rows": 9500}'
LIBV=V16 run V16 c4 '{}' '{"panel_rows": 8300}' '{"panel_rows": 10400}'
done
cp ablib/libROT.so paper_1203_2739_b200/libspmv_b200.so
