set -u
run() { cp ablib/lib$1.so paper_1203_2739_b200/libspmv_b200.so; shift; timeout 600 python scripts/ab_opts.py "$@" 2>&1 | tail -6; }
for r in 1 2; do
run BASE c4 '{}' '{"panel_rows": 16600}'
run ROT c4 '{}' '{"panel_rows": 16600}' '{"panel_rows": 16384}' '{"panel_rows": 13000}'
run BASE c3 '{}'
run ROT c3 '{}'
done
cp ablib/libROT.so paper_1203_2739_b200/libspmv_b200.so
