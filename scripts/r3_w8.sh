set -u
run() { cp ablib/lib$1.so paper_1203_2739_b200/libspmv_b200.so; echo "== $1"; shift; timeout 900 python scripts/ab_opts.py "$@" 2>&1 | tail -6; }
for r in 1 2; do
run PRO c4 '{}'
run W8N c4 '{"panel_rows": 5600}' '{"panel_rows": 4150}' '{"panel_rows": 6700}'
run PRO c3 '{}'
run W8N c3 '{"panel_rows": 1800}' '{"panel_rows": 3600}'
done
cp ablib/libPRO.so paper_1203_2739_b200/libspmv_b200.so
