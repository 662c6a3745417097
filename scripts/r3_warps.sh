# Panel CTAs of 4 / 8 / 16 warps (independent epoch barriers per CTA, several CTAs per SM)
# on C4's parts and C4/C5: prebuilt ablib/libW<n>.so, panel_rows options per variant.
set -u
mkdir -p gpurun_out
run() {  # lib cfg opts...
  cp ablib/lib$1.so paper_1203_2739_b200/libspmv_b200.so
  shift
  timeout 600 python scripts/ab_opts.py "$@" 2>&1 | tail -8
}
for r in 1 2; do
run W16 c4 '{}'
run W8 c4 '{"panel_rows": 8300}' '{"panel_rows": 5600}' '{"panel_rows": 4150}'
run W4 c4 '{"panel_rows": 4150}' '{"panel_rows": 2800}' '{"panel_rows": 2100}'
done
run W16 c5 '{}'
run W8 c5 '{"panel_rows": 8192}'
run W4 c5 '{"panel_rows": 4096}'
cp ablib/libW16.so paper_1203_2739_b200/libspmv_b200.so
