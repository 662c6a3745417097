set -u
for v in XSWARP XSW2 XSW512; do
  cp ablib/lib$v.so paper_1203_2739_b200/libspmv_b200.so
  echo "== $v"; timeout 600 python scripts/ab_kernels.py c2 rowtile xstaged 2>&1 | tail -2
done
