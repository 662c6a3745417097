set -u
for r in 1 2; do for v in PRO RTL1; do cp ablib/lib$v.so paper_1203_2739_b200/libspmv_b200.so; echo "== $v"; timeout 600 python scripts/ab_kernels.py c2 rowtile 2>&1 | tail -1; timeout 600 python scripts/ab_kernels.py c1 rowtile 2>&1 | tail -1; done; done
for v in PRO RTL1; do cp ablib/lib$v.so paper_1203_2739_b200/libspmv_b200.so; echo "== $v"; timeout 600 python scripts/ab_opts.py c4 '{"kernel": "rowtile"}' 2>&1 | tail -1; done
cp ablib/libPRO.so paper_1203_2739_b200/libspmv_b200.so
