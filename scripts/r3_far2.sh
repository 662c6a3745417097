set -u
run() { cp ablib/lib$1.so paper_1203_2739_b200/libspmv_b200.so; echo "== $1"; shift; timeout 900 python scripts/ab_opts.py "$@" 2>&1 | tail -4; }
for c in c4 c3; do for r in 1 2; do for v in ROT FAR R3 R6 R3D0 R1D0; do run $v $c '{}'; done; done; done
for v in ROT R3 R6 R3D0; do run $v c5 '{}'; done
cp ablib/libFAR.so paper_1203_2739_b200/libspmv_b200.so
