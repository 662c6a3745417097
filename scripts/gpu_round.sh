mkdir -p gpurun_out
cd scripts
echo "main: $(timeout 300 python c3_split.py 2>&1 | grep -E 'cold' | tr -d '\n')"
echo "foldwarp: $(SPMV_LIB=$PWD/../ablib/foldwarp.so timeout 300 python c3_split.py 2>&1 | grep -E 'cold' | tr -d '\n')"
for m in 0 1 2 3 4; do echo "c4 mode $m $(SPMV_PN_MODE=$m timeout 300 python ab.py c4 panel 2>&1 | tail -1)"; done
