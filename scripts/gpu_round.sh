mkdir -p gpurun_out
python -m paper_1203_2739_b200.build > /dev/null
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
cd scripts
for L in vec main; do
  if [ $L = vec ]; then export SPMV_LIB=$PWD/../ablib/vec.so; else unset SPMV_LIB; fi
  echo "$L c4 $(timeout 300 python ab.py c4 panel 2>&1 | tail -1)"
  echo "$L c3split $(timeout 300 python c3_split.py 2>&1 | grep -E 'fused_cold|single_cold' | tr -d '\n')"
  echo "$L c5 $(timeout 300 python ab.py c5 panel 2>&1 | tail -1)"
done
echo "main c5 mode 25 $(SPMV_PN_MODE=25 timeout 300 python ab.py c5 panel 2>&1 | tail -1)"
