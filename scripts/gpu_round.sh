mkdir -p gpurun_out
python -m paper_1203_2739_b200.build > /dev/null
cd scripts
for m in 0 24; do echo "c4 mode $m $(SPMV_PN_MODE=$m timeout 300 python ab.py c4 panel 2>&1 | tail -1)"; done
for m in 0 24; do echo "c5 mode $m $(SPMV_PN_MODE=$m timeout 300 python ab.py c5 panel 2>&1 | tail -1)"; done
for r in 18432 20480; do for m in 0 22; do echo "c5 rows $r mode $m $(SPMV_PN_ROWS=$r SPMV_PN_MODE=$m timeout 300 python ab.py c5 panel 2>&1 | tail -1)"; done; done
