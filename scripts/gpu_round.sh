set -x
mkdir -p gpurun_out
cd scripts
timeout 600 python diag_c5.py c5 > ../gpurun_out/r6_diag.json 2>&1 && \
PROFILE_ONE=1 timeout 1200 ncu --set full --clock-control none -k regex:"csr_stream|spmv_pipe" -s 12 -c 3 -o ../gpurun_out/r6_prof python diag_c5.py c5 > ../gpurun_out/r6_ncu.log 2>&1
cd ..
cat gpurun_out/r6_diag.json; tail -3 gpurun_out/r6_ncu.log
