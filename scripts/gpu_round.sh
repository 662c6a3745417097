set -x
mkdir -p gpurun_out
python -m paper_1203_2739_b200.build > /dev/null
python -c "import torch; p=torch.cuda.get_device_properties(0); print('persistingL2max', getattr(p,'persisting_l2_cache_max_size',None), 'L2', p.L2_cache_size)"
cd scripts
SPMV_L2_PERSIST_MB=48 K=64 KERNELS=panel timeout 300 python xs_probe.py 2>&1 | grep -E '"panel_ms"|Error' | sed "s/^/C5 persist48 /"
K=64 KERNELS=panel PROFILE_ONE=1 timeout 600 ncu --set full -k regex:panel -s 13 -c 1 -o ../gpurun_out/r30_pn_c5 python xs_probe.py > ../gpurun_out/r30_ncu.log 2>&1; tail -1 ../gpurun_out/r30_ncu.log
