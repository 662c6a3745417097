set -x
python -m paper_1203_2739_b200.build > /dev/null
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
SPMV_KERNEL=panel SPMV_PN_ROWS=700 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k split 2>&1 | tail -1
cd scripts
timeout 300 python c3_split.py 2>&1 | tail -9
python -c "
import sys; sys.path.insert(0,'..')
import synth, paper_1203_2739_b200 as sp
p=synth.make('c3'); h=sp.spmv_create(p.m,p.n,p.row_ptr,p.col,p.val,blocks=p.blocks,parts=p.parts,n_parts=p.n_parts); print(sp.spmv_get_info(h))"
