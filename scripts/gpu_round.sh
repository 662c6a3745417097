set -x
python -m paper_1203_2739_b200.build > /dev/null
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
cd scripts
timeout 300 python ab.py c4 panel
SPMV_LIB=/root/repo/ablib/vmax8.so timeout 300 python ab.py c4 panel | sed "s/^/vmax8 /"
SPMV_LIB=/root/repo/ablib/vmax32.so timeout 300 python ab.py c4 panel | sed "s/^/vmax32 /"
for w in c1 c2 c4; do python -c "
import os,sys; sys.path.insert(0,'..')
import synth, paper_1203_2739_b200 as sp
p=synth.make('$w'); h=sp.spmv_create(p.m,p.n,p.row_ptr,p.col,p.val,row_perm=p.row_perm,col_perm=p.col_perm,blocks=p.blocks)
i=sp.spmv_get_info(h); print('$w kernel', i['kernel'], 'panels', i['xs_panels'], 'pad', i['xs_pad_slots'], 'groups', i['xs_groups'])"; done
