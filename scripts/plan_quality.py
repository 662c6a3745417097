"""Host-only panel-plan quality on C5's block geometry and C4 (no GPU):
groups, padding, deferrals, predicted y wavefronts per group access and x
gather sectors per group, at the production panel size."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import synth  # noqa: E402
from paper_1203_2739_b200 import testing as T  # noqa: E402


def run(name, p, blocks, target):
    t = time.time()
    st = T.pn_plan_check(p.m, p.n, p.row_ptr, p.col, p.val, blocks, target)
    g = st["groups"]
    out = dict(cfg=name, groups=g, pad_frac=st["pads"] / (32 * g), deferred_frac=st["deferred"] / st["entries"],
               ywf_col_order=st["y_wavefronts_natural"], ywf=st["y_wavefronts_coloured"],
               sectors_per_group=st["gather_sectors"] / g, plan_s=round(time.time() - t, 1))
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["c5blk", "c4"]
    if "c5blk" in which:
        # two blocks of C5's geometry: 1M rows, 980K interior columns, border
        # U{0..3} over 1.28M columns (non-square stand-in; plan statistics only)
        synth.PRESETS["_c5blk"] = lambda **kw: synth._sb(2, 1_000_000, 980_000, 640_000, 12, 20, 0, 3, **kw)
        p = synth.make("_c5blk", scramble=0)
        run("c5blk", p, p.blocks, 16384)
    if "c4" in which:
        p = synth.make("c4")
        run("c4", p, None, 16384)
