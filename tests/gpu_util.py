"""Helpers for the -m gpu parity tests: run the CUDA path through the C ABI
(binding) and the oracle on the same seeded inputs."""
import numpy as np

import oracle
import paper_1203_2739_b200 as sp


def create(prob, **kw):
    return sp.spmv_create(prob.m, prob.n, prob.row_ptr, prob.col, prob.val, row_perm=prob.row_perm,
                          col_perm=prob.col_perm, blocks=prob.blocks,
                          parts=prob.parts if kw.pop("with_parts", True) else None,
                          n_parts=prob.n_parts, **kw)


PANEL = dict(kernel="panel")


def panel(rows):
    """spmv_options_t forcing the column-sorted panel kernel at `rows` y slots per panel."""
    return dict(kernel="panel", split_kernel="panel", panel_rows=rows)


def oracle_permuted(prob, x):
    """Oracle y and S for original-space x, mapped to PERMUTED space:
    y^[row_perm[i]] = y[i]; plus x^ (x^[col_perm[j]] = x[j])."""
    y, S = oracle.spmv(prob.row_ptr, prob.col, prob.val, x, nthreads=oracle.max_threads())
    if prob.row_perm is None:
        return oracle.permute_x(None, x), y, S
    return (oracle.permute_x(prob.col_perm, x), oracle.permute_x(prob.row_perm, y),
            oracle.permute_x(prob.row_perm, S))


def gpu_apply(h, xhat, m, flags=0, split=False):
    import torch
    xd = torch.from_numpy(np.ascontiguousarray(xhat)).cuda()
    yd = torch.full((m,), float("nan"), dtype=torch.float64, device="cuda")
    (sp.spmv_split_apply if split else sp.spmv_apply)(h, xd, yd, flags)
    torch.cuda.synchronize()
    return yd.cpu().numpy()


def assert_parity(y, yref, S, exact=False, what=""):
    if exact:
        bad = np.flatnonzero(y != yref)
        assert bad.size == 0, f"{what}: {bad.size} entries differ, first {bad[:5]} {y[bad[:5]]} vs {yref[bad[:5]]}"
        return
    nbad, worst, first = oracle.check(y, yref, S)
    assert nbad == 0, f"{what}: {nbad} entries beyond 1e-12*S (worst {worst:.3e}), first {first}: {y[first]} vs {yref[first]}"
