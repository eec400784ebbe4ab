"""Oracle-backed BlockOps for CPU tests of the ring driver's host logic (gloo).

Test infrastructure: the product driver (paper_2311_09431_b200.ring) is run unchanged
with this injected per-step compute so rotation, double buffering, LSE merging and the
travelling dK/dV accumulators can be checked over real process groups without a GPU.
"""

import threading

import numpy as np
import torch

from oracle import ringref as R


def _np(t):
    return t.detach().cpu().numpy().astype(np.float64)


class OracleBlockOps:
    # the fused backward adds into peer threads' home buffers: serialise the in-place adds
    # (the GPU path uses hardware reduce-adds)
    _add_lock = threading.Lock()

    def __init__(self):
        self.calls = []

    def fwd_block(self, q, k, v, o_acc, lse, out, scale, kind, first, last, tiles=None):
        self.calls.append(("fwd", int(kind), bool(first), bool(last)))
        c, hq, d = q.shape
        if tiles is not None and c % 128 == 0:  # what the kernel's counter reports
            cen = R.tile_census(int(kind), c, c, 128, 128)
            tiles += hq * (cen.n_full + cen.n_partial)
        if kind == R.FULLY_MASKED:
            o_blk = np.zeros((c, hq, d))
            l_blk = np.full((hq, c), -np.inf)
        else:
            st = R.Accum.fresh(c, hq, d)
            R.process_block(st, _np(q) * scale, _np(k), _np(v), kind, c, c)
            o_blk, l_blk = R.finalize(st, allow_dead=True)
        if first:
            o_new, l_new = o_blk, l_blk
        else:
            o_new, l_new = R.merge(_np(o_acc), _np(lse), o_blk, l_blk)
        lse.copy_(torch.tensor(l_new, dtype=lse.dtype))
        if last:
            out.copy_(torch.tensor(o_new, dtype=out.dtype))
        else:
            o_acc.copy_(torch.tensor(o_new, dtype=o_acc.dtype))

    def bwd_preprocess(self, out, dout, dsum, dq_acc):
        dsum.copy_(torch.tensor(np.einsum("shd,shd->hs", _np(dout), _np(out)), dtype=dsum.dtype))
        dq_acc.zero_()

    def bwd_block(self, q, k, v, dout, lse, dsum, dq_acc, dk_acc, dv_acc, scale, kind,
                  key_rows=None):
        self.calls.append(("bwd", int(kind)))
        dq, dk, dv = R.block_backward(_np(q), _np(k), _np(v), _np(dout), _np(lse), _np(dsum),
                                      int(kind), scale, key_rows=key_rows)
        dq_acc += torch.tensor(dq, dtype=dq_acc.dtype)
        with self._add_lock:
            dk_acc += torch.tensor(dk, dtype=dk_acc.dtype)
            dv_acc += torch.tensor(dv, dtype=dv_acc.dtype)

    def cast(self, src, dst):
        dst.copy_(src.to(dst.dtype))
