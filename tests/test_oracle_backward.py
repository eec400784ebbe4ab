"""Pin the builder's backward restatement (NOT REFERENCE -- ringsim has no
backward) by torch fp64 autograd of the reference forward formula
(attention.py:121-143) and by central finite differences.  CPU only."""

import numpy as np
import pytest
import torch

from oracle import ringref as R


def _torch_causal(q, k, v, scale, group):
    # attention.py:137-143 restated in torch, per head with GQA expansion
    kk = k.repeat_interleave(group, dim=1)
    vv = v.repeat_interleave(group, dim=1)
    s = torch.einsum("qhd,khd->hqk", q, kk) * scale
    n = q.shape[0]
    s = s.masked_fill(~torch.tril(torch.ones(n, n, dtype=torch.bool)), float("-inf"))
    p = torch.softmax(s, dim=-1)
    return torch.einsum("hqk,khd->qhd", p, vv)


@pytest.mark.parametrize("hq,hkv", [(2, 2), (4, 2), (4, 1)])
def test_dense_backward_matches_autograd(hq, hkv):
    rng = np.random.default_rng(hq * 10 + hkv)
    n, d = 24, 8
    q, k, v, do = (rng.standard_normal(s) for s in ((n, hq, d), (n, hkv, d), (n, hkv, d), (n, hq, d)))
    scale = 1 / np.sqrt(d)
    tq, tk, tv = (torch.tensor(x, requires_grad=True) for x in (q, k, v))
    out = _torch_causal(tq, tk, tv, scale, hq // hkv)
    out.backward(torch.tensor(do))
    dq, dk, dv = R.dense_backward(q, k, v, do, scale)
    o, _ = R.dense_forward(q, k, v, scale)
    assert np.max(np.abs(o - out.detach().numpy())) <= 1e-12
    for got, want in ((dq, tq.grad), (dk, tk.grad), (dv, tv.grad)):
        assert np.max(np.abs(got - want.numpy())) <= 1e-12


def test_dense_backward_finite_differences():
    rng = np.random.default_rng(5)
    n, h, d = 6, 1, 4
    q, k, v, do = (rng.standard_normal((n, h, d)) for _ in range(4))
    scale = 0.7
    dq, dk, dv = R.dense_backward(q, k, v, do, scale)

    def loss(q_, k_, v_):
        return float((R.dense_forward(q_, k_, v_, scale)[0] * do).sum())

    eps = 1e-6
    for arr, grad, which in ((q, dq, 0), (k, dk, 1), (v, dv, 2)):
        for idx in [(0, 0, 0), (3, 0, 2), (5, 0, 3), (2, 0, 1)]:
            args = [q.copy(), k.copy(), v.copy()]
            args[which][idx] += eps
            up = loss(*args)
            args[which][idx] -= 2 * eps
            dn = loss(*args)
            assert (up - dn) / (2 * eps) == pytest.approx(grad[idx], abs=1e-7)


@pytest.mark.parametrize("scheme", [R.STRIPED, R.CONTIGUOUS])
@pytest.mark.parametrize("n_dev", [1, 2, 4])
def test_ring_backward_equals_dense(scheme, n_dev):
    rng = np.random.default_rng(n_dev)
    n, hq, hkv, d = 32, 4, 2, 8
    q, k, v, do = (rng.standard_normal(s) for s in ((n, hq, d), (n, hkv, d), (n, hkv, d), (n, hq, d)))
    scale = 1 / np.sqrt(d)
    o, lse = R.dense_forward(q, k, v, scale)
    got = R.ring_backward(q, k, v, do, o, lse, n_dev, scheme, scale)
    want = R.dense_backward(q, k, v, do, scale)
    for g, w in zip(got, want):
        assert np.max(np.abs(g - w)) <= 1e-12


@pytest.mark.parametrize("scheme", [R.STRIPED, R.CONTIGUOUS])
def test_ring_forward_multihead_gqa_equals_dense(scheme):
    rng = np.random.default_rng(9)
    n, hq, hkv, d = 48, 4, 2, 8
    q, k, v = (rng.standard_normal(s) for s in ((n, hq, d), (n, hkv, d), (n, hkv, d)))
    o, lse, _ = R.ring_forward(q, k, v, 4, scheme, 0.5, tile_q=4, tile_k=6)
    od, lsed = R.dense_forward(q, k, v, 0.5)
    assert np.max(np.abs(o - od)) <= 1e-12
    assert np.max(np.abs(lse - lsed)) <= 1e-12
