"""GPU: tcgen05/TMA layout probe and the stripe permute kernel (K1), bit-exact."""

import numpy as np
import pytest
import torch

from oracle import ringref as R

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops():
    from paper_2311_09431_b200 import ops as _ops
    return _ops


def test_umma_probe_layouts(ops):
    g = torch.Generator(device="cuda").manual_seed(0)
    a, b, v = (torch.randn(128, 128, device="cuda", generator=g).bfloat16() for _ in range(3))
    import probe_lib
    s, o, y = probe_lib.probe_umma(a, b, v)
    torch.cuda.synchronize()
    s_ref = a.float() @ b.float().T
    o_ref = s.bfloat16().float() @ v.float()
    y_ref = b.float().T @ v.float()
    assert (s - s_ref).abs().max().item() < 1e-3
    assert (o - o_ref).abs().max().item() < 1e-2
    assert (y - y_ref).abs().max().item() < 1e-3


def test_umma_pair_probe_layouts(ops):
    """cta_group::2: A rows split over the CTA pair, B split by N, P and A staged in TMEM."""
    g = torch.Generator(device="cuda").manual_seed(1)
    a = torch.randn(256, 128, device="cuda", generator=g).bfloat16()
    b = torch.randn(128, 128, device="cuda", generator=g).bfloat16()
    v = torch.randn(128, 128, device="cuda", generator=g).bfloat16()
    import probe_lib
    s, o, s2 = probe_lib.probe_pair(a, b, v)
    torch.cuda.synchronize()
    s_ref = a.float() @ b.float().T
    assert (s - s_ref).abs().max().item() < 1e-3
    assert (o - s.bfloat16().float() @ v.float()).abs().max().item() < 1e-2
    assert (s2 - s_ref).abs().max().item() < 1e-3


@pytest.mark.parametrize("scheme", [0, 1])
@pytest.mark.parametrize("n_dev,n_seq,heads,d", [(4, 64, 2, 128), (8, 4096, 4, 64), (3, 12, 1, 64),
                                                 (2, 6, 3, 2)])
def test_permute_bit_exact(ops, scheme, n_dev, n_seq, heads, d):
    x = torch.randn(n_seq, heads, d, device="cuda").bfloat16()
    name = R.STRIPED if scheme == 1 else R.CONTIGUOUS
    want = np.concatenate(R.partition(x.view(torch.int16).cpu().numpy(), name, n_dev))
    got = torch.empty_like(x)
    ops.permute(x, got, n_dev, scheme, ops.PARTITION)
    assert np.array_equal(got.view(torch.int16).cpu().numpy(), want)
    back = torch.empty_like(x)
    ops.permute(got, back, n_dev, scheme, ops.GATHER)
    assert torch.equal(back.view(torch.int16), x.view(torch.int16))
    c = n_seq // n_dev
    for dev in range(n_dev):
        shard = torch.empty(c, heads, d, device="cuda", dtype=x.dtype)
        ops.permute(x, shard, n_dev, scheme, ops.PARTITION, dev)
        assert torch.equal(shard.view(torch.int16), got[dev * c:(dev + 1) * c].view(torch.int16))


def test_permute_companion_int64(ops):
    pos = torch.arange(32, device="cuda", dtype=torch.int64)
    out = torch.empty_like(pos)
    ops.permute(pos, out, 4, ops.STRIPED, ops.PARTITION)
    assert out.cpu().tolist() == R.permutation(R.STRIPED, 32, 4).tolist()
