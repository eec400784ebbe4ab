"""The reference's schedule-structure tests (pkg/tests/test_simulator.py:100-207) run
against the GPU backend: compat.simulate_gpu (simulate, simulator.py:358-368) and
compat.run_schedule_gpu (run_schedule, simulator.py:237-277) with ringsim-shaped configs.

d_head is 64 here (the kernels support 64 / 128; the reference's tests use 4): every
structural property is independent of d.  Coverage-exactly-once is checked on what the
KERNELS computed, not on host bookkeeping: with q = 0 every allowed pair has score 0, and
one-hot values v[y] = e_y make output row x equal to (1 / #keys attended) on exactly the
keys attended -- a pair computed twice (or never) changes the row."""

from types import SimpleNamespace

import numpy as np
import pytest

from oracle import ringref as R

pytestmark = pytest.mark.gpu

ALGOS = ["ring", "striped"]


def cfg(algo, n_devices, n_seq, d_head=64, tile_q=2, tile_k=2, scale=False, seed=0,
        precision="double"):
    return SimpleNamespace(algo=algo, n_devices=n_devices, n_seq=n_seq, d_head=d_head,
                           tile_q=tile_q, tile_k=tile_k, scale=scale, seed=seed,
                           precision=precision, dtype=np.float64,
                           block_size=n_seq // n_devices)


@pytest.fixture(scope="module")
def compat():
    from paper_2311_09431_b200 import compat as c
    return c


@pytest.mark.parametrize("algo", ALGOS)
def test_block_rotation_invariant(compat, algo):  # test_simulator.py:100-107
    n = 4
    run = compat.simulate_gpu(cfg(algo, n, 16))
    for ws in run.stats:
        for i, rs in enumerate(ws.rounds):
            assert rs.round == i
            assert rs.block_index == (ws.device - i) % n


def test_ring_round2_mask_extremes(compat):  # test_simulator.py:110-120
    config = cfg("ring", 4, 32)
    run = compat.simulate_gpu(config)
    c = config.block_size
    by_device = {ws.device: ws.rounds[2] for ws in run.stats}
    assert by_device[1].block_index == 3
    assert by_device[1].tiles_skipped == by_device[1].tiles_total
    assert by_device[1].interactions_computed == 0
    assert by_device[1].kernel_tiles_computed == 0  # the kernel launched nothing
    assert by_device[3].block_index == 1
    assert by_device[3].tiles_skipped == 0
    assert by_device[3].interactions_computed == c * c


@pytest.mark.parametrize("algo", ALGOS)
def test_work_counter_bounds(compat, algo):  # test_simulator.py:123-131
    run = compat.simulate_gpu(cfg(algo, 4, 32, tile_q=2, tile_k=4))
    area = 2 * 4
    for ws in run.stats:
        for rs in ws.rounds:
            assert rs.tiles_skipped + rs.tiles_partial + rs.tiles_full == rs.tiles_total
            assert rs.interactions_required <= rs.interactions_computed
            assert rs.interactions_computed <= rs.tiles_total * area


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("n_devices,n_seq", [(4, 32), (2, 64), (8, 64), (3, 48)])
def test_kernel_coverage_exactly_once(compat, algo, n_devices, n_seq):
    """test_simulator.py:134-154, observed through the kernels' outputs."""
    d = 64
    q = np.zeros((n_seq, d))
    k = np.random.default_rng(1).standard_normal((n_seq, d))
    v = np.eye(n_seq, d)  # v[y] = e_y
    run = compat.simulate_gpu(cfg(algo, n_devices, n_seq), inputs=(q, k, v))
    want = np.tril(np.ones((n_seq, n_seq))) / np.arange(1, n_seq + 1)[:, None]
    got = run.output[:, :n_seq]
    assert np.max(np.abs(got - want)) <= 4e-3  # bf16 output rounding of 1 / (x + 1)
    assert np.all(got[np.triu_indices(n_seq, 1)] == 0)  # no key after the query
    total_required = sum(rs.interactions_required for ws in run.stats for rs in ws.rounds)
    assert total_required == n_seq * (n_seq + 1) // 2


@pytest.mark.parametrize("algo", ALGOS)
def test_simulate_seeded_inputs_and_oracle_error(compat, algo):
    """inputs=None draws random_qkv(n_seq, d_head, seed) exactly as the reference
    (simulator.py:133-135, 360-361); oracle_error (simulator.py:371-374) within bf16."""
    config = cfg(algo, 4, 512, d_head=128, tile_q=128, tile_k=128, scale=True, seed=5)
    run = compat.simulate_gpu(config)
    rng = np.random.default_rng(5)
    q, k, v = (rng.standard_normal((512, 128)) for _ in range(3))
    assert np.array_equal(run.q, q) and np.array_equal(run.k, k) and np.array_equal(run.v, v)
    assert run.layout.scheme.value == ("contiguous" if algo == "ring" else "striped")
    ref, _ = R.dense_forward(R.bf16_round(q / np.sqrt(128)), R.bf16_round(k), R.bf16_round(v),
                             1.0)
    assert float(np.max(np.abs(run.output - ref[:, 0]))) <= 2e-2
    # outputs stay in local order; gather(outputs) == output (layout.py:103-117)
    perm = R.permutation(R.STRIPED if algo == "striped" else R.CONTIGUOUS, 512, 4)
    assert np.array_equal(np.concatenate(run.outputs), run.output[perm])


@pytest.mark.parametrize("algo", ALGOS)
def test_run_schedule_gpu_rejects_like_the_reference(compat, algo):
    """run_schedule's ValueErrors (simulator.py:245-260)."""
    from paper_2311_09431_b200.layout import Layout
    config = cfg(algo, 4, 64)
    other = "striped" if algo == "ring" else "contiguous"
    sh = SimpleNamespace(q=np.zeros((16, 64)), k=np.zeros((16, 64)), v=np.zeros((16, 64)))
    with pytest.raises(ValueError):
        compat.run_schedule_gpu(config, SimpleNamespace(layout=Layout(other, 64, 4),
                                                         shards=[sh] * 4))
    mine = "contiguous" if algo == "ring" else "striped"
    with pytest.raises(ValueError):
        compat.run_schedule_gpu(config, SimpleNamespace(layout=Layout(mine, 64, 4),
                                                         shards=[sh] * 3))
    bad = SimpleNamespace(q=np.zeros((16, 32)), k=np.zeros((16, 32)), v=np.zeros((16, 32)))
    with pytest.raises(ValueError):
        compat.run_schedule_gpu(config, SimpleNamespace(layout=Layout(mine, 64, 4),
                                                         shards=[bad] * 4))
