"""The map builder's row-ordering sort (sort.cu: one cooperative kernel with grid barriers,
or three kernels per pass) against numpy's stable argsort: exact permutation (stability
included) for the shapes the builder uses (27-bit neighbour masks of up to millions of rows)
and edge cases; many consecutive sorts cycle through the context's grid-barrier slots."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mk():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1904_08755_b200 as m
    return m


@pytest.mark.parametrize("n,bits", [(0, 27), (1, 27), (777, 9), (150_616, 27), (150_616, 8), (65_536, 16),
                                    (1_000_003, 27), (40_000, 31)])
def test_sort_perm_matches_stable_argsort(mk, n, bits):
    g = np.random.default_rng(n + bits)
    # skewed like neighbour masks: few distinct values dominate, many ties
    keys = np.where(g.random(n) < 0.7, g.integers(0, 64, n), g.integers(0, 1 << bits, n)).astype(np.int64)
    keys = (keys & ((1 << bits) - 1)).astype(np.int32)
    perm = mk.debug_sort_perm(torch.from_numpy(keys).cuda(), bits).cpu().numpy()
    assert np.array_equal(perm, np.argsort(keys, kind="stable"))


def test_sort_perm_many_calls_cycle_barrier_slots(mk):
    g = np.random.default_rng(5)
    keys = torch.from_numpy(g.integers(0, 1 << 27, 20_000).astype(np.int32)).cuda()
    want = np.argsort(keys.cpu().numpy(), kind="stable")
    outs = [mk.debug_sort_perm(keys, 27) for _ in range(300)]  # > 256 barrier slots
    for o in outs[::37] + outs[-3:]:
        assert np.array_equal(o.cpu().numpy(), want)
