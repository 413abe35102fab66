"""GPU parity of the embedding bag (exmy_embedding_bag; reading D25; SURVEY
8(f) row 3) against the oracle: sum / mean / per-sample weights, per-tensor
and per-row metadata, formats of width 3..9, ragged and empty bags, forced
generic decode.  Bit-exact (the accumulation order is part of D25)."""
import numpy as np
import pytest
import torch

import workloads as W

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(scope="module")
def exmy():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2405_13938_b200 as m
    m.force_generic(False)
    return m


def table(exmy, orc, rows, cols, fmt, seed, per_row):
    t = W.f32_embedding(rows, cols, seed=seed)
    t = t * torch.exp2(torch.randint(-6, 6, (rows, 1), generator=torch.Generator().manual_seed(seed)).float())
    bits = W.to_bits(t)
    d = t.to(DEV)
    if per_row:
        meta = orc.block_max_exponent(bits, (1, cols))
        p = exmy.encode_blocked(d, fmt, torch.from_numpy(meta.copy()).to(DEV), (1, cols), axis="cols")
        return p, meta.reshape(-1)
    e = orc.emax(orc.histogram(bits))
    return exmy.encode(d, fmt, e, axis="cols"), np.array([e], np.uint8)


@pytest.mark.parametrize("fmt", [(4, 2), (3, 1), (2, 4), (1, 1), (5, 3), (8, 0), (0, 8), (3, 3)],
                         ids=lambda f: f"e{f[0]}m{f[1]}")
@pytest.mark.parametrize("per_row", [False, True])
def test_bag_parity(exmy, orc, fmt, per_row):
    rows, cols = 500, 136
    p, meta = table(exmy, orc, rows, cols, fmt, fmt[0] * 9 + fmt[1], per_row)
    packed = p.data.cpu().numpy()
    rng = np.random.default_rng(fmt[1])
    sizes = rng.integers(0, 40, size=300)
    sizes[:4] = [0, 1, 2, 77]
    offsets = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    idx = rng.integers(0, rows, size=int(offsets[-1])).astype(np.int64)
    w = rng.standard_normal(idx.size).astype(np.float32)
    for mode in ("sum", "mean"):
        for weights in (None, w):
            got = exmy.embedding_bag(p, torch.from_numpy(idx), torch.from_numpy(offsets),
                                     None if weights is None else torch.from_numpy(weights), mode=mode)
            ref = orc.embedding_bag(packed, (rows, cols), fmt, meta, idx, offsets, weights, mode)
            np.testing.assert_array_equal(got.cpu().numpy().view(np.uint32), ref.view(np.uint32),
                                          err_msg=f"{mode} weights={weights is not None}")


def test_bag_force_generic(exmy, orc):
    rows, cols = 100, 64
    p, meta = table(exmy, orc, rows, cols, (3, 2), 4, False)
    idx = np.arange(rows, dtype=np.int64)[::-1].copy()
    offsets = np.array([0, 10, 10, 55, 100], np.int64)
    ref = orc.embedding_bag(p.data.cpu().numpy(), (rows, cols), (3, 2), meta, idx, offsets)
    exmy.force_generic(True)
    try:
        got = exmy.embedding_bag(p, torch.from_numpy(idx), torch.from_numpy(offsets))
    finally:
        exmy.force_generic(False)
    np.testing.assert_array_equal(got.cpu().numpy().view(np.uint32), ref.view(np.uint32))


def test_bag_equals_gather_sum(exmy):
    """sum over a one-index bag == the gathered row; agrees with decode_rows"""
    t = W.f32_embedding(1000, 128, seed=9).to(DEV)
    p = exmy.encode(t, "e4m2", axis="cols")
    idx = torch.tensor([5, 999, 0, 5], dtype=torch.int64)
    rows = exmy.decode_rows(p, idx)
    bag = exmy.embedding_bag(p, idx, torch.arange(5, dtype=torch.int64))
    assert torch.equal(bag, rows)
