"""rrsvd_b200_state_upload / _download: the whole MpsState (mps.hpp:31-41) in one
call each way — bit-exact round trip, agreement with the per-site entry points, pinned torch
buffers, and the contract checks of the reference constructor (bond dimensions must chain)."""
import numpy as np
import pytest
import torch

from paper_1504_00992_b200 import ContractViolation
from paper_1504_00992_b200 import models as M
from paper_1504_00992_b200.tebd import DeviceMps

pytestmark = pytest.mark.gpu


def test_state_round_trip_bit_exact(ctx):
    dims = [2, 3, 4, 3, 2]
    g, l = M.synthetic_saturated_mps(dims, 6, seed=3)
    mps = DeviceMps(dims, 6, 0.0, ctx=ctx)
    mps.upload(g, l)
    assert mps.all_dims() == [x.shape for x in g]
    out_g = [np.empty_like(x) for x in g]
    out_l = [np.empty_like(x) for x in l]
    mps.download(out_g, out_l)
    for a, b in zip(g, out_g):
        assert np.array_equal(a, b)
    for a, b in zip(l, out_l):
        assert np.array_equal(a, b)
    for s in range(len(dims)):  # the per-site entry points see the same state
        assert np.array_equal(mps.gamma(s), g[s])


def test_state_round_trip_pinned_torch(ctx):
    dims = [20] * 6
    g, l = M.synthetic_saturated_mps(dims, 40, seed=4)
    pg = [torch.from_numpy(x).pin_memory() for x in g]
    pl = [torch.from_numpy(x).pin_memory() for x in l]
    mps = DeviceMps(dims, 40, 0.0, ctx=ctx)
    mps.upload(pg, pl)
    og = [torch.empty(x.shape, dtype=torch.complex128).pin_memory() for x in g]
    ol = [torch.empty(x.shape, dtype=torch.float64).pin_memory() for x in l]
    mps.download(og, ol)
    assert all(np.array_equal(a, b.numpy()) for a, b in zip(g, og))
    assert all(np.array_equal(a, b.numpy()) for a, b in zip(l, ol))


def test_state_upload_rejects_broken_chain(ctx):
    dims = [2, 2, 2]
    g, l = M.synthetic_saturated_mps(dims, 2, seed=5)
    bad = [g[0], np.zeros((3, 2, 1), np.complex128), g[2]]  # left dim 3 != right dim of site 0
    mps = DeviceMps(dims, 2, 0.0, ctx=ctx)
    with pytest.raises(ContractViolation):
        mps.upload(bad, l)


def test_state_roundtrip_pipelined(ctx):
    """rrsvd_b200_state_roundtrip: the state goes device -> pinned host -> device per site on two
    streams; the host buffers then hold it bit-exactly and the device state is unchanged (a
    following step sees the same state)."""
    dims = [20] * 8
    g, l = M.synthetic_saturated_mps(dims, 40, seed=5)
    mps = DeviceMps(dims, 40, 0.0, ctx=ctx)
    mps.upload(g, l)
    hg = [torch.zeros(x.shape, dtype=torch.complex128).pin_memory() for x in g]
    hl = [torch.zeros(x.shape, dtype=torch.float64).pin_memory() for x in l]
    mps.roundtrip(hg, hl)
    for a, b in zip(g, hg):
        assert np.array_equal(a, b.numpy())
    for a, b in zip(l, hl):
        assert np.array_equal(a, b.numpy())
    og = [np.empty_like(x) for x in g]
    ol = [np.empty_like(x) for x in l]
    mps.download(og, ol)
    for a, b in zip(g, og):
        assert np.array_equal(a, b)
    for a, b in zip(l, ol):
        assert np.array_equal(a, b)
