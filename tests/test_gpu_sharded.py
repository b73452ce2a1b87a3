"""Row-sharded RRSVD on the device (SURVEY §8(e) level 2): K in-process shards through the C ABI
equal the single-call rrsvd_fixed_rank and the reference on config 1; the chol_inv entry point
equals the numpy restatement of its contract."""
import numpy as np
import pytest
import torch

import paper_1504_00992_b200 as P
from paper_1504_00992_b200.sharded import DeviceOps, LocalSum, ShardedRrsvd
from tests.conftest import cplx_randn
from tests.numpy_ops import chol_inv as np_chol_inv

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("l,shift", [(40, 0.0), (110, 10.0 * 2110), (400, 10.0 * 2400)])
def test_chol_inv_entry(ctx, l, shift):
    rng = np.random.default_rng(l)
    y = cplx_randn(rng, 2000, l)
    g = y.conj().T @ y
    t, nd = P.chol_inv(g, shift, ctx=ctx)
    want = np_chol_inv(g, shift)
    assert nd == 0
    assert np.linalg.norm(t - want) / np.linalg.norm(want) < 1e-12
    q = y @ t  # orthonormal up to the shift's perturbation
    assert np.linalg.norm(q.conj().T @ q - np.eye(l)) < 1e-6


@pytest.mark.parametrize("parts", [1, 2, 4])
def test_sharded_config1_matches_single_and_reference(ctx, ref, parts):
    n, k, p, q, seed = 512, 64, 10, 2, 7
    a = ref.structured_matrix(np.exp(-np.arange(n) / 10.0), n, 1, 2)
    ad = torch.from_numpy(a).cuda()
    bounds = [(n * r) // parts for r in range(parts + 1)]
    shards = [ad[bounds[r]:bounds[r + 1]].contiguous() for r in range(parts)]
    us, s, v, w = ShardedRrsvd(LocalSum(), DeviceOps(ctx)).fixed_rank(shards, n, k, p, q, seed)
    u = torch.cat(us).cpu().numpy()
    s, v = s.cpu().numpy(), v.cpu().numpy()
    one = P.rrsvd_fixed_rank(a, k, p, q, seed, ctx=ctx)
    u_r, s_r, v_r, w_r = ref.fixed_rank(a, k, p, q, seed)
    assert np.max(np.abs(s - one.sigma) / one.sigma) < 1e-12
    assert np.max(np.abs(s - s_r) / s_r) < 1e-10
    assert abs(w - w_r) < 1e-12
    rec, rec_r = (u * s) @ v.conj().T, (u_r * s_r) @ v_r.conj().T
    assert np.linalg.norm(rec - rec_r) / np.linalg.norm(rec_r) < 1e-10
