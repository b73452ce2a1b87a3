"""Row-sharded RRSVD (SURVEY §8(e) level 2) host logic on CPU: K in-process shards and gloo
world_size 2 reproduce the unsharded computation, and the algorithm matches the reference's
rrsvd_fixed_rank (randomized.cpp:109-122) on config-1's matrix."""
import os
import socket
import tempfile

import numpy as np
import pytest

from paper_1504_00992_b200.sharded import LocalSum, ShardedRrsvd
from tests.numpy_ops import NumpyOps

M, N, K, P, Q, SEED = 300, 200, 20, 6, 2, 7


def matrix():
    rng = np.random.default_rng(3)
    u, _ = np.linalg.qr(rng.standard_normal((M, N)) + 1j * rng.standard_normal((M, N)))
    v, _ = np.linalg.qr(rng.standard_normal((N, N)) + 1j * rng.standard_normal((N, N)))
    return (u * np.exp(-np.arange(N) / 8.0)) @ v.conj().T


def split(a, parts):
    bounds = [(a.shape[0] * r) // parts for r in range(parts + 1)]
    return [a[bounds[r]:bounds[r + 1]] for r in range(parts)]


def run_local(parts):
    a = matrix()
    us, s, v, w = ShardedRrsvd(LocalSum(), NumpyOps()).fixed_rank(split(a, parts), N, K, P, Q, SEED)
    return np.vstack(us), s, v, w


@pytest.mark.parametrize("parts", [2, 3, 5])
def test_local_shards_equal_unsharded(parts):
    u1, s1, v1, w1 = run_local(1)
    u, s, v, w = run_local(parts)
    assert np.max(np.abs(s - s1)) < 1e-13 * s1[0]
    assert abs(w - w1) < 1e-14
    assert np.linalg.norm((u * s) @ v.conj().T - (u1 * s1) @ v1.conj().T) < 1e-12 * np.linalg.norm(s1)


def test_sharded_matches_reference(ref):
    a = matrix()
    u, s, v, w = run_local(3)
    u_r, s_r, v_r, w_r = ref.fixed_rank(a, K, P, Q, SEED)
    assert np.max(np.abs(s - s_r) / s_r) < 1e-10
    assert abs(w - w_r) < 1e-12
    assert np.linalg.norm((u * s) @ v.conj().T - (u_r * s_r) @ v_r.conj().T) < 1e-10 * np.linalg.norm(s_r)


def _gloo_worker(rank, world, port_, outdir):
    import torch.distributed as dist

    from paper_1504_00992_b200.sharded import TorchSum
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port_}", rank=rank, world_size=world)
    shard = split(matrix(), world)[rank]
    us, s, v, w = ShardedRrsvd(TorchSum("cpu"), NumpyOps()).fixed_rank([shard], N, K, P, Q, SEED)
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), u=us[0], s=s, v=v, w=w)  # v: this rank's rows
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks_equal_unsharded():
    import torch.multiprocessing as mp
    u1, s1, v1, w1 = run_local(2)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port_ = sk.getsockname()[1]
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_gloo_worker, args=(2, port_, d), nprocs=2, join=True)
        z = [np.load(os.path.join(d, f"rank{r}.npz")) for r in range(2)]
    u = np.vstack([zz["u"] for zz in z])
    v = np.vstack([zz["v"] for zz in z])  # V is row-sharded like U
    for zz in z:  # replicated results identical on every rank
        assert np.array_equal(zz["s"], z[0]["s"]) and zz["w"] == z[0]["w"]
    assert v.shape == (N, K)
    s, w = z[0]["s"], float(z[0]["w"])
    assert np.max(np.abs(s - s1)) < 1e-13 * s1[0]
    assert abs(w - w1) < 1e-14
    assert np.linalg.norm((u * s) @ v.conj().T - (u1 * s1) @ v1.conj().T) < 1e-12 * np.linalg.norm(s1)
