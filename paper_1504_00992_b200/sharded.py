"""Row-sharded single-matrix RRSVD (SURVEY §8(e) level 2: config-4 interpretation (i) and the
config-5 sweep across GPUs).

A (m x n) is split by row blocks A_g.  The reference algorithm (randomized.cpp:88-122) is kept
step for step; only the reductions over the row dimension cross shards:

  Y_g = A_g Omega                        local (Omega replicated: same seed on every rank)
  QR of the distributed Y                shifted CholeskyQR: G = sum_g Y_g^H Y_g (all-reduce of
                                         l x l), T = chol_inv(G) replicated, Q_g = Y_g T
  Z = A^H Q = sum_g A_g^H Q_g            all-reduce of n x l; QR of Z replicated
  Y_g = A_g Q~                           local
  B^H = A^H Q                            all-reduce of n x l; SVD of B^H replicated (n x l)
  U_g = Q_g U_B                          local;  ||A||^2 = sum_g ||A_g||^2 (all-reduce)

Communication is O(q n l) per decimation against O(q m n l / G) of GEMM work per rank.  Every
rank may hold several shards (`shards` list): the local partial sums are added in a fixed order
before the cross-rank all-reduce, so K shards on one GPU (a loopback run) and K ranks with one
shard each compute the same sums up to the all-reduce's association.

`ops` supplies the device primitives: gemm, chol_inv, svd, omega, sumsq (DeviceOps runs them
through librrsvd_b200; the CPU tests plug numpy in).  `comm` sums a tensor over ranks
(LocalSum: one process; TorchSum: torch.distributed.all_reduce over NCCL or gloo).
"""
from __future__ import annotations

import numpy as np

from . import api
from ._lib import OMEGA_REFERENCE

FULL_PASSES, SPAN_PASSES = 4, 2  # pipeline.cuh kFullPasses / kSpanPasses


class LocalSum:
    """Single process: the sum over ranks is the identity."""
    world = 1
    rank = 0

    def allreduce(self, t):
        return t


class TorchSum:
    """torch.distributed all-reduce (SUM) on `device` ("cuda:i" for NCCL, "cpu" for gloo);
    complex tensors travel as their real view."""

    def __init__(self, device="cpu"):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.device = torch, dist, device
        self.rank, self.world = dist.get_rank(), dist.get_world_size()

    def allreduce(self, t):
        """Sum over ranks; numpy in -> numpy out (host arrays travel through `device`)."""
        torch = self.torch
        was_np = isinstance(t, np.ndarray)
        if was_np:
            t = torch.from_numpy(np.ascontiguousarray(t))
        t = t.to(self.device).contiguous()
        view = torch.view_as_real(t) if t.is_complex() else t
        self.dist.all_reduce(view)
        return t.cpu().numpy() if was_np else t


class DeviceOps:
    """Primitives on the B200 through the C ABI (torch CUDA tensors in and out)."""

    def __init__(self, ctx, device="cuda"):
        import torch
        self.ctx, self.device, self.torch = ctx, device, torch

    def gemm(self, a, adj_a, b):
        return api.gemm(a, adj_a, b, ctx=self.ctx)

    def chol_inv(self, g, shift_scale):
        return api.chol_inv(g, shift_scale, ctx=self.ctx)[0]

    def svd(self, a):
        return api.svd_full(a, ctx=self.ctx)

    def omega(self, n, l, seed, mode):
        return api.gaussian_test_matrix(n, l, seed, mode, ctx=self.ctx, device=self.device)

    def sumsq(self, a):
        return api.frobenius_norm(a, ctx=self.ctx) ** 2

    def zeros_like(self, a):
        return self.torch.zeros_like(a)

    def add(self, a, b):
        return a + b


class ShardedRrsvd:
    def __init__(self, comm, ops):
        self.comm, self.ops = comm, ops

    # -- reductions over the row dimension: fixed-order local sum, then across ranks
    def _rowsum(self, parts):
        acc = parts[0]
        for p in parts[1:]:
            acc = self.ops.add(acc, p)
        return self.comm.allreduce(acc)

    def _orth_sharded(self, ys, m_total, passes):
        """Shifted CholeskyQR over row-sharded Y (pipeline.cu orth_many's schedule)."""
        l = ys[0].shape[1]
        for p in range(passes):
            g = self._rowsum([self.ops.gemm(y, True, y) for y in ys])
            t = self.ops.chol_inv(g, 10.0 * (m_total + l) if p < min(passes, 2) else 0.0)
            ys = [self.ops.gemm(y, False, t) for y in ys]
        return ys

    def _orth_replicated(self, z, passes):
        return self._orth_sharded([z], z.shape[0], passes)[0]

    def sketched_svd(self, shards, n: int, l: int, q: int, seed: int, mode: int = OMEGA_REFERENCE):
        """rrsvd_sketched_svd (randomized.cpp:101-107) of the row-stacked shards.
        Returns (U row blocks, sigma (l), V (n x l), ||A||_F^2)."""
        ops = self.ops
        m_local = sum(a.shape[0] for a in shards)
        m_total = int(float(self.comm.allreduce(np.array([m_local], np.float64))[0]))
        if l > min(m_total, n):
            raise api.ContractViolation("randomized_range_finder: l exceeds min(m, n)")
        om = ops.omega(n, l, seed, mode)
        inter = SPAN_PASSES if q > 0 else FULL_PASSES
        qs = self._orth_sharded([ops.gemm(a, False, om) for a in shards], m_total, inter)
        for j in range(q):
            z = self._rowsum([ops.gemm(a, True, qg) for a, qg in zip(shards, qs)])
            qt = self._orth_replicated(z, SPAN_PASSES)
            qs = self._orth_sharded([ops.gemm(a, False, qt) for a in shards], m_total,
                                    SPAN_PASSES if j + 1 < q else FULL_PASSES)
        bh = self._rowsum([ops.gemm(a, True, qg) for a, qg in zip(shards, qs)])  # B^H = A^H Q
        u_z, sigma, v_z = ops.svd(bh)  # B^H = U_z S V_z^H  =>  B = V_z S U_z^H
        us = [ops.gemm(qg, False, v_z) for qg in qs]  # U = Q U_B, U_B = V_z
        total_sq = float(self.comm.allreduce(np.array([sum(ops.sumsq(a) for a in shards)], np.float64))[0])
        return us, sigma, u_z, total_sq

    def fixed_rank(self, shards, n: int, k: int, p: int, q: int, seed: int, mode: int = OMEGA_REFERENCE):
        """rrsvd_fixed_rank (randomized.cpp:109-122): (U row blocks (m_g x k), sigma (k), V (n x k), w)."""
        if k < 2 or p < 2:
            raise api.ContractViolation("rrsvd_fixed_rank: requires k >= 2 and p >= 2")
        us, sigma, v, total_sq = self.sketched_svd(shards, n, k + p, q, seed, mode)
        s = np.asarray(sigma.cpu() if hasattr(sigma, "cpu") else sigma)[:k]
        w = min(max(1.0 - float(np.sum(s ** 2)) / total_sq, 0.0), 1.0) if total_sq > 0 else 0.0
        return [u[:, :k] for u in us], sigma[:k], v[:, :k], w
