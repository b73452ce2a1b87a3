"""Row-sharded single-matrix RRSVD (SURVEY §8(e) level 2: config-4 interpretation (i) and the
config-5 sweep across GPUs).

A (m x n) is split by row blocks A_g.  The reference algorithm (randomized.cpp:88-122) is kept
step for step; only the reductions over the row dimension cross shards:

  Y_g = A_g Omega                        local (Omega replicated: same seed on every rank)
  QR of the distributed Y                shifted CholeskyQR: G = sum_g Y_g^H Y_g (all-reduce of
                                         l x l), T = chol_inv(G) replicated, Q_g = Y_g T
  Z = A^H Q = sum_g A_g^H Q_g            all-reduce of n x l; QR of Z row-sharded over the ranks
                                         (each its n/G rows), the orthonormal rows all-gathered
  Y_g = A_g Q~                           local
  B^H = A^H Q                            summed over ranks, then each rank keeps its row block
                                         of the n rows: B^H = Q_b X by a row-sharded CholeskyQR
                                         (l x l Gram all-reduce), X = Q_b^H B^H (l x l all-reduce),
                                         the SVD of the l x l X^H = W S K^H replicated (small):
                                         U_B = W, V = Q_b K row-sharded (pipeline.cu assemble_many's
                                         algorithm, distributed — no rank holds or factors n x l)
  U_g = Q_g U_B                          local;  ||A||^2 = sum_g ||A_g||^2 (all-reduce)

The CholeskyQR passes follow the device's adaptive schedule (pipeline.cu orth_many_adaptive): the
first, shifted pass reports whether a pivot fell near the shift (rrsvd_b200_chol_inv_flags);
only then do the extra passes run (full: 4 passes -> 2; the power iteration's bases: 4 -> 1 for a
well-conditioned Y).

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

FULL_PASSES, SPAN_PASSES, ROBUST_SPAN_PASSES = 4, 2, 3  # pipeline.cuh kFullPasses / kSpanPasses / kRobustSpanPasses


def _adjoint(x):
    """x^H as a dense array (torch: the conjugation materialised, not a conj-bit view)."""
    if isinstance(x, np.ndarray):
        return np.ascontiguousarray(x.conj().T)
    return x.conj().T.resolve_conj().contiguous()


class LocalSum:
    """Single process: the sum over ranks is the identity."""
    world = 1
    rank = 0

    def allreduce(self, t):
        return t

    def row_block(self, n):
        return 0, n

    def allgather_rows(self, block, n):
        return block


class TorchSum:
    """torch.distributed all-reduce (SUM) on `device` ("cuda:i" for NCCL, "cpu" for gloo);
    complex tensors travel as their real view."""

    def __init__(self, device="cpu"):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.device = torch, dist, device
        self.rank, self.world = dist.get_rank(), dist.get_world_size()

    def row_block(self, n):
        """This rank's rows [r0, r1) of an n-row replicated quantity."""
        return (n * self.rank) // self.world, (n * (self.rank + 1)) // self.world

    def allgather_rows(self, block, n):
        """The row blocks of all ranks (row_block order) stacked into the n-row whole."""
        torch = self.torch
        was_np = isinstance(block, np.ndarray)
        t = torch.from_numpy(np.ascontiguousarray(block)) if was_np else block
        t = t.to(self.device).contiguous()
        parts = []
        for r in range(self.world):
            r0, r1 = (n * r) // self.world, (n * (r + 1)) // self.world
            parts.append(torch.empty((r1 - r0,) + tuple(t.shape[1:]), dtype=t.dtype, device=self.device))
        view = (lambda u: torch.view_as_real(u)) if t.is_complex() else (lambda u: u)
        self.dist.all_gather([view(p) for p in parts], view(t))
        out = torch.cat(parts)
        return out.cpu().numpy() if was_np else out

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
    """Primitives on the B200 through the C ABI (torch CUDA tensors in and out).  prepare(shards)
    puts the shards on the INT8-emulated A-products (csrc/ozaki.cuh) when the library would use
    them for a batch of that size (RRSVD_B200_OZAKI, both sides >= 512, >= 8e6 entries): their
    residue planes are built once and every later gemm with that shard reuses them."""

    MIN_WORK = 8.0e6           # ozaki.cu ozaki_min_work
    MAX_BYTES = 32 * 2 ** 30   # ozaki.cu ozaki_max_bytes
    MAX_K = 32768              # int32 accumulators: inner dimension per emulated product

    def __init__(self, ctx, device="cuda"):
        import torch
        self.ctx, self.device, self.torch = ctx, device, torch
        self._oz = {}
        self._stream = set()

    def prepare(self, shards):
        """Shards whose residue planes fit the budget are prepared once for all their products;
        the others (wider than MAX_K columns, or beyond the budget: C4(i)'s 80000^2) are streamed —
        each product prepares its K-chunks, multiplies and releases them (the preparation then
        costs ~2x a product, still ~3x less than the FP64 product at these shapes)."""
        work = sum(float(a.shape[0]) * a.shape[1] for a in shards)
        if work < self.MIN_WORK:
            return
        used = 0.0
        for a in shards:
            m, n = a.shape
            t = api.ozaki_usable(m, min(n, self.MAX_K))
            if t == 0:
                continue
            planes = 2.0 * t * ((m + 127) // 128) * ((n + 127) // 128) * 16384
            if n <= self.MAX_K and used + planes <= self.MAX_BYTES:
                self._oz[a.data_ptr()] = api.OzakiOperator(a, t, ctx=self.ctx)
                used += planes
            else:
                self._stream.add((a.data_ptr(), t))

    def release(self):
        for op in self._oz.values():
            op.close()
        self._oz.clear()
        self._stream.clear()

    def _streamed(self, a, adj_a, b, t):
        """op(a) @ b by K-chunks of at most MAX_K columns of a, each prepared, applied, released."""
        m, n = a.shape
        nch = -(-n // self.MAX_K)
        out = None
        for c in range(nch):
            k0, k1 = (n * c) // nch, (n * (c + 1)) // nch
            op = api.OzakiOperator(a, t, ctx=self.ctx, col0=k0, ncols=k1 - k0)
            try:
                if adj_a:  # rows k0..k1 of A^H b: one chunk each
                    if out is None:
                        out = self.torch.empty((n, b.shape[1]), dtype=b.dtype, device=b.device)
                    op.mul(True, b, out=out[k0:k1])
                else:      # A b = sum over chunks of A[:, k0:k1] b[k0:k1]
                    if out is None:
                        out = self.torch.empty((m, b.shape[1]), dtype=b.dtype, device=b.device)
                    op.mul(False, b[k0:k1].contiguous(), out=out, accumulate=c > 0)
            finally:
                op.close()
        return out

    def gemm(self, a, adj_a, b):
        key = a.data_ptr() if hasattr(a, "data_ptr") else None
        op = self._oz.get(key) if key is not None else None
        if op is not None and op.a.data_ptr() == a.data_ptr() and tuple(op.a.shape) == tuple(a.shape):
            return op.mul(adj_a, b)
        for k, t in self._stream:
            if k == key:
                return self._streamed(a, adj_a, b, t)
        return api.gemm(a, adj_a, b, ctx=self.ctx)

    def chol_inv(self, g, shift_scale):
        t, _, ill = api.chol_inv(g, shift_scale, ctx=self.ctx, flags=True)
        return t, ill

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

    def _pass(self, ys, shift_scale):
        g = self._rowsum([self.ops.gemm(y, True, y) for y in ys])
        t, ill = self.ops.chol_inv(g, shift_scale)
        return [self.ops.gemm(y, False, t) for y in ys], ill

    def _orth_sharded(self, ys, m_total, passes):
        """CholeskyQR over row-sharded Y, the device's adaptive schedule (orth_many_adaptive):
        full = shifted | [ill] shifted, plain | plain;  span = shifted | [ill] shifted;
        robust span = shifted | [ill] shifted, plain, plain."""
        l = ys[0].shape[1]
        shift = 10.0 * (m_total + l)
        a, ill = self._pass(ys, shift)
        if ill:  # (ill is computed from the all-reduced Gram: the same decision on every rank)
            a, _ = self._pass(a, shift)
            if passes in (FULL_PASSES, ROBUST_SPAN_PASSES):
                a, _ = self._pass(a, 0.0)
            if passes == ROBUST_SPAN_PASSES:
                a, _ = self._pass(a, 0.0)
        if passes == FULL_PASSES:
            a, _ = self._pass(a, 0.0)
        return a

    def _orth_replicated(self, z, passes):
        return self._orth_sharded([z], z.shape[0], passes)[0]

    def sketched_svd(self, shards, n: int, l: int, q: int, seed: int, mode: int = OMEGA_REFERENCE):
        """rrsvd_sketched_svd (randomized.cpp:101-107) of the row-stacked shards.
        Returns (U row blocks, sigma (l), this rank's row block [r0, r1) of V (n x l), ||A||_F^2)."""
        ops = self.ops
        if hasattr(ops, "prepare"):
            ops.prepare(shards)
        try:
            return self._sketched_svd(shards, n, l, q, seed, mode)
        finally:
            if hasattr(ops, "release"):
                ops.release()

    def _sketched_svd(self, shards, n, l, q, seed, mode):
        ops = self.ops
        m_local = sum(a.shape[0] for a in shards)
        m_total = int(float(self.comm.allreduce(np.array([m_local], np.float64))[0]))
        if l > min(m_total, n):
            raise api.ContractViolation("randomized_range_finder: l exceeds min(m, n)")
        om = ops.omega(n, l, seed, mode)
        inter = ROBUST_SPAN_PASSES if q > 0 else FULL_PASSES
        qs = self._orth_sharded([ops.gemm(a, False, om) for a in shards], m_total, inter)
        r0, r1 = self.comm.row_block(n)
        for j in range(q):
            # Z = A^H Q (n x l): each rank orthonormalises its row block (row-sharded CholeskyQR),
            # then the rows are gathered for the next local product Y_g = A_g Q~
            z = self._rowsum([ops.gemm(a, True, qg) for a, qg in zip(shards, qs)])
            qt = self.comm.allgather_rows(self._orth_sharded([z[r0:r1]], n, ROBUST_SPAN_PASSES)[0], n)
            qs = self._orth_sharded([ops.gemm(a, False, qt) for a in shards], m_total,
                                    ROBUST_SPAN_PASSES if j + 1 < q else FULL_PASSES)
        bh = self._rowsum([ops.gemm(a, True, qg) for a, qg in zip(shards, qs)])[r0:r1]  # B^H = A^H Q
        qb = self._orth_sharded([bh], n, FULL_PASSES)[0]                      # B^H = Q_b X
        x = self.comm.allreduce(ops.gemm(qb, True, bh))                         # X = Q_b^H B^H (l x l)
        w, sigma, k = ops.svd(_adjoint(x))
        v = ops.gemm(qb, False, k)                                              # V rows = Q_b K
        us = [ops.gemm(qg, False, w) for qg in qs]                              # U = Q U_B, U_B = W
        total_sq = float(self.comm.allreduce(np.array([sum(ops.sumsq(a) for a in shards)], np.float64))[0])
        return us, sigma, v, total_sq

    def fixed_rank(self, shards, n: int, k: int, p: int, q: int, seed: int, mode: int = OMEGA_REFERENCE):
        """rrsvd_fixed_rank (randomized.cpp:109-122): (U row blocks (m_g x k), sigma (k), this
        rank's row block of V (comm.row_block(n) rows x k; all n rows on one rank), w)."""
        if k < 2 or p < 2:
            raise api.ContractViolation("rrsvd_fixed_rank: requires k >= 2 and p >= 2")
        us, sigma, v, total_sq = self.sketched_svd(shards, n, k + p, q, seed, mode)
        s = np.asarray(sigma.cpu() if hasattr(sigma, "cpu") else sigma)[:k]
        w = min(max(1.0 - float(np.sum(s ** 2)) / total_sq, 0.0), 1.0) if total_sq > 0 else 0.0
        return [u[:, :k] for u in us], sigma[:k], v[:, :k], w
