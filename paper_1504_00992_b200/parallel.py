"""Chain-block partition of TEBD across ranks: one process per GPU owns a
contiguous block of sites; same-parity bonds update locally and only boundary Γ/λ cross ranks.

Rank r owns sites [a_r, b_r) and the bonds a_r .. b_r-1 (the last one, b_r-1, is the boundary
bond to rank r+1).  Its local chain is the owned sites plus a GHOST copy of site b_r, so the
boundary bond is an ordinary bond of the local chain.  The bonds outside the local chain enter
as edge weights: left edge λ_{a_r-1} (owned by rank r-1), right edge λ_{b_r} (owned by r+1).

Per sweep (bond parity p):
  1. ghost refresh — rank r+1 → r: Γ_{b_r} and λ_{b_r};  rank r-1 → r: λ_{a_r-1};
  2. every rank runs the sweep on its local chain (all its parity-p bonds, batched on the GPU);
     the per-update seeds are the GLOBAL call indices, so results equal the single-GPU order
     (tebd.cpp:162,289-294);
  3. if the boundary bond had parity p, rank r returns the updated ghost Γ_{b_r} to rank r+1.
A site is never modified by two ranks in one sweep (bonds of one parity share no site).

Message volume per boundary and sweep: one Γ (χ·d·χ complex, 3.2 MB at config 3) each way plus
two λ vectors — microseconds on NVLink 5; there is no collective on the data path.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def partition(n_sites: int, world: int, first_block: int | None = None) -> list[tuple[int, int]]:
    """Contiguous blocks [a, b) of sites, near-equal bond counts."""
    if world < 1 or n_sites < 2 * world:
        raise ValueError("partition: need at least two sites per rank")
    if first_block is not None:
        rest = n_sites - first_block
        bounds = [0, first_block] + [first_block + (rest * (r + 1)) // (world - 1) for r in range(world - 1)]
    else:
        bounds = [(n_sites * r) // world for r in range(world + 1)]
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


# ------------------------------------------------------------------------------- comms

class LoopbackHub:
    """In-process mailbox connecting N simulated ranks (tests on one GPU / one CPU)."""

    def __init__(self, world: int):
        self.world = world
        self.box: dict[tuple[int, int], list] = {}

    def comm(self, rank: int) -> "LoopbackComm":
        return LoopbackComm(self, rank)


class LoopbackComm:
    """exchange() semantics over an in-process mailbox.  Simulated ranks run their phases one
    after another, so every rank first posts its sends (post) and then collects (collect)."""

    def __init__(self, hub: LoopbackHub, rank: int):
        self.hub, self.rank, self.world = hub, rank, hub.world

    def post(self, sends):
        for dst, obj in sends:
            self.hub.box.setdefault((self.rank, dst), []).append(obj)

    def collect(self, srcs):
        return [self.hub.box[(src, self.rank)].pop(0) for src in srcs]


class TorchComm:
    """Point-to-point over torch.distributed: NCCL with CUDA tensors on a GPU box, gloo with CPU
    tensors in the CPU tests.  An exchange is two grouped batches (shape headers, then payloads),
    so ranks can post all sends and receives at once without ordering deadlocks."""

    def __init__(self, device: str):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.device = torch, dist, device
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self._pending = []

    def _tensor(self, a):
        t = self.torch
        if isinstance(a, np.ndarray):
            a = t.from_numpy(np.ascontiguousarray(a))
        return a.to(self.device).contiguous()

    def _header(self, obj):
        t = self.torch
        if obj is None:
            return t.tensor([-1, 0, 0, 0, 0], dtype=t.int64, device=self.device), None
        a = self._tensor(obj)
        shape = list(a.shape) + [1] * (3 - a.dim())
        return t.tensor([a.dim(), 1 if a.is_complex() else 0] + shape, dtype=t.int64, device=self.device), a

    def _run(self, ops):
        if ops:
            for w in self.dist.batch_isend_irecv(ops):
                w.wait()

    def post(self, sends):
        self._pending = sends

    def collect(self, srcs):
        t, d = self.torch, self.dist
        sends, self._pending = self._pending, []
        hdrs = [self._header(obj) for _, obj in sends]
        rh = [t.empty(5, dtype=t.int64, device=self.device) for _ in srcs]
        self._run([d.P2POp(d.isend, h, dst) for (dst, _), (h, _) in zip(sends, hdrs)] +
                  [d.P2POp(d.irecv, h, src) for src, h in zip(srcs, rh)])
        out, ops = [], []
        for src, h in zip(srcs, rh):
            v = h.cpu().tolist()
            if v[0] < 0:
                out.append(None)
                continue
            buf = t.empty(v[2:2 + v[0]], dtype=t.complex128 if v[1] else t.float64, device=self.device)
            out.append(buf)
            ops.append(d.P2POp(d.irecv, buf, src))
        ops = [d.P2POp(d.isend, a, dst) for (dst, _), (_, a) in zip(sends, hdrs) if a is not None] + ops
        self._run(ops)
        return out


# ------------------------------------------------------------------------------- blocks

@dataclass
class BlockSpec:
    rank: int
    world: int
    a: int            # first owned global site
    b: int            # one past the last owned site
    n_global: int

    @property
    def has_ghost(self) -> bool:
        return self.rank + 1 < self.world

    @property
    def local_sites(self) -> list[int]:
        return list(range(self.a, self.b + (1 if self.has_ghost else 0)))

    @property
    def local_bonds(self) -> list[int]:  # global bond indices updated by this rank
        return list(range(self.a, self.b if self.has_ghost else self.b - 1))


class DeviceBlock:
    """A rank's local chain on its GPU (DeviceMps + rrsvd_b200_evolve)."""

    def __init__(self, spec: BlockSpec, site_dims, chi_max: int, trunc_tol: float = 0.0, ctx=None,
                 tensors: str = "torch"):
        from .tebd import DeviceMps
        self.spec = spec
        self.site_dims = [site_dims[s] for s in spec.local_sites]
        self.mps = DeviceMps(self.site_dims, chi_max, trunc_tol, ctx=ctx)
        self.edges = [None, None]
        self.tensors = tensors

    # state access (torch CUDA tensors for NCCL, numpy otherwise)
    def get_gamma(self, i: int):
        if self.tensors == "torch":
            import torch
            from ._lib import ptr, sz
            out = torch.empty(self.mps.dims(i), dtype=torch.complex128, device="cuda")
            from . import _lib as L
            self.mps.ctx.check(L.lib().rrsvd_b200_mps_get_site(self.mps.h, sz(i), None, ptr(out), None))
            return out
        return self.mps.gamma(i)

    def get_lambda(self, i: int):
        if self.tensors == "torch":
            import torch
            from . import _lib as L
            from ._lib import ptr, sz
            out = torch.empty(self.mps.dims(i)[2], dtype=torch.float64, device="cuda")
            self.mps.ctx.check(L.lib().rrsvd_b200_mps_get_site(self.mps.h, sz(i), None, None, ptr(out)))
            return out
        return self.mps.lam(i)

    def set_gamma(self, i: int, g, lam=None):
        self.mps.set_site(i, g, lam)

    def set_edges(self, left, right):
        from . import _lib as L
        from ._lib import ptr, sz

        def prep(x):
            if x is None or not isinstance(x, np.ndarray):
                return x
            return np.ascontiguousarray(x, np.float64)
        left, right = prep(left), prep(right)
        self.edges = [left, right]
        nl = 0 if left is None else int(left.shape[0])
        nr = 0 if right is None else int(right.shape[0])
        self.mps.ctx.check(L.lib().rrsvd_b200_mps_set_edge_lambdas(self.mps.h, ptr(left), sz(nl), ptr(right), sz(nr)))

    def sweep(self, parity: int, gates: dict, dt: float, backend, seed: int):
        """One sweep over the local bonds of this parity; gates keyed by GLOBAL bond."""
        from .tebd import evolve
        a = self.spec.a
        local_gates = {(0, gb - a): g for gb, g in gates.items()}
        backend.seed = seed
        return evolve(self.mps, {gb - a: None for gb in gates}, dt, 1, backend, record_updates=False,
                      gates=local_gates, plan=[((parity - a) % 2, 1.0)])  # parity of the LOCAL index


class ChainPartition:
    """Drives the partitioned evolve for one rank."""

    def __init__(self, block, comm, terms_bonds: list[int]):
        self.block, self.comm = block, comm
        self.spec = block.spec
        self.term_bonds = sorted(terms_bonds)  # global bonds that carry a term

    def _global_index(self, plan, step: int, sweep: int, bond: int) -> int:
        per_sweep = [sum(1 for j in self.term_bonds if j % 2 == p) for p, _ in plan]
        idx = step * sum(per_sweep) + sum(per_sweep[:sweep])
        p = plan[sweep][0]
        return idx + sum(1 for j in self.term_bonds if j % 2 == p and j < bond)

    # Each exchange is split in post (sends) and finish (receives + state updates) so that the
    # loopback driver can run all simulated ranks' posts before any rank collects.
    def refresh_post(self):
        """Step 1 sends: my first Γ (+ its right λ) to the left neighbour, my boundary λ
        (local bond nloc-2) to the right neighbour."""
        r, w, blk = self.spec.rank, self.spec.world, self.block
        nloc = len(self.spec.local_sites)
        sends = []
        if r > 0:
            sends += [(r - 1, blk.get_gamma(0)), (r - 1, blk.get_lambda(0) if nloc > 1 else None)]
        if r + 1 < w:
            sends.append((r + 1, blk.get_lambda(nloc - 2)))
        self.comm.post(sends)

    def refresh_finish(self):
        r, w, blk = self.spec.rank, self.spec.world, self.block
        srcs = ([r + 1, r + 1] if r + 1 < w else []) + ([r - 1] if r > 0 else [])
        got = self.comm.collect(srcs)
        left, right = blk.edges
        if r + 1 < w:
            blk.set_gamma(len(self.spec.local_sites) - 1, got[0], None)  # ghost site
            right = got[1]
            got = got[2:]
        if r > 0:
            left = got[0]
        blk.set_edges(left, right)

    def boundary_post(self, parity: int):
        """Step 3 sends: the updated ghost Γ back to its owner."""
        r, w = self.spec.rank, self.spec.world
        b = self.spec.b - 1
        sends = []
        if r + 1 < w and b % 2 == parity and b in self.term_bonds:
            sends.append((r + 1, self.block.get_gamma(len(self.spec.local_sites) - 1)))
        self.comm.post(sends)

    def boundary_finish(self, parity: int):
        r = self.spec.rank
        b = self.spec.a - 1  # the bond between my left neighbour and me
        srcs = [r - 1] if r > 0 and b % 2 == parity and b in self.term_bonds else []
        got = self.comm.collect(srcs)
        if got:
            self.block.set_gamma(0, got[0], None)

    def refresh_ghosts(self):
        self.refresh_post()
        self.refresh_finish()

    def return_boundary(self, parity: int):
        self.boundary_post(parity)
        self.boundary_finish(parity)

    def local_sweep(self, gates_by_sweep: dict, plan, s: int, t: int, dt: float, backend,
                    base_seed: int) -> float:
        """Step 2 for sweep s of step t; returns this rank's kept fraction of the sweep."""
        parity = plan[s][0]
        mine = set(self.spec.local_bonds)
        bonds = [j for j in self.term_bonds if j % 2 == parity and j in mine]
        if not bonds:
            return 1.0
        seed = base_seed + self._global_index(plan, t, s, bonds[0])
        g = {j: gates_by_sweep[(s, j)] for j in bonds}
        return self.block.sweep(parity, g, dt, backend, seed).kept_fraction

    def evolve(self, gates_by_sweep: dict, plan, dt: float, n_steps: int, backend, base_seed: int,
               step0: int = 0) -> float:
        """Real multi-process run (one rank per process).  gates_by_sweep[(sweep, global_bond)]
        → gate.  Returns this rank's kept-fraction product (multiply across ranks)."""
        kept = 1.0
        for t in range(n_steps):
            for s, (parity, _coef) in enumerate(plan):
                self.refresh_ghosts()
                kept *= self.local_sweep(gates_by_sweep, plan, s, step0 + t, dt, backend, base_seed)
                self.return_boundary(parity)
        self.refresh_ghosts()  # edges/ghosts current for observables
        return kept


def evolve_loopback(parts: list, gates_by_sweep: dict, plan, dt: float, n_steps: int, backends: list,
                    base_seed: int, step0: int = 0) -> float:
    """All ranks simulated in one process (LoopbackComm): every communication phase is posted by
    all ranks before any rank collects.  Used to check the partitioned device path on one GPU."""
    kept = 1.0
    for t in range(n_steps):
        for s, (parity, _coef) in enumerate(plan):
            for p in parts:
                p.refresh_post()
            for p in parts:
                p.refresh_finish()
            for p, be in zip(parts, backends):
                kept *= p.local_sweep(gates_by_sweep, plan, s, step0 + t, dt, be, base_seed)
            for p in parts:
                p.boundary_post(parity)
            for p in parts:
                p.boundary_finish(parity)
    for p in parts:  # edges/ghosts current for observables
        p.refresh_post()
    for p in parts:
        p.refresh_finish()
    return kept


# ------------------------------------------------------------------------------- native (C ABI)

class NativeLoopbackHub:
    """rrsvd_b200_loopback_hub: host-staged mailboxes between ranks run as host threads."""

    def __init__(self, nranks: int):
        import ctypes as C
        from . import _lib as L
        self.h = C.c_void_p()
        rc = L.lib().rrsvd_b200_loopback_hub_create(C.c_int(nranks), C.byref(self.h))
        if rc != 0:
            raise RuntimeError("loopback hub")

    def __del__(self):
        from . import _lib as L
        if getattr(self, "h", None) and L is not None:
            L.lib().rrsvd_b200_loopback_hub_destroy(self.h)
            self.h = None


class NativeComm:
    """rrsvd_b200_comm: the partition's transport behind the C ABI — NCCL between GPUs, or the
    host loopback between threads of one process."""

    def __init__(self, ctx, h):
        self.ctx, self.h = ctx, h

    @staticmethod
    def unique_id() -> bytes:
        import ctypes as C
        from . import _lib as L
        buf = (C.c_char * 128)()
        if L.lib().rrsvd_b200_comm_unique_id(buf) != 0:
            raise RuntimeError("ncclGetUniqueId failed (libnccl.so.2 not loadable?)")
        return bytes(buf)

    @classmethod
    def nccl(cls, ctx, nranks: int, rank: int, uid: bytes) -> "NativeComm":
        import ctypes as C
        from . import _lib as L
        h = C.c_void_p()
        buf = (C.c_char * 128).from_buffer_copy(uid)
        ctx.check(L.lib().rrsvd_b200_comm_create_nccl(ctx.h, C.c_int(nranks), C.c_int(rank), buf, C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def loopback(cls, ctx, hub: NativeLoopbackHub, rank: int) -> "NativeComm":
        import ctypes as C
        from . import _lib as L
        h = C.c_void_p()
        ctx.check(L.lib().rrsvd_b200_comm_create_loopback(ctx.h, hub.h, C.c_int(rank), C.byref(h)))
        return cls(ctx, h)

    def __del__(self):
        from . import _lib as L
        if getattr(self, "h", None) and L is not None and getattr(getattr(self, "ctx", None), "h", None):
            L.lib().rrsvd_b200_comm_destroy(self.h)  # (not after its context: see DeviceMps.__del__)
        self.h = None


def evolve_partitioned(block, comm: NativeComm, first_site: int, n_global: int, gates: dict, plan,
                       term_bonds, n_steps: int, backend, step0: int = 0):
    """rrsvd_b200_evolve_partitioned for one rank: `block` is a DeviceMps of the rank's local chain
    (owned sites + ghost), gates {(sweep, local bond): gate handle} (PreparedGates), term_bonds the
    GLOBAL bonds carrying a term.  Returns this rank's EvolveDiagnostics; advances backend.seed to
    where the unpartitioned evolve would leave it."""
    import ctypes as C
    from . import _lib as L
    from .tebd import EvolveDiag, EvolveDiagnostics, EvolveOptions, Sweep
    nb = block.n_sites - 1
    sweeps = (Sweep * len(plan))(*[Sweep(p, c) for p, c in plan])
    arr = (C.c_void_p * (len(plan) * nb))()
    for (s, lb), g in gates.items():
        arr[s * nb + lb] = g.value
    flags = (C.c_ubyte * (n_global - 1))(*[1 if j in set(term_bonds) else 0 for j in range(n_global - 1)])
    be = backend.to_c()
    opt = EvolveOptions(1.0, 1, backend.omega_mode)
    diag = EvolveDiag()
    rc = L.lib().rrsvd_b200_evolve_partitioned(block.h, comm.h, C.c_size_t(first_site), C.c_size_t(n_global),
                                               C.c_size_t(len(plan)), sweeps, arr, flags, C.c_size_t(n_steps),
                                               C.c_uint64(step0), C.byref(be), C.byref(opt), C.byref(diag))
    backend.seed = be.seed
    block.ctx.check(rc)
    return EvolveDiagnostics(diag.kept_fraction, int(diag.max_bond_dim), bool(diag.aborted), int(diag.abort_step),
                             int(diag.n_updates), [])
