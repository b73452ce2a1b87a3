"""Device-resident MPS and TEBD evolution — mirror of rrsvd::tebd::MpsState / evolve
(mps.hpp:31-41, tebd.hpp:142-144) over the C ABI (rrsvd_b200_mps_* / rrsvd_b200_evolve)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from ._lib import ptr, sz
from .api import DecimationBackend, _ctx
from .models import bond_gate, trotter_plan_3rd


class Sweep(C.Structure):
    _fields_ = [("bond_parity", C.c_int), ("coefficient", C.c_double)]


class EvolveOptions(C.Structure):
    _fields_ = [("abort_discarded_threshold", C.c_double), ("renormalize", C.c_int),
                ("omega_mode", C.c_int)]


class EvolveDiag(C.Structure):
    _fields_ = [("kept_fraction", C.c_double), ("max_bond_dim", C.c_uint64), ("aborted", C.c_int),
                ("abort_step", C.c_uint64), ("n_updates", C.c_uint64)]


class UpdateRecord(C.Structure):
    _fields_ = [("step", C.c_uint64), ("bond", C.c_uint64), ("chi", C.c_uint64),
                ("discarded_weight", C.c_double), ("t_theta_us", C.c_double),
                ("t_gate_us", C.c_double), ("t_svd_us", C.c_double), ("randomized_path", C.c_int)]


@dataclass
class EvolveDiagnostics:
    """rrsvd::tebd::EvolveDiagnostics (tebd.hpp:132-138)."""
    kept_fraction: float
    max_bond_dim: int
    aborted: bool
    abort_step: int
    n_updates: int
    updates: list = field(default_factory=list)


class DeviceMps:
    """MpsState held in HBM.  Starts as the product state |0…0> (mps_product_state)."""

    def __init__(self, site_dims, chi_max: int = 0, trunc_tolerance: float = 0.0, ctx=None):
        self.ctx = _ctx(ctx)
        self.site_dims = [int(d) for d in site_dims]
        dims = (C.c_size_t * len(self.site_dims))(*self.site_dims)
        h = C.c_void_p()
        self.ctx.check(L.lib().rrsvd_b200_mps_create(self.ctx.h, sz(len(self.site_dims)), dims, sz(chi_max),
                                                     C.c_double(trunc_tolerance), C.byref(h)))
        self.h = h
        self.chi_max = chi_max

    def __del__(self):
        # (module globals are gone at interpreter exit; and a context finalised first — the cycle
        # collector runs finalisers in no particular order — has taken the state's memory with it)
        if getattr(self, "h", None) and L is not None and getattr(getattr(self, "ctx", None), "h", None):
            L.lib().rrsvd_b200_mps_destroy(self.h)
        self.h = None

    @property
    def n_sites(self) -> int:
        return len(self.site_dims)

    def set_site(self, site: int, gamma, lam=None):
        g = np.ascontiguousarray(gamma, np.complex128) if isinstance(gamma, np.ndarray) else gamma
        l_ = np.ascontiguousarray(lam, np.float64) if isinstance(lam, np.ndarray) else lam
        dl, _, dr = g.shape
        self.ctx.check(L.lib().rrsvd_b200_mps_set_site(self.h, sz(site), sz(dl), sz(dr), ptr(g), ptr(l_)))

    def load(self, gammas, lambdas):
        self.upload(gammas, lambdas)

    def upload(self, gammas, lambdas=None):
        """The whole state in one call (rrsvd_b200_state_upload: all copies queued, one sync).
        gammas: numpy arrays or (pinned) torch tensors (dim_left, d, dim_right); lambdas: per
        bond (len n-1) or None."""
        n = self.n_sites
        dims = (C.c_size_t * (3 * n))()
        gp = (C.c_void_p * n)()
        lp = (C.c_void_p * n)()
        keep = []
        for s_, g in enumerate(gammas):
            g = np.ascontiguousarray(g, np.complex128) if isinstance(g, np.ndarray) else g
            keep.append(g)
            dl, _, dr = g.shape
            dims[3 * s_], dims[3 * s_ + 1], dims[3 * s_ + 2] = dl, 0, dr
            gp[s_] = ptr(g).value
            if lambdas is not None and s_ < len(lambdas) and lambdas[s_] is not None:
                lam = lambdas[s_]
                lam = np.ascontiguousarray(lam, np.float64) if isinstance(lam, np.ndarray) else lam
                keep.append(lam)
                lp[s_] = ptr(lam).value
        self.ctx.check(L.lib().rrsvd_b200_state_upload(self.h, dims, gp, lp))

    def download(self, gammas, lambdas=None):
        """Fill pre-shaped buffers (rrsvd_b200_state_download: one sync) — gammas[i] must have
        the current dims(i) shape; lambdas[i] (optional) the bond's dimension."""
        n = self.n_sites
        gp = (C.c_void_p * n)(*[ptr(g).value for g in gammas])
        lp = None
        if lambdas is not None:
            lp = (C.c_void_p * n)(*([ptr(x).value if x is not None else None for x in lambdas]
                                    + [None] * (n - len(lambdas))))
        self.ctx.check(L.lib().rrsvd_b200_state_download(self.h, None, gp, lp))

    def roundtrip(self, gammas, lambdas=None):
        """Download into pre-shaped (pinned) host buffers and upload back from them, pipelined per
        site on two streams (rrsvd_b200_state_roundtrip): the state through host memory between
        consecutive steps, the two copy directions overlapped."""
        n = self.n_sites
        gp = (C.c_void_p * n)(*[ptr(g).value for g in gammas])
        lp = None
        if lambdas is not None:
            lp = (C.c_void_p * n)(*([ptr(x).value if x is not None else None for x in lambdas]
                                    + [None] * (n - len(lambdas))))
        self.ctx.check(L.lib().rrsvd_b200_state_roundtrip(self.h, gp, lp))

    def all_dims(self):
        n = self.n_sites
        dims = (C.c_size_t * (3 * n))()
        self.ctx.check(L.lib().rrsvd_b200_state_download(self.h, dims, None, None))
        return [tuple(int(dims[3 * i + j]) for j in range(3)) for i in range(n)]

    def dims(self, site: int):
        d3 = (C.c_size_t * 3)()
        self.ctx.check(L.lib().rrsvd_b200_mps_get_site(self.h, sz(site), d3, None, None))
        return tuple(int(x) for x in d3)

    def gamma(self, site: int) -> np.ndarray:
        out = np.empty(self.dims(site), np.complex128)
        self.ctx.check(L.lib().rrsvd_b200_mps_get_site(self.h, sz(site), None, ptr(out), None))
        return out

    def lam(self, bond: int) -> np.ndarray:
        out = np.empty(self.dims(bond)[2], np.float64)
        self.ctx.check(L.lib().rrsvd_b200_mps_get_site(self.h, sz(bond), None, None, ptr(out)))
        return out

    def bond_dims(self):
        return [self.dims(b)[2] for b in range(self.n_sites - 1)]

    def expectation_local(self, site: int, op) -> complex:
        op = np.ascontiguousarray(op, np.complex128)
        out = np.empty(2)
        self.ctx.check(L.lib().rrsvd_b200_expectation_local(self.h, sz(site), ptr(op), ptr(out)))
        return complex(out[0], out[1])

    def schmidt_entropy(self, bond: int) -> float:
        out = C.c_double()
        self.ctx.check(L.lib().rrsvd_b200_schmidt_entropy(self.h, sz(bond), C.byref(out)))
        return out.value


def build_gates(site_dims, terms: dict, dt: float, plan=None):
    """One gate per (sweep, bond): exp(-i·c·dt·h_b) (tebd.cpp:276-285), shared across sweeps
    with equal coefficients.  Returns (plan, {(sweep, bond): gate})."""
    plan = plan or trotter_plan_3rd(dt)
    cache, gates = {}, {}
    for s, (par, coef) in enumerate(plan):
        for b in range(len(site_dims) - 1):
            if b % 2 != par or b not in terms:
                continue
            key = (b, coef)
            if key not in cache:
                cache[key] = np.ascontiguousarray(bond_gate(terms[b], coef * dt), np.complex128)
            gates[(s, b)] = cache[key]
    return plan, gates


class PreparedGates(dict):
    """{(sweep, bond): rrsvd_b200_gate handle} — gates resident on the device with their block
    structure analysed once (rrsvd_b200_gate_create); reused across evolve calls."""

    def __init__(self, gates: dict, ctx):
        super().__init__()
        self.ctx = ctx
        self._owned = []
        made = {}
        for key, g in gates.items():
            if id(g) not in made:
                arr = np.ascontiguousarray(g, np.complex128) if isinstance(g, np.ndarray) else g
                h = C.c_void_p()
                ctx.check(L.lib().rrsvd_b200_gate_create(ctx.h, ptr(arr), sz(arr.shape[0]), C.byref(h)))
                made[id(g)] = h
                self._owned.append(h)
            self[key] = made[id(g)]

    def n_blocks(self, key) -> int:
        n = C.c_size_t()
        L.lib().rrsvd_b200_gate_blocks(self[key], C.byref(n))
        return int(n.value)

    def __del__(self):
        alive = L is not None and getattr(getattr(self, "ctx", None), "h", None)  # (see DeviceMps.__del__)
        for h in getattr(self, "_owned", []) if alive else []:
            L.lib().rrsvd_b200_gate_destroy(h)
        self._owned = []


def evolve(mps: DeviceMps, terms: dict, dt: float, n_steps: int, backend: DecimationBackend,
           abort_discarded_threshold: float = 1.0, renormalize: bool = True, record_updates: bool = True,
           gates=None, plan=None) -> EvolveDiagnostics:
    """rrsvd::tebd::evolve (tebd.cpp:260-326) on the device; advances backend.seed.
    `gates` may be raw matrices (prepared for this call) or a PreparedGates table."""
    if gates is None:
        plan, gates = build_gates(mps.site_dims, terms, dt, plan)
    nb = mps.n_sites - 1
    sweeps = (Sweep * len(plan))(*[Sweep(p, c) for p, c in plan])
    keep = []
    arr = (C.c_void_p * (len(plan) * nb))()
    prepared = isinstance(gates, PreparedGates) or (len(gates) > 0 and all(
        isinstance(v, C.c_void_p) for v in gates.values()))
    for (s, b), g in gates.items():
        keep.append(g)
        arr[s * nb + b] = g.value if prepared else ptr(g).value
    be = backend.to_c()
    opt = EvolveOptions(abort_discarded_threshold, int(renormalize), backend.omega_mode)
    diag = EvolveDiag()
    nrec = n_steps * sum(len(range(p, nb, 2)) for p, _ in plan) if record_updates else 0
    recs = (UpdateRecord * max(nrec, 1))()
    fn = L.lib().rrsvd_b200_evolve_prepared if prepared else L.lib().rrsvd_b200_evolve
    rc = fn(mps.h, sz(len(plan)), sweeps, arr, sz(n_steps), C.byref(be), C.byref(opt), C.byref(diag),
            recs if record_updates else None, sz(nrec))
    backend.seed = be.seed  # advanced even when a sweep throws (the calls before it took seeds)
    mps.ctx.check(rc)
    ups = [{"step": r.step, "bond": r.bond, "chi": r.chi, "discarded_weight": r.discarded_weight,
            "t_theta_us": r.t_theta_us, "t_gate_us": r.t_gate_us, "t_svd_us": r.t_svd_us,
            "backend": "rrsvd" if r.randomized_path else "det"}
           for r in recs[:min(nrec, diag.n_updates)]] if record_updates else []
    return EvolveDiagnostics(diag.kept_fraction, int(diag.max_bond_dim), bool(diag.aborted),
                             int(diag.abort_step), int(diag.n_updates), ups)
