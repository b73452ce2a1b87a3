"""Host-side mirror of the reference C++ API for the TEBD decimation path, over the C ABI.

Names, argument meaning and error behaviour follow the reference (`rrsvd::` /
`rrsvd::tebd::`, /root/reference/proj/core/include/rrsvd/*.hpp) so parity tests read like the
reference's own tests.  Every numeric call executes on the B200 through librrsvd_b200.so;
numpy inputs take the end-to-end path (the library stages host memory), torch CUDA tensors
take the device path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from ._lib import OMEGA_PHILOX, OMEGA_REFERENCE, Context, ContractViolation, ptr, sz  # noqa: F401

_default_ctx: Context | None = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def _ctx(ctx):
    return ctx if ctx is not None else default_context()


def _is_torch(x) -> bool:
    return hasattr(x, "data_ptr") and not isinstance(x, np.ndarray)


def _prep(x, dtype=np.complex128):
    if x is None:
        return None
    if _is_torch(x):
        return x.contiguous()
    return np.ascontiguousarray(x, dtype=dtype)


def _empty(like, shape, dtype):
    """Output buffer on the same side (host/device) as `like`."""
    if like is not None and _is_torch(like):
        import torch
        tdt = torch.complex128 if dtype == np.complex128 else torch.float64
        return torch.empty(shape, dtype=tdt, device=like.device)
    return np.empty(shape, dtype)


def _shape(x):
    return tuple(x.shape)


# ------------------------------------------------------------------------ linalg.hpp

def gemm(a, adj_a: bool, b, adj_b: bool = False, ctx=None):
    """rrsvd::gemm (linalg.cpp:20-35): op(a) @ op(b), op ∈ {N, ᴴ}."""
    c = _ctx(ctx)
    a, b = _prep(a), _prep(b)
    ar, ac = _shape(a)
    br, bc = _shape(b)
    m, k = (ac, ar) if adj_a else (ar, ac)
    kb, n = (bc, br) if adj_b else (br, bc)
    if k != kb:
        raise ContractViolation("gemm: inner dimension mismatch")
    out = _empty(a, (m, n), np.complex128)
    c.check(L.lib().rrsvd_b200_zgemm(c.h, int(adj_a), int(adj_b), sz(m), sz(n), sz(k), ptr(a), sz(ac), ptr(b),
                                     sz(bc), ptr(out), sz(n)))
    return out


def ozaki_gemm(a, adj_a: bool, b, moduli: int = 16, ctx=None):
    """op(a) @ b through the INT8 tensor-core emulation of the RRSVD A-products (csrc/ozaki.cuh,
    the Chinese-remainder scheme with `moduli` residue moduli; 16 = FP64-class accuracy)."""
    c = _ctx(ctx)
    a, b = _prep(a), _prep(b)
    ar, ac = _shape(a)
    br, bc = _shape(b)
    m, k = (ac, ar) if adj_a else (ar, ac)
    if k != br:
        raise ContractViolation("ozaki_gemm: inner dimension mismatch")
    out = _empty(a, (m, bc), np.complex128)
    c.check(L.lib().rrsvd_b200_ozaki_zgemm(c.h, int(adj_a), sz(m), sz(bc), sz(k), ptr(a), sz(ac), ptr(b), sz(bc),
                                           ptr(out), sz(bc), int(moduli)))
    return out


class OzakiOperator:
    """A prepared once for many emulated products (rrsvd_b200_ozaki_prepare / _apply / _release):
    the residue planes stay on the device until close()."""

    def __init__(self, a, moduli: int = 15, ctx=None, col0: int = 0, ncols=None):
        """a: the matrix; (col0, ncols): a column block of it (a K-chunk of a wider A's products)."""
        self.ctx = _ctx(ctx)
        self.a = _prep(a)
        rows, cols = _shape(self.a)
        ncols = cols - col0 if ncols is None else ncols
        if col0 < 0 or ncols <= 0 or col0 + ncols > cols:
            raise ContractViolation("OzakiOperator: bad column block")
        self.m, self.n = rows, ncols
        base = ptr(self.a)
        view = C.c_void_p(base.value + 16 * col0)
        self.h = C.c_void_p()
        self.ctx.check(L.lib().rrsvd_b200_ozaki_prepare(self.ctx.h, view, sz(self.m), sz(self.n), sz(cols),
                                                          int(moduli), C.byref(self.h)))

    def mul(self, adj: bool, x, out=None, accumulate: bool = False):
        """op(A) @ x (op = ᴴ when adj); into `out` (device) and added to it with accumulate."""
        x = _prep(x)
        k, l = _shape(x)
        if k != (self.m if adj else self.n):
            raise ContractViolation("OzakiOperator.mul: inner dimension mismatch")
        if out is None:
            out = _empty(x, (self.n if adj else self.m, l), np.complex128)
        self.ctx.check(L.lib().rrsvd_b200_ozaki_apply(self.ctx.h, self.h, int(adj), ptr(x), sz(l), sz(l), ptr(out),
                                                        sz(l), int(accumulate)))
        return out

    def close(self):
        if self.h and getattr(getattr(self, "ctx", None), "h", None):  # (a closed context took the planes)
            L.lib().rrsvd_b200_ozaki_release(self.h)
        self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ozaki_usable(m: int, n: int) -> int:
    """Moduli count the library would use for an m x n A (0: off / outside the emulation)."""
    return int(L.lib().rrsvd_b200_ozaki_usable(sz(m), sz(n)))


def matmul(a, b, ctx=None):
    return gemm(a, False, b, False, ctx)


def qr(a, ctx=None):
    """rrsvd::qr (linalg.cpp:49-65): thin orthonormal Q (m x n) and R = QᴴA."""
    c = _ctx(ctx)
    a = _prep(a)
    m, n = _shape(a)
    q = _empty(a, (m, n), np.complex128)
    r = _empty(a, (n, n), np.complex128)
    c.check(L.lib().rrsvd_b200_qr(c.h, ptr(a), sz(m), sz(n), ptr(q), ptr(r)))
    return q, r


def svd_full(a, ctx=None):
    """rrsvd::svd_full (linalg.cpp:67-88): U (m x r), sigma (r), V (n x r)."""
    c = _ctx(ctx)
    a = _prep(a)
    m, n = _shape(a)
    r = min(m, n)
    u = _empty(a, (m, r), np.complex128)
    s = _empty(a, (r,), np.float64)
    v = _empty(a, (n, r), np.complex128)
    c.check(L.lib().rrsvd_b200_svd(c.h, ptr(a), sz(m), sz(n), ptr(u), ptr(s), ptr(v)))
    return u, s, v


def chol_inv(g, shift_scale: float = 0.0, ctx=None, flags: bool = False):
    """T = R^-1 with G + s I = R^H R, s = shift_scale * 2^-53 * tr(G) (rrsvd_b200_chol_inv_flags):
    one CholeskyQR factor step on an already-formed (e.g. all-reduced) Gram matrix.
    Returns (T, number of dependent columns[, ill]) — ill: a pivot fell below 1e4 x the shift."""
    c = _ctx(ctx)
    g = _prep(g)
    l = _shape(g)[0]
    t = _empty(g, (l, l), np.complex128)
    nd, ill = C.c_int(), C.c_int()
    c.check(L.lib().rrsvd_b200_chol_inv_flags(c.h, ptr(g), sz(l), C.c_double(shift_scale), ptr(t), C.byref(nd),
                                              C.byref(ill)))
    return (t, nd.value, bool(ill.value)) if flags else (t, nd.value)


def frobenius_norm(a, ctx=None) -> float:
    c = _ctx(ctx)
    a = _prep(a)
    out = C.c_double()
    m = a.shape[0]
    n = int(np.prod(a.shape[1:])) if len(a.shape) > 1 else 1
    c.check(L.lib().rrsvd_b200_frobenius_norm(c.h, ptr(a), sz(m), sz(n), C.byref(out)))
    return out.value


# ------------------------------------------------------------------------ randomized.hpp

@dataclass
class SvdResult:
    """rrsvd::SvdResult (linalg.hpp:17-26)."""
    u: object
    sigma: object
    v: object
    discarded_weight: float = 0.0
    achieved_rank: int = 0
    tolerance_certified: bool = True


def gaussian_test_matrix(n: int, l: int, seed: int, mode: int = OMEGA_REFERENCE, ctx=None,
                         device=None):
    """rrsvd::gaussian_test_matrix (randomized.cpp:79-86), generated on the device."""
    c = _ctx(ctx)
    if device is not None:
        import torch
        out = torch.empty((n, l), dtype=torch.complex128, device=device)
    else:
        out = np.empty((n, l), np.complex128)
    c.check(L.lib().rrsvd_b200_gaussian_test_matrix(c.h, sz(n), sz(l), C.c_uint64(seed), C.c_int(mode),
                                                    ptr(out)))
    return out


def rrsvd_sketched_svd(a, l: int, q: int, seed: int, omega=None, mode: int = OMEGA_REFERENCE,
                       ctx=None) -> SvdResult:
    """randomized.cpp:101-107."""
    c = _ctx(ctx)
    a, omega = _prep(a), _prep(omega)
    m, n = _shape(a)
    u = _empty(a, (m, l), np.complex128)
    s = _empty(a, (l,), np.float64)
    v = _empty(a, (n, l), np.complex128)
    w = C.c_double()
    c.check(L.lib().rrsvd_b200_sketched_svd(c.h, ptr(a), sz(m), sz(n), sz(l), sz(q), C.c_uint64(seed),
                                            C.c_int(mode), ptr(omega), ptr(u), ptr(s), ptr(v),
                                            C.byref(w)))
    return SvdResult(u, s, v, w.value, l)


def rrsvd_fixed_rank(a, k: int, p: int, q: int, seed: int, omega=None,
                     mode: int = OMEGA_REFERENCE, vectors: bool = True, ctx=None) -> SvdResult:
    """randomized.cpp:109-122 (RrsvdParams{k, p, q, seed})."""
    c = _ctx(ctx)
    a, omega = _prep(a), _prep(omega)
    m, n = _shape(a)
    u = _empty(a, (m, k), np.complex128) if vectors else None
    s = _empty(a, (k,), np.float64)
    v = _empty(a, (n, k), np.complex128) if vectors else None
    w = C.c_double()
    c.check(L.lib().rrsvd_b200_fixed_rank(c.h, ptr(a), sz(m), sz(n), sz(k), sz(p), sz(q),
                                          C.c_uint64(seed), C.c_int(mode), ptr(omega), ptr(u), ptr(s),
                                          ptr(v), C.byref(w)))
    return SvdResult(u, s, v, w.value, k)


def rrsvd_fixed_precision(a, epsilon: float, probe_count: int, initial_l: int, q: int, seed: int,
                          mode: int = OMEGA_REFERENCE, vectors: bool = True, ctx=None,
                          growth_block: int = 0) -> SvdResult:
    """randomized.cpp:124-176 (AccuracyCheckParams{epsilon, probe_count, growth_block}):
    range finder at initial_l, then probe rounds that certify max_j ||(I-QQ^H) A w_j|| <= eps
    or grow the basis by growth_block columns (0 doubles it).  Returns all l columns; tolerance_certified as the reference."""
    c = _ctx(ctx)
    a = _prep(a)
    m, n = _shape(a)
    mn = min(m, n)
    u = _empty(a, (m * mn,), np.complex128) if vectors else None
    s = _empty(a, (mn,), np.float64)
    v = _empty(a, (n * mn,), np.complex128) if vectors else None
    lo, cert, w = C.c_size_t(), C.c_int(), C.c_double()
    c.check(L.lib().rrsvd_b200_fixed_precision(c.h, ptr(a), sz(m), sz(n), sz(initial_l), sz(q),
                                               sz(probe_count), sz(growth_block), C.c_double(epsilon), C.c_uint64(seed),
                                               C.c_int(mode), ptr(u), ptr(s), ptr(v), C.byref(lo),
                                               C.byref(cert), C.byref(w)))
    l = lo.value
    uu = u[:m * l].reshape(m, l) if vectors else None
    vv = v[:n * l].reshape(n, l) if vectors else None
    return SvdResult(uu, s[:l], vv, w.value, l, bool(cert.value))


def rrsvd_fixed_rank_batch(As, k: int, p: int, q: int, seeds, mode: int = OMEGA_PHILOX,
                           vectors: bool = False, ctx=None):
    """Many same-shaped rrsvd_fixed_rank calls batched through every pipeline stage.
    Returns (list of sigma arrays, discarded weights)."""
    c = _ctx(ctx)
    As = [_prep(a) for a in As]
    cnt = len(As)
    m, n = _shape(As[0])
    S = [_empty(As[0], (k,), np.float64) for _ in range(cnt)]
    U = [_empty(As[0], (m, k), np.complex128) for _ in range(cnt)] if vectors else None
    V = [_empty(As[0], (n, k), np.complex128) for _ in range(cnt)] if vectors else None
    P = C.c_void_p * cnt
    w = (C.c_double * cnt)()
    seeds_arr = (C.c_uint64 * cnt)(*[int(s) for s in seeds])
    c.check(L.lib().rrsvd_b200_fixed_rank_batch(
        c.h, sz(cnt), P(*[ptr(a) for a in As]), sz(m), sz(n), sz(k), sz(p), sz(q), seeds_arr, C.c_int(mode),
        P(*[ptr(u) for u in U]) if U else None, P(*[ptr(s) for s in S]), P(*[ptr(v) for v in V]) if V else None, w))
    return (S, list(w)) if not vectors else (U, S, V, list(w))


# ------------------------------------------------------------------------ tebd.hpp

@dataclass
class DecimationBackend:
    """rrsvd::tebd::DecimationBackend (tebd.hpp:65-85); `seed` advances once per decimate."""
    randomized: bool = False
    target_rank: int = 0
    oversampling: int = 0
    power_iterations: int = 2
    accuracy_check: bool = False
    epsilon: float = 1e-3
    probe_count: int = 10
    det_crossover: int = 256
    seed: int = 0
    omega_mode: int = OMEGA_REFERENCE

    def to_c(self) -> L.Backend:
        return L.Backend(int(self.randomized), self.target_rank, self.oversampling,
                         self.power_iterations, int(self.accuracy_check), self.epsilon,
                         self.probe_count, self.det_crossover, self.seed)


@dataclass
class DecimationResult:
    """rrsvd::tebd::DecimationResult (tebd.hpp:87-96)."""
    gamma_left: object
    lam: object
    gamma_right: object
    discarded: float
    chi: int
    randomized_path: bool
    tolerance_certified: bool
    pseudo_inverse_applied: bool


def build_theta_unfolded(g1, g2, ll, lm, lr, ctx=None):
    """build_theta (tebd.cpp:76-124) in the unfolded layout M[(a,i),(j,b)] (m x n)."""
    c = _ctx(ctx)
    g1, g2 = _prep(g1), _prep(g2)
    cl, d1, cm = _shape(g1)
    _, d2, cr = _shape(g2)
    ll_, lm_, lr_ = (_prep(x, np.float64) for x in (ll, lm, lr))
    out = _empty(g1, (cl * d1, d2 * cr), np.complex128)
    c.check(L.lib().rrsvd_b200_build_theta_unfolded(c.h, ptr(g1), ptr(g2), ptr(ll_), ptr(lm_), ptr(lr_),
                                                    sz(cl), sz(d1), sz(cm), sz(d2), sz(cr), ptr(out)))
    return out


def apply_gate_unfolded(gate, m_in, d1: int, d2: int, ctx=None):
    """apply_gate_to_theta (tebd.cpp:126-139) on the unfolded M."""
    c = _ctx(ctx)
    gate, m_in = _prep(gate), _prep(m_in)
    rows, cols = _shape(m_in)
    cl, cr = rows // d1, cols // d2
    out = _empty(m_in, (rows, cols), np.complex128)
    c.check(L.lib().rrsvd_b200_apply_gate_unfolded(c.h, ptr(gate), sz(d1), sz(d2), sz(cl), sz(cr),
                                                   ptr(m_in), ptr(out)))
    return out


def theta_to_unfolded(theta, ctx=None):
    c = _ctx(ctx)
    theta = _prep(theta)
    d1, d2, cl, cr = _shape(theta)
    out = _empty(theta, (cl * d1, d2 * cr), np.complex128)
    c.check(L.lib().rrsvd_b200_theta_to_unfolded(c.h, ptr(theta), sz(d1), sz(d2), sz(cl), sz(cr), ptr(out)))
    return out


def unfolded_to_theta(m, d1: int, d2: int, ctx=None):
    c = _ctx(ctx)
    m = _prep(m)
    rows, cols = _shape(m)
    cl, cr = rows // d1, cols // d2
    out = _empty(m, (d1, d2, cl, cr), np.complex128)
    c.check(L.lib().rrsvd_b200_unfolded_to_theta(c.h, ptr(m), sz(d1), sz(d2), sz(cl), sz(cr), ptr(out)))
    return out


def build_theta(g1, g2, ll, lm, lr, ctx=None):
    """build_theta returning the reference ThetaTensor layout (i, j, a, b) (tebd.hpp:23-28)."""
    g1t, g2t = _prep(g1), _prep(g2)
    m = build_theta_unfolded(g1t, g2t, ll, lm, lr, ctx)
    return unfolded_to_theta(m, _shape(g1t)[1], _shape(g2t)[1], ctx)


def apply_gate_to_theta(theta, gate, ctx=None):
    theta = _prep(theta)
    d1, d2, _, _ = _shape(theta)
    m = apply_gate_unfolded(gate, theta_to_unfolded(theta, ctx), d1, d2, ctx)
    return unfolded_to_theta(m, d1, d2, ctx)


def decimate_unfolded(m, d1: int, d2: int, ll, lr, chi_max: int, trunc_tol: float,
                      backend: DecimationBackend, renormalize: bool = True, omega=None,
                      ctx=None) -> DecimationResult:
    """decimate (tebd.cpp:141-237) of the unfolded two-site matrix; advances backend.seed."""
    c = _ctx(ctx)
    m = _prep(m)
    rows, cols = _shape(m)
    cl, cr = rows // d1, cols // d2
    minor = min(rows, cols)
    ll_, lr_, omega = _prep(ll, np.float64), _prep(lr, np.float64), _prep(omega)
    # the accuracy check may grow the bond past chi_max (tebd.cpp:177-179)
    kmax = minor if (chi_max == 0 or backend.accuracy_check) else min(minor, chi_max)
    gl = _empty(m, (cl * d1 * kmax,), np.complex128)
    lam = _empty(m, (kmax,), np.float64)
    gr = _empty(m, (kmax * d2 * cr,), np.complex128)
    info = L.DecimInfo()
    be = backend.to_c()
    call_seed = backend.seed
    c.check(L.lib().rrsvd_b200_decimate_unfolded(
        c.h, ptr(m), sz(d1), sz(d2), sz(cl), sz(cr), ptr(ll_), ptr(lr_), sz(chi_max),
        C.c_double(trunc_tol), C.byref(be), C.c_uint64(call_seed), C.c_int(backend.omega_mode),
        ptr(omega), C.c_int(int(renormalize)), ptr(gl), ptr(lam), ptr(gr), C.byref(info)))
    backend.seed += 1  # tebd.cpp:162 — consumed even on the deterministic path, after the Θ checks
    k = int(info.chi)
    return DecimationResult(gl[:cl * d1 * k].reshape(cl, d1, k), lam[:k],
                            gr[:k * d2 * cr].reshape(k, d2, cr), info.discarded, k,
                            bool(info.randomized_path), bool(info.tolerance_certified),
                            bool(info.pseudo_inverse_applied))


def decimate(theta, ll, lr, chi_max: int, trunc_tol: float, backend: DecimationBackend,
             renormalize: bool = True, omega=None, ctx=None) -> DecimationResult:
    """decimate with the reference ThetaTensor (i, j, a, b) input (tebd.hpp:107-110)."""
    theta = _prep(theta)
    d1, d2, _, _ = _shape(theta)
    return decimate_unfolded(theta_to_unfolded(theta, ctx), d1, d2, ll, lr, chi_max, trunc_tol,
                             backend, renormalize, omega, ctx)


def probe_peak(what: int = 0, ctx=None) -> float:
    """Measured device peak in TFLOP/s: 0 = FP64 DMMA (mma.sync f64), 1 = FP64 DFMA."""
    c = _ctx(ctx)
    out = C.c_double()
    c.check(L.lib().rrsvd_b200_probe_peak(c.h, C.c_int(what), C.byref(out)))
    return out.value
