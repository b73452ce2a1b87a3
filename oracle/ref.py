"""oracle/ref.py — TEST INFRASTRUCTURE, NOT PRODUCT CODE.

ctypes bindings to ``oracle/_ref/librrsvd_ref.so``: the UNMODIFIED reference C++ core
(``/root/reference/proj/core/src``) compiled by ``oracle/Makefile`` against OpenBLAS 0.3.15.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / reference arm
may import this module; it is the parity checker and the CPU timing arm, never the product.

All complex arrays are numpy complex128, C-contiguous, row-major — the reference's
``DenseMatrix`` / ``Tensor3`` memory (dense_matrix.hpp:26-27, mps.hpp:20-25).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "librrsvd_ref.so")

# OpenBLAS 0.3.15 DYNAMIC_ARCH misdetects AVX-512 Xeons as Prescott;
# pin the core type unless the caller already chose one.  Must precede the dlopen.
os.environ.setdefault("OPENBLAS_CORETYPE", "SkylakeX")

_lib = None


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"reference error {code}: {msg}")
        self.code = code


class ContractViolation(RefError):
    pass


class NumericFailure(RefError):
    pass


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(
                f"{LIB_PATH} missing: run `make -C oracle` (needs /root/reference)")
        _lib = C.CDLL(LIB_PATH)
        _lib.ref_last_error.restype = C.c_char_p
        _lib.ref_blas_core.restype = C.c_char_p
        _lib.ref_blas_config.restype = C.c_char_p
        _lib.ref_mps_product.restype = C.c_void_p
        _lib.ref_mps_free.argtypes = [C.c_void_p]
    return _lib


def _check(rc: int):
    if rc == 0:
        return
    msg = lib().ref_last_error().decode()
    if rc == 1:
        raise ContractViolation(rc, msg)
    if rc == 2:
        raise NumericFailure(rc, msg)
    raise RefError(rc, msg)


def _p(a: np.ndarray | None):
    if a is None:
        return None
    assert a.flags.c_contiguous
    return a.ctypes.data_as(C.c_void_p)


def _c(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.complex128)


def _d(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


U64 = C.c_uint64


def set_threads(n: int):
    lib().ref_set_threads(int(n))


def blas_info() -> dict:
    return {"core": lib().ref_blas_core().decode(), "config": lib().ref_blas_config().decode(),
            "threads": lib().ref_get_threads()}


# ---------------------------------------------------------------- randomized.hpp / linalg.hpp

def gaussian_test_matrix(n: int, l: int, seed: int) -> np.ndarray:
    """randomized.cpp:79-86 — mt19937_64 + Box–Muller, row-major n x l."""
    out = np.empty((n, l), np.complex128)
    _check(lib().ref_gaussian_test_matrix(U64(n), U64(l), U64(seed), _p(out)))
    return out


def gemm(a, adj_a: bool, b, adj_b: bool) -> np.ndarray:
    a, b = _c(a), _c(b)
    m = a.shape[1] if adj_a else a.shape[0]
    n = b.shape[0] if adj_b else b.shape[1]
    out = np.empty((m, n), np.complex128)
    _check(lib().ref_gemm(_p(a), U64(a.shape[0]), U64(a.shape[1]), int(adj_a), _p(b),
                          U64(b.shape[0]), U64(b.shape[1]), int(adj_b), _p(out)))
    return out


def qr(a):
    a = _c(a)
    m, n = a.shape
    q = np.empty((m, n), np.complex128)
    r = np.empty((n, n), np.complex128)
    _check(lib().ref_qr(_p(a), U64(m), U64(n), _p(q), _p(r)))
    return q, r


def frobenius_norm(a) -> float:
    a = _c(a)
    out = C.c_double()
    _check(lib().ref_frobenius_norm(_p(a), U64(a.shape[0]), U64(a.size // max(a.shape[0], 1)),
                                    C.byref(out)))
    return out.value


def svd_full(a):
    a = _c(a)
    m, n = a.shape
    k = min(m, n)
    u = np.empty((m, k), np.complex128)
    s = np.empty(k, np.float64)
    v = np.empty((n, k), np.complex128)
    _check(lib().ref_svd_full(_p(a), U64(m), U64(n), _p(u), _p(s), _p(v)))
    return u, s, v


def singular_values(a):
    a = _c(a)
    s = np.empty(min(a.shape), np.float64)
    _check(lib().ref_singular_values(_p(a), U64(a.shape[0]), U64(a.shape[1]), _p(s)))
    return s


def sketched_svd(a, l: int, q: int, seed: int):
    """rrsvd_sketched_svd (randomized.cpp:101-107): U (m x l), sigma (l), V (n x l), w."""
    a = _c(a)
    m, n = a.shape
    u = np.empty((m, l), np.complex128)
    s = np.empty(l, np.float64)
    v = np.empty((n, l), np.complex128)
    w = C.c_double()
    _check(lib().ref_sketched_svd(_p(a), U64(m), U64(n), U64(l), U64(q), U64(seed), _p(u), _p(s),
                                  _p(v), C.byref(w)))
    return u, s, v, w.value


def fixed_rank(a, k: int, p: int, q: int, seed: int, vectors: bool = True):
    """rrsvd_fixed_rank (randomized.cpp:109-122)."""
    a = _c(a)
    m, n = a.shape
    u = np.empty((m, k), np.complex128) if vectors else None
    s = np.empty(k, np.float64)
    v = np.empty((n, k), np.complex128) if vectors else None
    w = C.c_double()
    _check(lib().ref_fixed_rank(_p(a), U64(m), U64(n), U64(k), U64(p), U64(q), U64(seed), _p(u),
                                _p(s), _p(v), C.byref(w)))
    return u, s, v, w.value


def fixed_precision(a, eps: float, probes: int, initial_l: int, q: int, seed: int, growth_block: int = 0):
    """rrsvd_fixed_precision (randomized.cpp:124-176) -> (u, s, v, w, certified)."""
    a = _c(a)
    m, n = a.shape
    mn = min(m, n)
    u = np.empty(m * mn, np.complex128)
    s = np.empty(mn, np.float64)
    v = np.empty(n * mn, np.complex128)
    lo, cert, w = U64(), C.c_int(), C.c_double()
    _check(lib().ref_fixed_precision(_p(a), U64(m), U64(n), U64(initial_l), U64(q), U64(probes),
                                     U64(growth_block), C.c_double(eps), U64(seed), _p(u), _p(s), _p(v), C.byref(lo),
                                     C.byref(cert), C.byref(w)))
    l = lo.value
    return u[:m * l].reshape(m, l), s[:l], v[:n * l].reshape(n, l), w.value, bool(cert.value)


def range_finder(a, l: int, q: int, seed: int):
    a = _c(a)
    m, n = a.shape
    out = np.empty((m, l), np.complex128)
    _check(lib().ref_range_finder(_p(a), U64(m), U64(n), U64(l), U64(q), U64(seed), _p(out)))
    return out


def spectrum_exponential(n: int, ratio: float) -> np.ndarray:
    out = np.empty(n, np.float64)
    _check(lib().ref_spectrum_exponential(U64(n), C.c_double(ratio), _p(out)))
    return out


def structured_matrix(sigma, m: int, u_seed: int, v_seed: int) -> np.ndarray:
    """matgen.cpp:27-35: U (m x n) diag(sigma) V^H, n = len(sigma)."""
    sigma = _d(sigma)
    out = np.empty((m, sigma.size), np.complex128)
    _check(lib().ref_structured_matrix(_p(sigma), U64(sigma.size), U64(m), U64(u_seed),
                                       U64(v_seed), _p(out)))
    return out


# ---------------------------------------------------------------- tebd.hpp hot trio

def build_theta(g1, g2, ll, lm, lr):
    """tebd.cpp:76-124.  g1 (cl,d1,cm), g2 (cm,d2,cr); ll/lr None = open end.
    Returns theta in the reference (i, j, a, b) layout, shape (d1, d2, cl, cr)."""
    g1, g2 = _c(g1), _c(g2)
    cl, d1, cm = g1.shape
    _, d2, cr = g2.shape
    out = np.empty((d1, d2, cl, cr), np.complex128)
    ll_ = None if ll is None else _d(ll)
    lr_ = None if lr is None else _d(lr)
    lm_ = _d(lm)
    _check(lib().ref_build_theta(_p(g1), _p(g2), _p(ll_), _p(lm_), _p(lr_), U64(cl), U64(d1),
                                 U64(cm), U64(d2), U64(cr), _p(out)))
    return out


def apply_gate(theta, gate):
    """tebd.cpp:126-139.  theta (d1,d2,cl,cr)."""
    theta, gate = _c(theta), _c(gate)
    d1, d2, cl, cr = theta.shape
    out = np.empty_like(theta)
    _check(lib().ref_apply_gate(_p(theta), U64(d1), U64(d2), U64(cl), U64(cr), _p(gate), _p(out)))
    return out


class RefBackend(C.Structure):
    """Mirror of rrsvd::tebd::DecimationBackend (tebd.hpp:65-85)."""
    _fields_ = [("kind", C.c_int), ("target_rank", U64), ("oversampling", U64),
                ("power_iterations", U64), ("accuracy_check", C.c_int), ("epsilon", C.c_double),
                ("probe_count", U64), ("det_crossover", U64), ("seed", U64)]


class RefDecimInfo(C.Structure):
    _fields_ = [("discarded", C.c_double), ("chi", U64), ("randomized_path", C.c_int),
                ("tolerance_certified", C.c_int), ("pseudo_inverse_applied", C.c_int)]


@dataclass
class Backend:
    randomized: bool = False
    target_rank: int = 0
    oversampling: int = 0
    power_iterations: int = 2
    accuracy_check: bool = False
    epsilon: float = 1e-3
    probe_count: int = 10
    det_crossover: int = 256
    seed: int = 0

    def to_c(self) -> RefBackend:
        return RefBackend(int(self.randomized), self.target_rank, self.oversampling,
                          self.power_iterations, int(self.accuracy_check), self.epsilon,
                          self.probe_count, self.det_crossover, self.seed)


@dataclass
class Decimation:
    gamma_left: np.ndarray
    lam: np.ndarray
    gamma_right: np.ndarray
    discarded: float
    chi: int
    randomized_path: bool
    tolerance_certified: bool
    pseudo_inverse_applied: bool


def decimate(theta, ll, lr, chi_max: int, trunc_tol: float, backend: Backend,
             renormalize: bool = True) -> Decimation:
    """tebd.cpp:141-237.  Advances backend.seed by one, like the reference."""
    theta = _c(theta)
    d1, d2, cl, cr = theta.shape
    kmax = min(d1 * cl, d2 * cr)
    if backend.accuracy_check:
        kmax = min(d1 * cl, d2 * cr)
    gl = np.zeros(cl * d1 * kmax, np.complex128)
    lam = np.zeros(kmax, np.float64)
    gr = np.zeros(kmax * d2 * cr, np.complex128)
    be = backend.to_c()
    info = RefDecimInfo()
    ll_ = None if ll is None else _d(ll)
    lr_ = None if lr is None else _d(lr)
    _check(lib().ref_decimate(_p(theta), U64(d1), U64(d2), U64(cl), U64(cr), _p(ll_), _p(lr_),
                              U64(chi_max), C.c_double(trunc_tol), C.byref(be), int(renormalize),
                              _p(gl), _p(lam), _p(gr), C.byref(info)))
    backend.seed = be.seed
    k = int(info.chi)
    return Decimation(gl[:cl * d1 * k].reshape(cl, d1, k).copy(), lam[:k].copy(),
                      gr[:k * d2 * cr].reshape(k, d2, cr).copy(), info.discarded, k,
                      bool(info.randomized_path), bool(info.tolerance_certified),
                      bool(info.pseudo_inverse_applied))


def bond_gate(h, scale: float) -> np.ndarray:
    h = _c(h)
    out = np.empty_like(h)
    _check(lib().ref_bond_gate(_p(h), U64(h.shape[0]), C.c_double(scale), _p(out)))
    return out


def ising_terms(n: int, coupling: float, field: float) -> list[np.ndarray]:
    out = np.empty((n - 1, 4, 4), np.complex128)
    _check(lib().ref_ising_terms(U64(n), C.c_double(coupling), C.c_double(field), _p(out)))
    return list(out)


def heisenberg_terms(n: int, coupling: float) -> list[np.ndarray]:
    out = np.empty((n - 1, 4, 4), np.complex128)
    _check(lib().ref_heisenberg_terms(U64(n), C.c_double(coupling), _p(out)))
    return list(out)


def stieltjes(nodes, h2, n_chain: int):
    nodes, h2 = _d(nodes), _d(h2)
    out = np.empty(2 * n_chain, np.float64)
    _check(lib().ref_stieltjes(_p(nodes), _p(h2), U64(nodes.size), U64(n_chain), _p(out)))
    return out[0], out[1:1 + n_chain].copy(), out[1 + n_chain:].copy()


def chain_terms(t0, omegas, hoppings, boson_dim: int, h_sys, coupling) -> list[np.ndarray]:
    n_chain = len(omegas)
    coeffs = _d(np.concatenate([[t0], omegas, hoppings]))
    h_sys, coupling = _c(h_sys), _c(coupling)
    ds = h_sys.shape[0]
    sizes = [(ds * boson_dim) ** 2] + [boson_dim ** 4] * (n_chain - 1)
    out = np.empty(sum(sizes), np.complex128)
    _check(lib().ref_chain_terms(_p(coeffs), U64(n_chain), U64(boson_dim), _p(h_sys),
                                 _p(coupling), U64(ds), _p(out)))
    terms, off = [], 0
    for s in sizes:
        d = int(round(s ** 0.5))
        terms.append(out[off:off + s].reshape(d, d).copy())
        off += s
    return terms


# ---------------------------------------------------------------- MPS handle

class RefMps:
    """An rrsvd::tebd::MpsState owned by the reference library."""

    def __init__(self, dims, locals_, chi_max: int = 0, tol: float = 0.0):
        dims = np.ascontiguousarray(dims, dtype=np.uint64)
        flat = _c(np.concatenate([np.asarray(v, np.complex128) for v in locals_]))
        self.n = dims.size
        self.h = lib().ref_mps_product(U64(self.n), _p(dims), _p(flat), U64(chi_max),
                                       C.c_double(tol))
        if not self.h:
            raise ContractViolation(1, lib().ref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_mps_free(C.c_void_p(self.h))
            self.h = None

    def shapes(self):
        out = np.empty(3 * self.n, np.uint64)
        _check(lib().ref_mps_shape(C.c_void_p(self.h), _p(out)))
        return [tuple(int(x) for x in out[3 * s:3 * s + 3]) for s in range(self.n)]

    def gamma(self, site: int) -> np.ndarray:
        l, d, r = self.shapes()[site]
        g = np.empty((l, d, r), np.complex128)
        _check(lib().ref_mps_get(C.c_void_p(self.h), U64(site), _p(g), None))
        return g

    def lam(self, bond: int) -> np.ndarray:
        r = self.shapes()[bond][2]
        g = np.empty(self.shapes()[bond], np.complex128)
        out = np.empty(r, np.float64)
        _check(lib().ref_mps_get(C.c_void_p(self.h), U64(bond), _p(g), _p(out)))
        return out

    def set_site(self, site: int, gamma, lam=None):
        gamma = _c(gamma)
        l, d, r = gamma.shape
        lam_ = None if lam is None else _d(lam)
        _check(lib().ref_mps_set(C.c_void_p(self.h), U64(site), U64(l), U64(d), U64(r), _p(gamma),
                                 _p(lam_)))

    def evolve(self, terms: dict, dt: float, n_steps: int, backend: Backend,
               abort_threshold: float = 1.0, renormalize: bool = True) -> dict:
        bonds = np.array(sorted(terms), np.uint64)
        mats = _c(np.concatenate([_c(terms[int(b)]).ravel() for b in bonds]))
        be = backend.to_c()
        diag = np.zeros(6, np.float64)
        _check(lib().ref_evolve(C.c_void_p(self.h), _p(bonds), _p(mats), U64(bonds.size),
                                C.c_double(dt), U64(n_steps), C.byref(be),
                                C.c_double(abort_threshold), int(renormalize), _p(diag)))
        backend.seed = be.seed
        return {"kept_fraction": diag[0], "max_bond_dim": int(diag[1]), "aborted": bool(diag[2]),
                "abort_step": int(diag[3]), "n_updates": int(diag[4]), "update_us": float(diag[5])}

    def expectation_local(self, site: int, op) -> complex:
        op = _c(op)
        out = np.empty(2, np.float64)
        _check(lib().ref_expectation_local(C.c_void_p(self.h), U64(site), _p(op), _p(out)))
        return complex(out[0], out[1])

    def schmidt_entropy(self, bond: int) -> float:
        out = C.c_double()
        _check(lib().ref_schmidt_entropy(C.c_void_p(self.h), U64(bond), C.byref(out)))
        return out.value

    def dense(self) -> np.ndarray:
        total = int(np.prod([s[1] for s in self.shapes()]))
        out = np.empty(total, np.complex128)
        _check(lib().ref_dense_coefficients(C.c_void_p(self.h), _p(out)))
        return out


# ---- file formats and the experiment drivers -----------------------

def _s(text: str) -> bytes:
    return text.encode()


def write_rrsm(path: str, a):
    a = _c(a)
    _check(lib().ref_write_rrsm(_s(path), _p(a), U64(a.shape[0]), U64(a.shape[1])))


def read_rrsm(path: str) -> np.ndarray:
    r, c = U64(), U64()
    _check(lib().ref_read_rrsm_dims(_s(path), C.byref(r), C.byref(c)))
    out = np.empty((r.value, c.value), np.complex128)
    _check(lib().ref_read_rrsm(_s(path), _p(out)))
    return out


def write_value_lines(path: str, values):
    v = _d(values)
    _check(lib().ref_write_value_lines(_s(path), _p(v), U64(v.size)))


def write_coefficients(path: str, t0: float, omegas, hoppings):
    om, hop = _d(omegas), _d(hoppings if len(hoppings) else [0.0])
    _check(lib().ref_write_coefficients(_s(path), C.c_double(t0), _p(om), U64(om.size), _p(hop)))


def run_tebd(out: str, model: str = "ising", coeffs: str = "", sites: int = 6, chi: int = 32, dt: float = 1e-3,
             steps: int = 100, backend: str = "det", epsilon: float = 0.0, q: int = 2, oversampling: int = 0,
             crossover: int = 256, coupling: float = 1.0, field: float = 1.0, trunc_tolerance: float = 0.0,
             abort_threshold: float = 1.0, boson_dim: int = 4, sys_epsilon: float = 1.0, sys_delta: float = 1.0,
             seed: int = 1, observables_out: str = "", state_out: str = "") -> int:
    """experiments.cpp run_tebd (the reference's `tebd-run`); returns its exit code."""
    D = C.c_double
    return int(lib().ref_run_tebd(_s(model), _s(coeffs), U64(sites), U64(chi), D(dt), U64(steps), _s(backend),
                                  D(epsilon), U64(q), U64(oversampling), U64(crossover), D(coupling), D(field),
                                  D(trunc_tolerance), D(abort_threshold), U64(boson_dim), D(sys_epsilon),
                                  D(sys_delta), U64(seed), _s(out), _s(observables_out), _s(state_out)))
