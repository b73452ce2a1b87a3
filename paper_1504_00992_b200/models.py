"""Host-side model builders for the benchmarks and parity runs (off the hot path).

Restatements of the reference's CPU-cheap preprocessing, which the survey marks out of scope
for the device: bond Hamiltonians (tebd.cpp:375-404), the TEDOPA chain
map (chainmap.cpp:58-68,108-153,197-252), the 3rd-order Trotter plan (tebd.cpp:67-74) and
bond gates exp(-i·s·h) (tebd.cpp:239-258).  They produce INPUTS for the device path; the
CPU tests pin them against the reference library.
"""
from __future__ import annotations

import numpy as np

from ._lib import ContractViolation

SX = np.array([[0, 1], [1, 0]], np.complex128)
SY = np.array([[0, -1j], [1j, 0]], np.complex128)
SZ = np.array([[1, 0], [0, -1]], np.complex128)


def trotter_plan_3rd(dt: float):
    """tebd.cpp:67-74: sweeps (bond parity, coefficient) = (1, ½), (0, 1), (1, ½)."""
    if dt == 0.0:
        raise ValueError("trotter_plan_3rd: dt must be nonzero")
    return [(1, 0.5), (0, 1.0), (1, 0.5)]


def ising_terms(n: int, coupling: float, field: float) -> list[np.ndarray]:
    """tebd.cpp:375-388: H = -J Σ σzσz - g Σ σx, fields split between neighbouring bonds."""
    if n < 2:
        raise ValueError("ising_terms: need at least two sites")
    i2 = np.eye(2)
    terms = []
    for b in range(n - 1):
        h = -coupling * np.kron(SZ, SZ)
        h = h - field * (1.0 if b == 0 else 0.5) * np.kron(SX, i2)
        h = h - field * (1.0 if b + 2 == n else 0.5) * np.kron(i2, SX)
        terms.append(h.astype(np.complex128))
    return terms


def heisenberg_terms(n: int, coupling: float) -> list[np.ndarray]:
    """tebd.cpp:390-404."""
    h = coupling * (np.kron(SX, SX) + np.kron(SY, SY) + np.kron(SZ, SZ))
    return [h.astype(np.complex128) for _ in range(n - 1)]


def sparsity_blocks(h: np.ndarray) -> list[np.ndarray]:
    """Index sets of the connected components of the exact nonzero pattern of a square matrix
    (a symmetric pattern: h is Hermitian).  h is block-diagonal up to this permutation."""
    n = h.shape[0]
    parent = list(range(n))

    def find(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x
    rows, cols = np.nonzero(h)
    for r, c in zip(rows, cols):
        a, b = find(int(r)), find(int(c))
        if a != b:
            parent[a] = b
    groups: dict[int, list[int]] = {}
    for i in range(n):
        groups.setdefault(find(i), []).append(i)
    return [np.array(g) for g in sorted(groups.values(), key=lambda g: g[0])]


def bond_gate(h: np.ndarray, scale: float) -> np.ndarray:
    """exp(-i·scale·h) of a Hermitian term via its eigendecomposition (tebd.cpp:239-258).

    The exponential is taken block by block over the connected components of h's exact
    sparsity pattern — the same matrix function, but exact zeros stay exact (eigendecomposing
    the full matrix leaks ~1e-17 noise across blocks when eigenvalues of different blocks are
    degenerate).  TEDOPA boson-boson terms conserve the total excitation number, so their gates
    are block-diagonal; the device applies such gates block-sparsely."""
    h = np.asarray(h, np.complex128)
    if h.ndim != 2 or h.shape[0] != h.shape[1]:
        raise ContractViolation("bond_gate: term must be square")
    # tebd.cpp:241-246: the same Hermiticity test as the reference, before any factorisation
    if h.size and np.max(np.abs(h - h.conj().T)) > 1e-9 * max(1.0, float(np.max(np.abs(h)))):
        raise ContractViolation("bond_gate: term is not Hermitian")
    out = np.zeros(h.shape, np.complex128)
    for idx in sparsity_blocks(h):
        hb = h[np.ix_(idx, idx)]
        w, v = np.linalg.eigh(hb)
        out[np.ix_(idx, idx)] = (v * np.exp(-1j * scale * w)) @ v.conj().T
    return out


def trapezoid_measure(nodes: np.ndarray, h2: np.ndarray):
    """chainmap.cpp:58-68."""
    n = nodes.size
    w = np.empty(n)
    w[0] = 0.5 * (nodes[1] - nodes[0])
    w[-1] = 0.5 * (nodes[-1] - nodes[-2])
    w[1:-1] = 0.5 * (nodes[2:] - nodes[:-2])
    return nodes, w * h2


def stieltjes_coefficients(nodes: np.ndarray, weights: np.ndarray, n_chain: int):
    """Discretised Stieltjes with full reorthogonalisation (chainmap.cpp:108-153).
    Returns (t0, omegas[n_chain], hoppings[n_chain-1])."""
    x, w = nodes, weights
    beta0 = float(np.sum(w))
    polys = [np.full(x.size, 1.0 / np.sqrt(beta0))]
    alpha = np.zeros(n_chain)
    beta = np.zeros(n_chain)
    for j in range(n_chain):
        pj = polys[j]
        u = x * pj
        alpha[j] = np.dot(w * u, pj)
        if j + 1 == n_chain:
            break
        u = u - alpha[j] * pj
        if j > 0:
            u = u - np.sqrt(beta[j - 1]) * polys[j - 1]
        for _ in range(2):
            for pk in polys:
                u = u - np.dot(w * u, pk) * pk
        b = np.dot(w * u, u)
        if not (b > 0.0 and np.isfinite(b)):
            raise ArithmeticError(f"recurrence breakdown at coefficient {j + 1}")
        beta[j] = b
        polys.append(u / np.sqrt(b))
    return np.sqrt(beta0), alpha, np.sqrt(beta[:n_chain - 1])


def ohmic_chain(n_chain: int = 100, n_nodes: int = 20001):
    """The config-3 bath: h²(x) = x on [0, 1] with 20001 trapezoid nodes."""
    x = np.linspace(0.0, 1.0, n_nodes)
    nodes, w = trapezoid_measure(x, x.copy())
    return stieltjes_coefficients(nodes, w, n_chain)


def build_chain_terms(t0, omegas, hoppings, boson_dim: int, h_sys: np.ndarray,
                      coupling: np.ndarray) -> tuple[list[int], list[np.ndarray]]:
    """chainmap.cpp:197-252: system ⊗ boson bond plus boson-boson bonds; on-site ω split evenly
    between the two bonds of a site (full share on the last bond).  Returns (site_dims, terms)."""
    n_chain = len(omegas)
    d_sys = h_sys.shape[0]
    b = np.diag(np.sqrt(np.arange(1, boson_dim, dtype=float)), 1).astype(np.complex128)
    bd = b.conj().T
    num = np.diag(np.arange(boson_dim, dtype=float)).astype(np.complex128)
    ib = np.eye(boson_dim, dtype=np.complex128)
    isys = np.eye(d_sys, dtype=np.complex128)

    def left_share(n):
        return 1.0 if n + 1 == n_chain else 0.5

    terms = []
    h = np.kron(h_sys, ib) + t0 * np.kron(coupling, b + bd) + left_share(0) * omegas[0] * np.kron(isys, num)
    terms.append(h)
    for n in range(1, n_chain):
        h = hoppings[n - 1] * np.kron(bd, b) + hoppings[n - 1] * np.kron(b, bd)
        h = h + (1.0 - left_share(n - 1)) * omegas[n - 1] * np.kron(num, ib)
        h = h + left_share(n) * omegas[n] * np.kron(ib, num)
        terms.append(h)
    return [d_sys] + [boson_dim] * n_chain, terms


def tedopa_system(n_chain: int = 100, boson_dim: int = 20, eps: float = 1.0, delta: float = 1.0):
    """Spin-boson TEDOPA chain of config 3: h_sys = ½ε σz + ½Δ σx, A = σz (experiments.cpp
    tedopa-chain branch), ohmic bath mapped to n_chain oscillators of dimension boson_dim."""
    t0, om, hop = ohmic_chain(n_chain)
    h_sys = 0.5 * eps * SZ + 0.5 * delta * SX
    return build_chain_terms(t0, om, hop, boson_dim, h_sys, SZ)


def saturated_bond_dims(site_dims, chi: int) -> list[int]:
    """χ_b = min(χ, Π_{s≤b} d_s, Π_{s>b} d_s): the largest canonical bond dimensions."""
    n = len(site_dims)
    out = []
    for b in range(n - 1):
        left = 1
        for s in range(b + 1):
            left = min(left * site_dims[s], chi)
        right = 1
        for s in range(b + 1, n):
            right = min(right * site_dims[s], chi)
        out.append(min(chi, left, right))
    return out


def synthetic_saturated_mps(site_dims, chi: int, seed: int = 0, decay: float = 0.9):
    """The timing state of SURVEY §8(d) C2/C3: χ-saturated bonds, Gaussian Γ/√(χ_l d), λ ∝ decay^i
    normalised.  Returns (gammas, lambdas) as numpy arrays."""
    rng = np.random.default_rng(seed)
    bonds = saturated_bond_dims(site_dims, chi)
    n = len(site_dims)
    gammas, lambdas = [], []
    for s in range(n):
        cl = 1 if s == 0 else bonds[s - 1]
        cr = 1 if s == n - 1 else bonds[s]
        g = (rng.standard_normal((cl, site_dims[s], cr)) + 1j * rng.standard_normal((cl, site_dims[s], cr)))
        gammas.append(g / np.sqrt(cl * site_dims[s]))
    for b in range(n - 1):
        v = decay ** np.arange(bonds[b])
        lambdas.append(v / np.linalg.norm(v))
    return gammas, lambdas


# ---- mixed states: the MPDO in Liouville space (config 4's shape) -----------------------------
# The reference evolves pure states only (mps.hpp:121-134).  A density operator is evolved as
# the "MPS" of vec(rho) with site dimension d^2 (site index k*d + b: ket k, bra b) under the
# Liouvillian terms L_b = H_b (x) 1 - 1 (x) H_b^T on (kets, bras): exp(-i dt L_b) = U (x) U* with
# U = exp(-i dt H_b) — the two-site gate "applied as U (x) U* factors".  Both the reference's own
# evolve (tebd.cpp:260-326, bond_gate = exp(-i dt L_b) via zheevd) and the device run it
# unchanged; the gates of number-conserving terms stay block-sparse (kets x bras sectors).

def liouville_term(h: np.ndarray, d1: int, d2: int) -> np.ndarray:
    """L = H (x) 1 - 1 (x) H^T for a two-site H on (k1, k2), in the MPDO ordering
    ((k1 d1 + b1) d2^2 + (k2 d2 + b2)) of the doubled sites."""
    h = np.asarray(h, np.complex128).reshape(d1, d2, d1, d2)  # H[k1, k2, k1', k2']
    e1, e2 = np.eye(d1), np.eye(d2)
    # L[k1 b1 k2 b2, k1' b1' k2' b2'] = H[k1 k2, k1' k2'] d(b1 b1') d(b2 b2')
    #                                  - d(k1 k1') d(k2 k2') H[b1' b2', b1 b2]
    L = np.einsum("acxz,by,dw->abcdxyzw", h, e1, e2)
    L -= np.einsum("ax,cz,ywbd->abcdxyzw", e1, e2, h)
    n = d1 * d1 * d2 * d2
    return L.reshape(n, n)


def mpdo_terms(site_dims, terms):
    """(doubled site dims, Liouvillian bond terms) of a pure-state chain's Hamiltonian terms."""
    dims2 = [d * d for d in site_dims]
    out = [liouville_term(h, site_dims[b], site_dims[b + 1]) for b, h in enumerate(terms)]
    return dims2, out


def mpdo_local(psi: np.ndarray) -> np.ndarray:
    """vec(|psi><psi|) in the (k d + b) site ordering: psi (x) conj(psi)."""
    psi = np.asarray(psi, np.complex128)
    return np.kron(psi, psi.conj())

