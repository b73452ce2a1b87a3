"""Host-side model builders (inputs of the device path) pinned against the reference library."""
import numpy as np
import pytest

from paper_1504_00992_b200 import models as M


def test_ising_heisenberg_terms(ref):
    for n in (2, 3, 7):
        for a, b in zip(M.ising_terms(n, 1.3, 0.7), ref.ising_terms(n, 1.3, 0.7)):
            assert np.array_equal(a, b)
        for a, b in zip(M.heisenberg_terms(n, 0.9), ref.heisenberg_terms(n, 0.9)):
            assert np.array_equal(a, b)


def test_bond_gate(ref):
    rng = np.random.default_rng(0)
    for dd in (4, 16, 36):
        h = rng.standard_normal((dd, dd)) + 1j * rng.standard_normal((dd, dd))
        h = h + h.conj().T
        assert np.max(np.abs(M.bond_gate(h, 0.37) - ref.bond_gate(h, 0.37))) < 1e-12


def test_stieltjes_and_chain_terms(ref):
    x = np.linspace(0.0, 1.0, 2001)
    t0, om, hop = M.ohmic_chain(12, 2001)
    rt0, rom, rhop = ref.stieltjes(x, x.copy(), 12)
    assert abs(t0 - rt0) < 1e-14 and np.max(np.abs(om - rom)) < 1e-12 and np.max(np.abs(hop - rhop)) < 1e-12
    h_sys = 0.5 * M.SZ + 0.5 * M.SX
    dims, terms = M.build_chain_terms(t0, om, hop, 5, h_sys, M.SZ)
    rterms = ref.chain_terms(rt0, rom, rhop, 5, h_sys, M.SZ)
    assert dims == [2] + [5] * 12
    for a, b in zip(terms, rterms):
        assert np.max(np.abs(a - b)) < 1e-12


def test_saturated_dims():
    assert M.saturated_bond_dims([2] + [20] * 100, 100)[:3] == [2, 40, 100]
    assert M.saturated_bond_dims([2] + [20] * 100, 100)[-2:] == [100, 20]
    assert M.saturated_bond_dims([2] * 64, 128)[:8] == [2, 4, 8, 16, 32, 64, 128, 128]


def test_trotter_plan():
    plan = M.trotter_plan_3rd(0.01)
    assert plan == [(1, 0.5), (0, 1.0), (1, 0.5)]
    with pytest.raises(ValueError):
        M.trotter_plan_3rd(0.0)


def test_liouvillian_mpdo_terms(ref):
    """The MPDO mapping (models.liouville_term): exp(-i dt L) vec(rho) = vec(U rho U^H) in the
    (ket, bra) site ordering, L Hermitian, and the reference's own bond_gate (zheevd,
    tebd.cpp:239-258) of L equals U (x) U* arranged on the doubled sites."""
    from scipy.linalg import expm
    rng = np.random.default_rng(5)
    d1, d2 = 2, 3
    a = rng.standard_normal((6, 6)) + 1j * rng.standard_normal((6, 6))
    h = a + a.conj().T
    L = M.liouville_term(h, d1, d2)
    assert np.max(np.abs(L - L.conj().T)) == 0.0
    psi = rng.standard_normal(6) + 1j * rng.standard_normal(6)
    psi /= np.linalg.norm(psi)
    u = expm(-0.3j * h)
    rho_t = u @ np.outer(psi, psi.conj()) @ u.conj().T

    def vec(r):  # rho[(k1 k2), (b1 b2)] -> (k1 b1 k2 b2)
        return r.reshape(d1, d2, d1, d2).transpose(0, 2, 1, 3).reshape(-1)
    assert np.max(np.abs(expm(-0.3j * L) @ vec(np.outer(psi, psi.conj())) - vec(rho_t))) < 1e-13
    g_ref = ref.bond_gate(L, 0.3)
    assert np.max(np.abs(g_ref - expm(-0.3j * L))) < 1e-12
    # the local product state of the MPDO
    assert np.allclose(M.mpdo_local(np.array([0.6, 0.8j])), np.kron([0.6, 0.8j], np.conj([0.6, 0.8j])))
