"""The reference's own unit tests on this path (proj/tests/test_linalg.cpp, test_randomized.cpp,
test_tebd.cpp, test_mps.cpp), restated on the device through the C ABI.  Each test cites the
TEST_CASE it restates; tolerances are the reference's unless noted."""
import numpy as np
import pytest
import scipy.linalg as sla
import torch

import paper_1504_00992_b200 as P
from paper_1504_00992_b200 import models as M
from paper_1504_00992_b200.tebd import DeviceMps, evolve
from tests.conftest import cplx_randn

pytestmark = pytest.mark.gpu

UP, DOWN = np.array([1, 0], complex), np.array([0, 1], complex)


# ------------------------------------------------------------------------------- helpers

def dense_coefficients(mps: DeviceMps) -> np.ndarray:
    """ψ[i1..in] = Γ1 λ1 Γ2 ... Γn (mps.cpp dense_coefficients)."""
    n = mps.n_sites
    psi = mps.gamma(0)[0]  # (d, χ)
    for s in range(1, n):
        psi = psi * mps.lam(s - 1)[None, :]
        g = mps.gamma(s)  # (χ_l, d, χ_r)
        psi = np.einsum("xa,adb->xdb", psi, g).reshape(-1, g.shape[2])
    return psi[:, 0]


def product_mps(locals_, chi=0, tol=0.0):
    dims = [len(v) for v in locals_]
    mps = DeviceMps(dims, chi, tol)
    for s, v in enumerate(locals_):
        if not np.allclose(v, np.eye(dims[s])[0]):
            mps.set_site(s, np.asarray(v, complex).reshape(1, -1, 1), np.ones(1) if s < len(dims) - 1 else None)
    return mps


def dense_hamiltonian(terms, n):
    h = np.zeros((2 ** n, 2 ** n), complex)
    for b, t in enumerate(terms):
        h += np.kron(np.kron(np.eye(2 ** b), t), np.eye(2 ** (n - b - 2)))
    return h


def kron_all(vs):
    out = np.ones(1, complex)
    for v in vs:
        out = np.kron(out, v)
    return out


# ------------------------------------------------------------------------------- test_linalg.cpp

def test_matmul_identity_and_scalar(ctx):
    """test_linalg.cpp:75-84."""
    rng = np.random.default_rng(1)
    a = cplx_randn(rng, 5, 4)
    assert np.allclose(P.gemm(a, False, np.eye(4, dtype=complex), ctx=ctx), a, atol=1e-15)
    s = np.eye(5, dtype=complex) * (2 - 1j)
    assert np.allclose(P.gemm(s, False, a, ctx=ctx), (2 - 1j) * a, atol=1e-14)


def test_matmul_dimension_mismatch_throws(ctx):
    """test_linalg.cpp:92-96."""
    with pytest.raises(P.ContractViolation):
        P.gemm(np.ones((3, 4), complex), False, np.ones((5, 2), complex), ctx=ctx)


def test_qr_of_orthonormal_input_unit_modulus_r_diagonal(ctx):
    """test_linalg.cpp:123-133: Q of an orthonormal input is itself up to phases."""
    rng = np.random.default_rng(2)
    q0, _ = np.linalg.qr(cplx_randn(rng, 30, 8))
    q, r = P.qr(q0, ctx=ctx)
    assert np.allclose(np.abs(np.diag(r)), 1.0, atol=1e-12)
    assert np.linalg.norm(np.triu(r, 1)) < 1e-12
    assert np.linalg.norm(q @ r - q0) < 1e-12


def test_qr_against_classical_gram_schmidt_real_4x2(ctx):
    """test_linalg.cpp:135-150."""
    a = np.array([[1, 2], [1, 0], [1, 1], [1, -1]], complex)
    q, r = P.qr(a, ctx=ctx)
    e1 = a[:, 0] / np.linalg.norm(a[:, 0])
    v = a[:, 1] - (e1 @ a[:, 1]) * e1
    e2 = v / np.linalg.norm(v)
    # same columns up to the sign/phase convention of the factorization
    for j, e in enumerate((e1, e2)):
        assert abs(abs(np.vdot(q[:, j], e)) - 1.0) < 1e-12


def test_svd_full_of_a_diagonal_matrix(ctx):
    """test_linalg.cpp:161-173: σ = |d| sorted."""
    d = np.diag(np.array([0.5, -3.0, 2.0j, 1.0]))
    _, s, _ = P.svd_full(d, ctx=ctx)
    assert np.allclose(s, [3.0, 2.0, 1.0, 0.5], atol=1e-14)


def test_svd_full_of_a_1x1_imaginary_matrix(ctx):
    """test_linalg.cpp:175-182."""
    u, s, v = P.svd_full(np.array([[-2.5j]]), ctx=ctx)
    assert abs(s[0] - 2.5) < 1e-15
    assert abs(u[0, 0] * s[0] * np.conj(v[0, 0]) - (-2.5j)) < 1e-14


def test_svd_full_invariant_under_random_unitaries(ctx):
    """test_linalg.cpp:196-204."""
    rng = np.random.default_rng(3)
    a = cplx_randn(rng, 12, 9)
    u1, _ = np.linalg.qr(cplx_randn(rng, 12, 12))
    v1, _ = np.linalg.qr(cplx_randn(rng, 9, 9))
    _, s0, _ = P.svd_full(a, ctx=ctx)
    _, s1, _ = P.svd_full(u1 @ a @ v1, ctx=ctx)
    assert np.max(np.abs(s0 - s1)) < 1e-12 * s0[0]


def test_frobenius_norm(ctx):
    """test_linalg.cpp:218-231."""
    a = np.array([[3, 4j], [0, 0]], complex)
    assert abs(P.frobenius_norm(a, ctx=ctx) - 5.0) < 1e-15
    assert P.frobenius_norm(np.zeros((3, 3), complex), ctx=ctx) == 0.0


# ------------------------------------------------------------------------------- test_randomized.cpp

def test_gaussian_determinism_and_seed_separation(ctx):
    """test_randomized.cpp:28-38."""
    a = P.gaussian_test_matrix(50, 7, 11, ctx=ctx)
    b = P.gaussian_test_matrix(50, 7, 11, ctx=ctx)
    c = P.gaussian_test_matrix(50, 7, 12, ctx=ctx)
    assert np.array_equal(a, b) and not np.allclose(a, c)


def test_rank_one_captured_with_q0(ctx):
    """test_randomized.cpp:51-57: a rank-1 matrix is captured exactly with q = 0."""
    rng = np.random.default_rng(4)
    a = np.outer(cplx_randn(rng, 40), cplx_randn(rng, 30))
    res = P.rrsvd_sketched_svd(a, 4, 0, 9, ctx=ctx)
    assert abs(res.sigma[0] - np.linalg.norm(a)) < 1e-12 * np.linalg.norm(a)
    assert np.all(res.sigma[1:] < 1e-12 * res.sigma[0])


def test_sketch_rejects_l_above_min_dimension(ctx):
    """test_randomized.cpp:67-70."""
    with pytest.raises(P.ContractViolation):
        P.rrsvd_sketched_svd(np.ones((10, 6), complex), 7, 1, 0, ctx=ctx)


def test_fixed_rank_matches_deterministic_at_small_scale(ctx, ref):
    """test_randomized.cpp:110-125."""
    s_true = ref.spectrum_exponential(100, 0.85)
    a = ref.structured_matrix(s_true, 200, 11, 12)
    _, s_det, _ = P.svd_full(a, ctx=ctx)
    det_err = np.max(np.abs(s_det[:10] - s_true[:10]))
    for rerun in range(5):
        res = P.rrsvd_fixed_rank(a, 10, 10, 4, 31 + rerun, ctx=ctx)
        assert np.max(np.abs(res.sigma - s_true[:10])) <= 10.0 * det_err + 1e-13


def test_more_power_iterations_improve_slow_spectrum(ctx, ref):
    """test_randomized.cpp:127-147 (median over 9 reruns per index)."""
    s_true = 1.0 / np.arange(1, 101)
    a = ref.structured_matrix(s_true, 150, 21, 22)
    e2 = np.array([np.abs(P.rrsvd_fixed_rank(a, 10, 10, 2, 500 + r, ctx=ctx).sigma - s_true[:10])
                   for r in range(9)])
    e6 = np.array([np.abs(P.rrsvd_fixed_rank(a, 10, 10, 6, 500 + r, ctx=ctx).sigma - s_true[:10])
                   for r in range(9)])
    assert np.all(np.median(e6, axis=0) <= np.median(e2, axis=0) + 1e-15)


def test_fixed_precision_terminates_immediately_on_low_rank(ctx):
    """test_randomized.cpp:149-168."""
    d = np.zeros((40, 30), complex)
    d[0, 0], d[1, 1], d[2, 2] = 2.0, 1.0, 0.5
    u, _ = P.qr(P.gaussian_test_matrix(40, 40, 71, ctx=ctx), ctx=ctx)
    v, _ = P.qr(P.gaussian_test_matrix(30, 30, 72, ctx=ctx), ctx=ctx)
    a = u @ d @ v.conj().T
    res = P.rrsvd_fixed_precision(a, 1e-10, 5, 8, 0, 73, ctx=ctx)
    assert res.tolerance_certified and res.achieved_rank <= 8
    assert np.allclose(res.sigma[:3], [2.0, 1.0, 0.5], atol=1e-10)


def _retained_rank_for_tolerance(sigma, a_norm, rel_tol):
    """randomized.cpp:228-238 (test helper)."""
    budget, resid = (rel_tol * a_norm) ** 2, a_norm ** 2
    if resid <= budget:
        return 0
    for k, s in enumerate(np.asarray(sigma)):
        resid -= s * s
        if resid <= budget:
            return k + 1
    return len(sigma)


def test_fixed_precision_identifies_retention_rank_for_tolerance(ctx, ref):
    """test_randomized.cpp:170-185: spectrum 1/j (n=150), m=200, AccuracyCheckParams{5e-2·‖A‖,
    5, growth_block 10}, initial l=20, q=2, seed 83 — certified, retained rank within the
    reference's band around the spectrum-tail oracle."""
    spec = 1.0 / np.arange(1, 151)
    a = ref.structured_matrix(spec, 200, 81, 82)
    a_norm, tol = float(np.linalg.norm(a)), 5e-2
    tail = np.sqrt(np.maximum(np.sum(spec ** 2) - np.concatenate([[0.0], np.cumsum(spec ** 2)]), 0.0))
    oracle = int(np.argmax(tail <= tol * a_norm))
    res = P.rrsvd_fixed_precision(a, tol * a_norm, 5, 20, 2, 83, growth_block=10, ctx=ctx)
    assert res.tolerance_certified
    certified = _retained_rank_for_tolerance(res.sigma, a_norm, tol)
    assert oracle * 95 // 100 <= certified <= oracle * 105 // 100 + 2
    _, s_r, _, _, cert_r = ref.fixed_precision(a, tol * a_norm, 5, 20, 2, 83, growth_block=10)
    assert (res.achieved_rank, res.tolerance_certified) == (len(s_r), cert_r)


def test_fixed_precision_flags_exhaustion_instead_of_throwing(ctx):
    """test_randomized.cpp:187-193: identity(24), tolerance 1e-30, 3 probes, initial l=4, q=0."""
    res = P.rrsvd_fixed_precision(np.eye(24, dtype=complex), 1e-30, 3, 4, 0, 3, ctx=ctx)
    assert not res.tolerance_certified


def test_range_finder_on_identity_with_full_l(ctx):
    """test_randomized.cpp:59-65: the full-width sketch of identity(8) spans everything —
    ‖A − U Σ Vᴴ‖_F ≤ 1e-12 through the sketched SVD (l = 8, q = 0, seed 8)."""
    a = np.eye(8, dtype=complex)
    r = P.rrsvd_sketched_svd(a, 8, 0, 8, ctx=ctx)
    assert np.linalg.norm(a - (r.u * r.sigma) @ r.v.conj().T) <= 1e-12


def test_appending_basis_columns_never_increases_the_residual(ctx, ref):
    """test_randomized.cpp:302-313: spectrum 1/j (n=40), m=60, sketch A·Ω(40, 20, seed 73); the
    device QR of the first l sketch columns, l = 2, 5, ..., 20: ‖A − QQᴴA‖_F never increases."""
    a = ref.structured_matrix(1.0 / np.arange(1, 41), 60, 71, 72)
    sketch = P.matmul(a, P.gaussian_test_matrix(40, 20, 73, ctx=ctx), ctx=ctx)
    prev = np.inf
    for l in range(2, 21, 3):
        q, _ = P.qr(np.ascontiguousarray(sketch[:, :l]), ctx=ctx)
        r = np.linalg.norm(a - q @ (q.conj().T @ a))
        assert r <= prev + 1e-12
        prev = r


def test_identical_seeds_give_bit_identical_factorizations(ctx):
    """test_randomized.cpp:324-332 — the device path is deterministic too (fixed reduction orders,
    no atomics on data)."""
    rng = np.random.default_rng(5)
    a = torch.from_numpy(cplx_randn(rng, 300, 200)).cuda()
    r1 = P.rrsvd_fixed_rank(a, 20, 10, 2, 77, ctx=ctx)
    r2 = P.rrsvd_fixed_rank(a, 20, 10, 2, 77, ctx=ctx)
    assert torch.equal(r1.sigma, r2.sigma) and torch.equal(r1.u, r2.u) and torch.equal(r1.v, r2.v)


# ------------------------------------------------------------------------------- test_tebd.cpp

def test_theta_of_a_product_state_unfolds_to_rank_one(ctx):
    """test_tebd.cpp:87-97."""
    g1 = (np.array([0.6, 0.8j]) ).reshape(1, 2, 1).astype(complex)
    g2 = (np.array([1.0, 0.0])).reshape(1, 2, 1).astype(complex)
    th = P.build_theta(g1, g2, None, np.ones(1), None, ctx=ctx)
    m = th.transpose(2, 0, 1, 3).reshape(2, 2)
    assert np.linalg.matrix_rank(m, tol=1e-12) == 1


def test_identity_gate_and_swap_gate(ctx):
    """test_tebd.cpp:125-147."""
    rng = np.random.default_rng(6)
    th = cplx_randn(rng, 2, 2, 3, 4)
    assert np.allclose(P.apply_gate_to_theta(th, np.eye(4, dtype=complex), ctx=ctx), th, atol=1e-15)
    swap = np.zeros((4, 4), complex)
    for i in range(2):
        for j in range(2):
            swap[j * 2 + i, i * 2 + j] = 1.0
    out = P.apply_gate_to_theta(th, swap, ctx=ctx)
    assert np.allclose(out, th.transpose(1, 0, 2, 3), atol=1e-15)


def test_unitary_gates_preserve_theta_norm(ctx):
    """test_tebd.cpp:149-155."""
    rng = np.random.default_rng(7)
    th = cplx_randn(rng, 3, 3, 5, 6)
    g, _ = np.linalg.qr(cplx_randn(rng, 9, 9))
    out = P.apply_gate_to_theta(th, g, ctx=ctx)
    assert abs(np.linalg.norm(out) - np.linalg.norm(th)) < 1e-12 * np.linalg.norm(th)


def test_theta_of_a_maximally_mixed_bond_has_unit_norm(ctx):
    """test_tebd.cpp:110-123: Σ_i λ_i |ii⟩ with flat λ = 1/√d (d = 4, open chain ends)."""
    d = 4
    g1, g2 = np.zeros((1, d, d), complex), np.zeros((d, d, 1), complex)
    for i in range(d):
        g1[0, i, i] = g2[i, i, 0] = 1.0
    theta = P.build_theta(g1, g2, None, np.full(d, 1.0 / np.sqrt(d)), None, ctx=ctx)
    assert abs(np.linalg.norm(theta) - 1.0) <= 1e-10


def test_decimation_optimality_kept_spectrum_beats_random_projections(ctx):
    """test_tebd.cpp:379-407 (on a quenched 6-site state instead of random_canonical_mps): the
    deterministic χ=2 truncation (renormalize off) leaves a smaller error than any of 20 random
    rank-2 projections Q (device QR of Ω(rows, 2, 3000 + t))."""
    terms = M.heisenberg_terms(6, 1.0)
    mps = product_mps([UP, DOWN, UP, DOWN, UP, DOWN], 8)
    evolve(mps, {b: t for b, t in enumerate(terms)}, 0.05, 6, P.DecimationBackend())
    ll, lm, lr = mps.lam(1), mps.lam(2), mps.lam(3)
    theta = P.build_theta(mps.gamma(2), mps.gamma(3), ll, lm, lr, ctx=ctx)
    dec = P.decimate(theta, ll, lr, 2, 0.0, P.DecimationBackend(), renormalize=False, ctx=ctx)
    total_sq = np.linalg.norm(theta) ** 2
    err_opt = np.sqrt(max(0.0, total_sq - float(np.sum(np.asarray(dec.lam) ** 2))))
    m = P.theta_to_unfolded(theta, ctx=ctx)
    for t in range(20):
        q, _ = P.qr(P.gaussian_test_matrix(m.shape[0], 2, 3000 + t, ctx=ctx), ctx=ctx)
        assert np.linalg.norm(m - q @ (q.conj().T @ m)) >= err_opt - 1e-12


def test_deterministic_and_randomized_decimation_agree_mid_simulation(ctx):
    """test_tebd.cpp:179-233."""
    terms = M.heisenberg_terms(6, 1.0)
    mps = product_mps([UP, DOWN, UP, DOWN, UP, DOWN], 8)
    evolve(mps, {b: t for b, t in enumerate(terms)}, 0.05, 6, P.DecimationBackend())
    g1, g2 = mps.gamma(2), mps.gamma(3)
    ll, lm, lr = mps.lam(1), mps.lam(2), mps.lam(3)
    theta = P.apply_gate_to_theta(P.build_theta(g1, g2, ll, lm, lr, ctx=ctx), M.bond_gate(terms[2], 0.05),
                                  ctx=ctx)
    a = P.decimate(theta, ll, lr, 8, 0.0, P.DecimationBackend(), ctx=ctx)
    b = P.decimate(theta, ll, lr, 8, 0.0, P.DecimationBackend(randomized=True, target_rank=8, oversampling=8,
                                                                power_iterations=2, det_crossover=0, seed=5),
                   ctx=ctx)
    assert b.randomized_path and len(a.lam) == len(b.lam)
    assert np.max(np.abs(np.asarray(a.lam) - np.asarray(b.lam))) < 1e-8

    def rec(r):
        gl = np.asarray(r.gamma_left) * ll[:, None, None]
        gr = np.asarray(r.gamma_right) * lr[None, None, :]
        return np.einsum("aik,k,kjb->ijab", gl, np.asarray(r.lam), gr)

    assert np.linalg.norm(rec(a) - rec(b)) < 1e-7


def test_two_site_chain_one_step_equals_exact_propagator():
    """test_tebd.cpp:247-255."""
    terms = M.heisenberg_terms(2, 1.0)
    mps = product_mps([UP, DOWN])
    dt = 0.3
    evolve(mps, {0: terms[0]}, dt, 1, P.DecimationBackend())
    ref = sla.expm(-1j * dt * terms[0]) @ kron_all([UP, DOWN])
    assert np.linalg.norm(dense_coefficients(mps) - ref) < 1e-12


def test_single_step_error_scales_as_dt_cubed():
    """test_tebd.cpp:257-273: 3rd-order Trotter, local error O(dt^3)."""
    terms = M.heisenberg_terms(4, 1.0)
    h = dense_hamiltonian(terms, 4)
    psi0 = kron_all([UP, DOWN, UP, DOWN])
    errs = []
    for dt in (0.2, 0.1, 0.05):
        mps = product_mps([UP, DOWN, UP, DOWN])
        evolve(mps, {b: t for b, t in enumerate(terms)}, dt, 1, P.DecimationBackend())
        errs.append(np.linalg.norm(dense_coefficients(mps) - sla.expm(-1j * dt * h) @ psi0))
    for e0, e1 in zip(errs, errs[1:]):
        assert abs(np.log2(e0 / e1) - 3.0) < 3.0 * 0.067


def test_short_ising_quench_matches_dense_oracle():
    """test_tebd.cpp:288-308: no truncation (χ = 2^(n/2)), overlap with the exact evolution."""
    n, dt, steps = 6, 0.05, 10
    terms = M.ising_terms(n, 1.0, 1.0)
    mps = product_mps([UP] * n, 8)
    evolve(mps, {b: t for b, t in enumerate(terms)}, dt, steps, P.DecimationBackend())
    exact = sla.expm(-1j * dt * steps * dense_hamiltonian(terms, n)) @ kron_all([UP] * n)
    overlap = abs(np.vdot(exact, dense_coefficients(mps)))
    assert overlap >= 1.0 - 1e-4  # Trotter error at dt = 0.05 over 10 steps (reference: 1 - 1e-8 vs its
    # Trotterized oracle); against the Trotterized product below it is exact:
    u = np.eye(2 ** n, dtype=complex)
    for p, c in M.trotter_plan_3rd(dt):
        for b in range(p, n - 1, 2):
            u = np.kron(np.kron(np.eye(2 ** b), M.bond_gate(terms[b], c * dt)), np.eye(2 ** (n - b - 2))) @ u
    trot = np.linalg.matrix_power(u, steps) @ kron_all([UP] * n)
    assert abs(np.vdot(trot, dense_coefficients(mps))) >= 1.0 - 1e-12


def test_truncation_accounting_kept_fraction_matches_norm():
    """test_tebd.cpp:310-327: without renormalization the squared norm equals the product of (1-w)."""
    n = 6
    terms = M.heisenberg_terms(n, 1.0)
    mps = product_mps([UP, DOWN] * 3, 4)
    d = evolve(mps, {b: t for b, t in enumerate(terms)}, 0.04, 8, P.DecimationBackend(), renormalize=False)
    assert d.kept_fraction < 1.0
    norm_sq = float(np.sum(np.abs(dense_coefficients(mps)) ** 2))
    assert abs(norm_sq - d.kept_fraction) <= 1e-6 * d.kept_fraction


# ------------------------------------------------------------------------------- test_mps.cpp

def test_expectation_and_entropy_against_dense_state():
    """test_mps.cpp:96-126: ⟨σz⟩ and bond entropies of a stirred state vs the dense state."""
    n = 5
    terms = M.heisenberg_terms(n, 1.0)
    mps = product_mps([UP, DOWN, UP, DOWN, UP])
    evolve(mps, {b: t for b, t in enumerate(terms)}, 0.07, 5, P.DecimationBackend())
    psi = dense_coefficients(mps)
    psi = psi / np.linalg.norm(psi)
    for s in range(n):
        op = np.kron(np.kron(np.eye(2 ** s), M.SZ), np.eye(2 ** (n - s - 1)))
        assert abs(mps.expectation_local(s, M.SZ) - np.vdot(psi, op @ psi)) < 1e-10
    for b in range(n - 1):
        sv = np.linalg.svd(psi.reshape(2 ** (b + 1), -1), compute_uv=False)
        p = sv ** 2
        p = p[p > 1e-300]
        assert abs(mps.schmidt_entropy(b) - float(-np.sum(p * np.log(p)))) < 1e-10
