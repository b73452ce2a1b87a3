"""The reference's acceptance criteria on this path (proj/tests/acceptance.cpp), on the device."""
import numpy as np
import pytest
import scipy.linalg as sla

import paper_1504_00992_b200 as P
from paper_1504_00992_b200 import models as M
from paper_1504_00992_b200.tebd import DeviceMps, PreparedGates, build_gates, evolve
from tests.test_gpu_reference_suite import DOWN, UP, dense_coefficients, dense_hamiltonian, kron_all, product_mps

pytestmark = pytest.mark.gpu


def spectrum_exponential(n, ratio):
    """matgen.cpp:37-52 (normalised)."""
    s = ratio ** np.arange(n, dtype=float)
    return s / np.sqrt(np.sum(s * s))


def discarded_weight(s, k):
    return float(np.sum(s[k:] ** 2) / np.sum(s ** 2))


def calibrate_exponential_ratio(n, k, target):
    """matgen.cpp:79-93: bisection on the discarded weight."""
    lo, hi = 1e-6, 1.0 - 1e-12
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if discarded_weight(spectrum_exponential(n, mid), k) < target:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def test_criterion2_fixed_rank_accuracy(ctx, ref):
    """acceptance.cpp:80-106: 1500x750, k = p = 50, q = 4, w = 4e-4 at k: every one of 20 reruns
    within 10x the deterministic SVD's error against the exact spectrum."""
    m, n, k, p, q = 1500, 750, 50, 50, 4
    s_true = spectrum_exponential(n, calibrate_exponential_ratio(n, k, 4e-4))
    a = ref.structured_matrix(s_true, m, 21, 22)
    _, s_det, _ = P.svd_full(a, ctx=ctx)
    det_err = np.max(np.abs(s_det[:k] - s_true[:k]))
    for rerun in range(20):
        rr = P.rrsvd_fixed_rank(a, k, p, q, 300 + rerun, ctx=ctx)
        assert np.max(np.abs(rr.sigma - s_true[:k])) <= 10.0 * det_err


def run_quench(n, dt, steps, sample_every, backend, chi):
    """acceptance.cpp:227-252: all-up Ising (J = g = 1) quench, magnetisation samples."""
    terms = {b: t for b, t in enumerate(M.ising_terms(n, 1.0, 1.0))}
    mps = DeviceMps([2] * n, chi, 1e-24)
    plan, gh = build_gates([2] * n, terms, dt)
    gates = PreparedGates(gh, mps.ctx)
    mags, lams = [], []
    for step in range(steps):
        evolve(mps, terms, dt, 1, backend, record_updates=False, gates=gates, plan=plan)
        if (step + 1) % sample_every == 0:
            mags += [mps.expectation_local(s, M.SZ).real for s in range(n)]
            lams.append([mps.lam(b) for b in range(n - 1)])
    return np.array(mags), lams


def test_criterion6_magnetisation_trace_and_trotter_order():
    """acceptance.cpp:254-318: ⟨σz⟩(t) of the quench within 1e-6 of the exact evolution at 10
    sample times; global error at fixed horizon scales as dt^2 (slopes 2.0 ± 0.2)."""
    n, dt, steps, every = 6, 1e-3, 1000, 100
    mags, _ = run_quench(n, dt, steps, every, P.DecimationBackend(), 32)
    h = dense_hamiltonian(M.ising_terms(n, 1.0, 1.0), n)
    psi0 = kron_all([UP] * n)
    worst, idx = 0.0, 0
    for sample in range(1, steps // every + 1):
        psi = sla.expm(-1j * dt * sample * every * h) @ psi0
        for s in range(n):
            op = np.kron(np.kron(np.eye(2 ** s), M.SZ), np.eye(2 ** (n - s - 1)))
            worst = max(worst, abs(mags[idx] - np.vdot(psi, op @ psi).real))
            idx += 1
    assert worst <= 1e-6
    terms4 = M.heisenberg_terms(4, 1.0)
    start = kron_all([UP, DOWN, UP, DOWN])
    ref = sla.expm(-1j * 0.5 * dense_hamiltonian(terms4, 4)) @ start
    errors = []
    for dt4 in (0.02, 0.01, 0.005):
        mps = product_mps([UP, DOWN, UP, DOWN], 16)
        evolve(mps, {b: t for b, t in enumerate(terms4)}, dt4, int(0.5 / dt4 + 0.5), P.DecimationBackend(),
               record_updates=False)
        errors.append(np.linalg.norm(dense_coefficients(mps) - ref))
    for e0, e1 in zip(errors, errors[1:]):
        assert abs(np.log2(e0 / e1) - 2.0) <= 0.2


@pytest.mark.parametrize("omega_mode", [P.OMEGA_REFERENCE, P.OMEGA_PHILOX])
def test_criterion7_backend_equivalence(omega_mode):
    """acceptance.cpp:320-363: deterministic vs randomized (accuracy check on, ε = 1e-3) quench —
    observables and Schmidt values within 1e-6 at every sample; with the reference's Ω stream and
    with the GPU's own Philox sketch (the criterion is the reference's statistical tolerance for
    any Gaussian sketch)."""
    n, chi = 6, 32
    a_m, a_l = run_quench(n, 1e-3, 1000, 50, P.DecimationBackend(), chi)
    rnd = P.DecimationBackend(randomized=True, target_rank=chi, oversampling=chi, power_iterations=2,
                              accuracy_check=True, epsilon=1e-3, det_crossover=0, seed=99,
                              omega_mode=omega_mode)
    b_m, b_l = run_quench(n, 1e-3, 1000, 50, rnd, chi)
    assert np.max(np.abs(a_m - b_m)) <= 1e-6
    worst = 0.0
    for sa, sb in zip(a_l, b_l):
        for la, lb in zip(sa, sb):
            c = min(len(la), len(lb))
            worst = max(worst, np.max(np.abs(la[:c] - lb[:c]) / la[0]),
                        np.max(la[c:] / la[0], initial=0.0), np.max(lb[c:] / la[0], initial=0.0))
    assert worst <= 1e-6
