"""Device-resident evolve (tebd.cpp:260-326) vs the reference evolve on the same model, seed and
backend: observables ⟨σz⟩(t) / ⟨n⟩(t) and bond entropies within 1e-8 (BASELINE north star)."""
import numpy as np
import pytest

import paper_1504_00992_b200 as P
from paper_1504_00992_b200 import models as Mdl
from paper_1504_00992_b200.tebd import DeviceMps, evolve

pytestmark = pytest.mark.gpu


def run_both(ref, site_dims, terms, dt, steps, chi, be_kwargs, tol=0.0, locals_=None):
    n = len(site_dims)
    locals_ = locals_ or [np.eye(d, dtype=complex)[0] for d in site_dims]
    rm = ref.RefMps(site_dims, locals_, chi, tol)
    dm = DeviceMps(site_dims, chi, tol)
    for s, v in enumerate(locals_):
        if not np.allclose(v, np.eye(site_dims[s])[0]):
            dm.set_site(s, np.asarray(v, complex).reshape(1, -1, 1), np.ones(1) if s < n - 1 else None)
    rbe = ref.Backend(**be_kwargs)
    dbe = P.DecimationBackend(**be_kwargs)
    tmap = {b: t for b, t in enumerate(terms)}
    rd = rm.evolve(tmap, dt, steps, rbe)
    dd = evolve(dm, tmap, dt, steps, dbe)
    assert rbe.seed == dbe.seed
    return rm, dm, rd, dd


def observables_match(ref_mps, dev_mps, ops, atol=1e-8):
    n = dev_mps.n_sites
    for s in range(n):
        a = ref_mps.expectation_local(s, ops[s])
        b = dev_mps.expectation_local(s, ops[s])
        assert abs(a - b) < atol, (s, a, b)
    for b in range(n - 1):
        assert abs(ref_mps.schmidt_entropy(b) - dev_mps.schmidt_entropy(b)) < atol, b


def test_ising_quench_deterministic(ref):
    """Ising quench from all-up (test_tebd.cpp:288-308 shape), deterministic decimation."""
    n, dt, steps, chi = 10, 0.02, 25, 16
    terms = Mdl.ising_terms(n, 1.0, 1.0)
    rm, dm, rd, dd = run_both(ref, [2] * n, terms, dt, steps, chi, {})
    assert dd.n_updates == rd["n_updates"]
    assert abs(dd.kept_fraction - rd["kept_fraction"]) < 1e-10
    assert dd.max_bond_dim == rd["max_bond_dim"]
    observables_match(rm, dm, [Mdl.SZ] * n)


def test_ising_randomized_reference_stream(ref):
    """Randomized decimation everywhere (det_crossover 0, k=p=8, q=2) with the reference Ω
    stream regenerated on the device, χ cap active: observables within 1e-8 of the reference.
    (A model without exact Schmidt degeneracies at the cut: with SU(2)-degenerate values, e.g.
    Heisenberg from Néel, ANY two SVD implementations may keep different vectors.)"""
    n, dt, steps, chi = 8, 0.05, 12, 8
    terms = Mdl.ising_terms(n, 1.0, 0.7)
    kw = dict(randomized=True, target_rank=8, oversampling=8, power_iterations=2, det_crossover=0, seed=5)
    rm, dm, rd, dd = run_both(ref, [2] * n, terms, dt, steps, chi, kw)
    assert rd["kept_fraction"] < 1.0  # truncation actually happens
    assert abs(dd.kept_fraction - rd["kept_fraction"]) < 1e-8
    observables_match(rm, dm, [Mdl.SZ] * n)


def test_ising_fixed_precision_bond_growth(ref):
    """Accuracy check on (tebd.cpp:173-179): k=p=4 sketches that fail the probe test grow past
    chi_max; χ profile, kept fraction and observables follow the reference (reference Ω stream,
    probes seeded seed + φ·draw as randomized.cpp:136-140)."""
    n, dt, steps, chi = 8, 0.05, 10, 6
    terms = Mdl.ising_terms(n, 1.0, 0.7)
    kw = dict(randomized=True, target_rank=4, oversampling=4, power_iterations=2, det_crossover=0,
              accuracy_check=True, epsilon=1e-6, probe_count=2, seed=9)
    rm, dm, rd, dd = run_both(ref, [2] * n, terms, dt, steps, chi, kw)
    assert rd["max_bond_dim"] > chi  # the check actually grew bonds past the cap
    assert dd.max_bond_dim == rd["max_bond_dim"]
    assert abs(dd.kept_fraction - rd["kept_fraction"]) < 1e-8
    observables_match(rm, dm, [Mdl.SZ] * n)


def test_tedopa_small_chain(ref):
    """A short spin-boson TEDOPA chain (config-3 model at small d, χ): system ⟨σz⟩ and boson
    occupations ⟨n⟩ within 1e-8; randomized path on the wide bonds."""
    n_chain, d, chi = 5, 4, 12
    t0, om, hop = Mdl.ohmic_chain(n_chain, 2001)
    site_dims, terms = Mdl.build_chain_terms(t0, om, hop, d, 0.5 * Mdl.SZ + 0.5 * Mdl.SX, Mdl.SZ)
    kw = dict(randomized=True, target_rank=chi, oversampling=4, power_iterations=2, det_crossover=8, seed=11)
    rm, dm, rd, dd = run_both(ref, site_dims, terms, 0.05, 10, chi, kw)
    ops = [Mdl.SZ] + [np.diag(np.arange(d)).astype(complex)] * n_chain
    assert any(u["backend"] == "rrsvd" for u in dd.updates)
    observables_match(rm, dm, ops)


def test_abort_threshold_and_records():
    """tebd.cpp:317-321 abort semantics (test_tebd.cpp:329-341) and UpdateRecord timings."""
    n = 6
    terms = {b: t for b, t in enumerate(Mdl.heisenberg_terms(n, 1.0))}
    neel = [np.array([1, 0], complex) if s % 2 == 0 else np.array([0, 1], complex) for s in range(n)]
    dm = DeviceMps([2] * n, 2, 0.0)
    for s, v in enumerate(neel):
        dm.set_site(s, v.reshape(1, 2, 1), np.ones(1) if s < n - 1 else None)
    diag = evolve(dm, terms, 0.1, 50, P.DecimationBackend(), abort_discarded_threshold=1e-8)
    assert diag.aborted and diag.abort_step < 50
    assert diag.updates and all(u["t_svd_us"] > 0 for u in diag.updates)


def test_gate_identity_preserves_state():
    """Zero Hamiltonian leaves the state unchanged (test_tebd.cpp:275-286)."""
    n = 4
    dm = DeviceMps([2] * n, 8)
    diag = evolve(dm, {b: np.zeros((4, 4), complex) for b in range(n - 1)}, 0.1, 3, P.DecimationBackend())
    assert all(u["discarded_weight"] < 1e-15 for u in diag.updates)
    assert abs(dm.expectation_local(0, Mdl.SZ) - 1.0) < 1e-14
