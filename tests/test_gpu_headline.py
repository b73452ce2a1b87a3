"""Parity at the benchmarked shapes themselves (BASELINE configs[1] and [2]).

* the headline decimation: C3 2000 x 2000 unfolding, RRSVD k = 100, p = 10, q = 2, the reference
  Omega stream regenerated on the device (tebd.cpp:141-237, randomized.cpp:17-45);
* evolve traces at C2 scale — Ising L = 64, chi = 128, 20 steps from the product state, as
  run_tebd / acceptance.cpp:227-252 start — deterministic (the reference default) and with the
  RRSVD forced (det_crossover = 0);
* a d = 20, chi = 100 TEDOPA chain (spin + 10 oscillators, the config-3 model) for 2 steps with
  the headline backend (RRSVD p = 10, q = 2, default crossover): the wide bonds reach the C3
  unfolding (2000 x 2000) inside the run;
* the statistical tolerance of the GPU's own RNG (Philox) stated on a TEBD-evolved C3 Theta:
  20 reference seeds vs 8 device seeds.
Bars (north star): lambda / sigma within 1e-10, discarded weight within 1e-10, observables
<sigma_z>, <n> and bond entropies within 1e-8.
"""
import numpy as np
import pytest

import paper_1504_00992_b200 as P
from paper_1504_00992_b200 import models as Mdl
from paper_1504_00992_b200.tebd import DeviceMps, evolve
from tests.conftest import cplx_randn
from tests.test_gpu_parity import random_fragment, theta_from

pytestmark = pytest.mark.gpu

NUM20 = np.diag(np.arange(20)).astype(complex)


def test_decimate_headline_c3_p10(ctx, ref):
    """The benchmarked decimation: 2000 x 2000 (chi_l = chi_r = 100, d = 20), chi_max = 100,
    RRSVD k = 100, p = 10 (l = 110), q = 2, reference Omega stream regenerated on the device."""
    rng = np.random.default_rng(2000)
    g1, g2, ll, lm, lr = random_fragment(rng, 100, 20, 100, 20, 100, decay=0.85)
    gate, _ = np.linalg.qr(cplx_randn(rng, 400, 400))
    theta = ref.apply_gate(ref.build_theta(g1, g2, ll, lm, lr), gate)
    kw = dict(randomized=True, target_rank=100, oversampling=10, power_iterations=2, det_crossover=256, seed=77)
    be, rbe = P.DecimationBackend(**kw), ref.Backend(**kw)
    got = P.decimate(theta, ll, lr, 100, 0.0, be, ctx=ctx)
    want = ref.decimate(theta, ll, lr, 100, 0.0, rbe)
    assert got.randomized_path and want.randomized_path
    assert be.seed == rbe.seed == 78
    assert got.chi == want.chi == 100
    assert np.max(np.abs(np.asarray(got.lam) - want.lam)) < 1e-10
    assert abs(got.discarded - want.discarded) < 1e-10
    rec_g, rec_r = theta_from(got, ll, lr), theta_from(want, ll, lr)
    assert np.linalg.norm(rec_g - rec_r) / np.linalg.norm(rec_r) < 1e-9


def run_both(ref, site_dims, terms, dt, steps, chi, kw, locals_=None, chunks=1):
    """Evolve the reference MpsState and the device MPS side by side; yields after each chunk."""
    n = len(site_dims)
    locals_ = locals_ or [np.eye(d, dtype=complex)[0] for d in site_dims]
    rm = ref.RefMps(site_dims, locals_, chi, 0.0)
    dm = DeviceMps(site_dims, chi, 0.0)
    for s, v in enumerate(locals_):
        if not np.allclose(v, np.eye(site_dims[s])[0]):
            dm.set_site(s, np.asarray(v, complex).reshape(1, -1, 1), np.ones(1) if s < n - 1 else None)
    rbe, dbe = ref.Backend(**kw), P.DecimationBackend(**kw)
    tmap = dict(enumerate(terms))
    per = steps // chunks
    for _ in range(chunks):
        rd = rm.evolve(tmap, dt, per, rbe)
        dd = evolve(dm, tmap, dt, per, dbe)
        assert rbe.seed == dbe.seed
        yield rm, dm, rd, dd


def compare(rm, dm, ops, atol=1e-8):
    n = dm.n_sites
    assert [s[2] for s in rm.shapes()[:-1]] == dm.bond_dims()
    worst = 0.0
    for s in range(n):
        worst = max(worst, abs(rm.expectation_local(s, ops[s]) - dm.expectation_local(s, ops[s])))
    for b in range(n - 1):
        worst = max(worst, abs(rm.schmidt_entropy(b) - dm.schmidt_entropy(b)))
    assert worst < atol, worst
    return worst


@pytest.mark.parametrize("backend", ["deterministic", "rrsvd"])
def test_evolve_trace_c2_scale(ref, backend):
    """BASELINE configs[1]: Ising chain L = 64, d = 2, chi = 128, 3rd-order Trotter, 20 steps of
    dt = 0.05 from all-up; <sigma_z>(t) on every site and every bond entropy compared after each
    5-step chunk (a trace, 4 samples), plus chi profile, kept fraction and update count."""
    n, chi = 64, 128
    kw = {} if backend == "deterministic" else dict(randomized=True, target_rank=chi, oversampling=10,
                                                    power_iterations=2, det_crossover=0, seed=3)
    for rm, dm, rd, dd in run_both(ref, [2] * n, Mdl.ising_terms(n, 1.0, 1.0), 0.05, 20, chi, kw, chunks=4):
        assert dd.n_updates == rd["n_updates"] and dd.max_bond_dim == rd["max_bond_dim"]
        assert abs(dd.kept_fraction - rd["kept_fraction"]) < 1e-10
        compare(rm, dm, [Mdl.SZ] * n)
    assert dm.bond_dims()[n // 2] >= 8  # the state is genuinely entangled by the end


def tedopa_d20(n_chain=10, seed=7):
    t0, om, hop = Mdl.ohmic_chain(n_chain, 2001)
    dims, terms = Mdl.build_chain_terms(t0, om, hop, 20, 0.5 * Mdl.SZ + 0.5 * Mdl.SX, Mdl.SZ)
    rng = np.random.default_rng(seed)
    bos = cplx_randn(rng, n_chain, 20)
    locals_ = [np.array([1, 0], complex)] + [v / np.linalg.norm(v) for v in bos]
    return dims, terms, locals_


HEADLINE_KW = dict(randomized=True, target_rank=100, oversampling=10, power_iterations=2, det_crossover=256, seed=11)
TEDOPA_DT = 0.2


def test_evolve_tedopa_d20_chi100(ref):
    """BASELINE configs[2] model at its own d and chi: spin + 10 oscillators (d = 20), chi = 100,
    2 steps, RRSVD p = 10 / q = 2 with the reference default crossover (so the n = 2000 bonds take
    the randomized path exactly as in the benchmark); random local oscillator states so that the
    interior bonds saturate chi within the run.  <sigma_z>, <n_k> and entropies within 1e-8."""
    dims, terms, locals_ = tedopa_d20()
    ops = [Mdl.SZ] + [NUM20] * (len(dims) - 1)
    for rm, dm, rd, dd in run_both(ref, dims, terms, TEDOPA_DT, 2, 100, HEADLINE_KW, locals_, chunks=2):
        assert dd.n_updates == rd["n_updates"] and dd.max_bond_dim == rd["max_bond_dim"]
        assert abs(dd.kept_fraction - rd["kept_fraction"]) < 1e-10
        compare(rm, dm, ops)
    wide = [u for u in dd.updates if u["backend"] == "rrsvd"]
    assert wide, "no bond reached the randomized (n > 256) path"
    assert max(dm.bond_dims()) == 100


def test_philox_envelope_on_evolved_c3_theta(ctx, ref):
    """The stated statistical tolerance of the GPU's own RNG at the headline shape: the Theta of a
    chi-saturated interior bond of the evolved d = 20 chain (2000 x 2000, after its gate), decimated
    with k = 100, p = 10, q = 2 under 20 reference seeds (mt19937_64) and 8 Philox seeds.  Per kept
    lambda index and for w: |mean_dev - mean_ref| <= 5 s_ref sqrt(1/8 + 1/20) (+ a rounding floor
    of 1e-13 lambda_1, 1e-14 for w); spreads s_dev / s_ref in [1/6, 6] where the reference spread
    is above the floor, geometric mean in [1/2, 2].  DESIGN.md §4 records the measured envelope."""
    dims, terms, locals_ = tedopa_d20()
    dm = DeviceMps(dims, 100)
    for s, v in enumerate(locals_):
        dm.set_site(s, v.reshape(1, -1, 1), np.ones(1) if s < len(dims) - 1 else None)
    evolve(dm, dict(enumerate(terms)), TEDOPA_DT, 2, P.DecimationBackend(**HEADLINE_KW))
    bd = dm.bond_dims()
    b = next(b for b in range(2, len(dims) - 2) if bd[b - 1] == 100 and bd[b + 1] == 100)
    g1, g2 = dm.gamma(b), dm.gamma(b + 1)
    ll, lm, lr = dm.lam(b - 1), dm.lam(b), dm.lam(b + 1)
    gate = Mdl.bond_gate(terms[b], TEDOPA_DT)
    theta = ref.apply_gate(ref.build_theta(g1, g2, ll, lm, lr), gate)
    assert theta.shape == (20, 20, 100, 100)
    ref_l, ref_w = [], []
    for t in range(20):
        r = ref.decimate(theta, ll, lr, 100, 0.0, ref.Backend(**{**HEADLINE_KW, "seed": 1000 + t}))
        ref_l.append(r.lam)
        ref_w.append(r.discarded)
    dev_l, dev_w = [], []
    for t in range(8):
        be = P.DecimationBackend(**{**HEADLINE_KW, "seed": 5000 + t}, omega_mode=P.OMEGA_PHILOX)
        r = P.decimate(theta, ll, lr, 100, 0.0, be, ctx=ctx)
        assert r.chi == 100
        dev_l.append(np.asarray(r.lam))
        dev_w.append(r.discarded)
    ref_l, ref_w, dev_l, dev_w = map(np.array, (ref_l, ref_w, dev_l, dev_w))
    floor = 1e-13 * ref_l[0, 0]
    mu, sd = ref_l.mean(0), ref_l.std(0, ddof=1)
    dmu, dsd = dev_l.mean(0), dev_l.std(0, ddof=1)
    band = 5 * sd * np.sqrt(1 / 8 + 1 / 20) + floor
    assert np.all(np.abs(dmu - mu) <= band), np.max(np.abs(dmu - mu) / band)
    live = sd > 10 * floor
    ratio = dsd[live] / sd[live]
    assert live.sum() > 0 and np.all((ratio >= 1 / 6) & (ratio <= 6.0)), (ratio.min(), ratio.max())
    assert 0.5 <= np.exp(np.mean(np.log(ratio))) <= 2.0
    mw, sw = ref_w.mean(), ref_w.std(ddof=1)
    assert abs(dev_w.mean() - mw) <= 5 * sw * np.sqrt(1 / 8 + 1 / 20) + 1e-14
    assert 1 / 6 <= dev_w.std(ddof=1) / sw <= 6.0
    print(f"\n[envelope] bond {b}: max|dλ|/λ1 over seeds (ref) {np.max(sd) / mu[0]:.2e}, "
          f"|Δmean|/band max {np.max(np.abs(dmu - mu) / band):.2f}, spread ratio "
          f"{ratio.min():.2f}..{ratio.max():.2f} (geo {np.exp(np.mean(np.log(ratio))):.2f}), "
          f"w ref {mw:.3e}±{sw:.1e} dev {dev_w.mean():.3e}±{dev_w.std(ddof=1):.1e}")


def test_evolve_continues_after_abort_with_reference_seeds(ref):
    """tebd.cpp:317-321 abort inside a batched sweep, then a second evolve call on the same
    backend: the seed counter must be where the reference's is (the bonds after the aborting one
    take no seed), so the continued randomized run matches the reference's to 1e-8."""
    n, chi = 10, 6
    terms = Mdl.ising_terms(n, 1.0, 0.7)
    kw = dict(randomized=True, target_rank=6, oversampling=4, power_iterations=2, det_crossover=0, seed=21)
    rm, dm = ref.RefMps([2] * n, [np.array([1, 0], complex)] * n, chi, 0.0), DeviceMps([2] * n, chi, 0.0)
    rbe, dbe = ref.Backend(**kw), P.DecimationBackend(**kw)
    tmap = dict(enumerate(terms))
    rd = rm.evolve(tmap, 0.1, 30, rbe, abort_threshold=1e-7)
    dd = evolve(dm, tmap, 0.1, 30, dbe, abort_discarded_threshold=1e-7)
    assert rd["aborted"] and dd.aborted and rd["abort_step"] == dd.abort_step
    assert rbe.seed == dbe.seed, (rbe.seed, dbe.seed)
    rm.evolve(tmap, 0.1, 5, rbe)
    evolve(dm, tmap, 0.1, 5, dbe)
    assert rbe.seed == dbe.seed
    compare(rm, dm, [Mdl.SZ] * n)


def test_evolve_rejected_theta_leaves_state_consistent(ref):
    """A non-finite Theta inside a batched sweep (here: a NaN gate on one bond) raises
    contract_violation like the reference (tebd.cpp:156-160) and leaves the device state
    self-consistent: every site's dims match its buffer, all stored values are finite, and the
    rejected bond keeps its previous Gamma / lambda."""
    n = 8
    dm = DeviceMps([2] * n, 8)
    terms = dict(enumerate(Mdl.ising_terms(n, 1.0, 1.0)))
    evolve(dm, terms, 0.05, 2, P.DecimationBackend())
    before = [dm.gamma(s) for s in range(n)]
    lam3 = dm.lam(3)
    plan, gates = __import__("paper_1504_00992_b200.tebd", fromlist=["build_gates"]).build_gates(
        dm.site_dims, terms, 0.05)
    bad = {k: (np.full_like(g, np.nan) if k[1] == 3 else g) for k, g in gates.items()}
    be = P.DecimationBackend(seed=40)
    with pytest.raises(P.ContractViolation):
        evolve(dm, terms, 0.05, 1, be, gates=bad, plan=plan)
    for s in range(n):
        g = dm.gamma(s)
        assert g.shape == dm.dims(s) and np.all(np.isfinite(g))
    assert np.array_equal(dm.gamma(3), before[3]) and np.array_equal(dm.gamma(4), before[4])
    assert np.array_equal(dm.lam(3), lam3)
    # the failed sweep's first parity (bond 1, 3, 5): bond 1 committed (seed 40), bond 3 rejected
    # before taking a seed -> the counter stands at 41, where the reference's would
    assert be.seed == 41
    evolve(dm, terms, 0.05, 1, P.DecimationBackend())  # the state is usable again


def test_mpdo_tedopa_chain_matches_reference(ref):
    """BASELINE configs[3] shape at a feasible d: the mixed-state TEDOPA chain as
    an MPDO — vec(rho) with site dimension d^2 (spin 2 -> 4, oscillators d = 3 -> 9), Liouvillian
    terms L = H (x) 1 - 1 (x) H^T, so every two-site gate is U (x) U* (block-sparse for the
    number-conserving oscillator bonds) — evolved by the reference's own evolve and on the device
    with the same seeds: <sigma_z (x) 1> on the spin, <n (x) 1> on the oscillators and every bond
    entropy within 1e-8, identical chi profile."""
    n_chain, d, chi = 4, 3, 24
    t0, om, hop = Mdl.ohmic_chain(n_chain, 2001)
    dims, terms = Mdl.build_chain_terms(t0, om, hop, d, 0.5 * Mdl.SZ + 0.5 * Mdl.SX, Mdl.SZ)
    dims2, lterms = Mdl.mpdo_terms(dims, terms)
    rng = np.random.default_rng(3)
    psis = [np.array([1, 0], complex)] + [v / np.linalg.norm(v) for v in cplx_randn(rng, n_chain, d)]
    locals_ = [Mdl.mpdo_local(p) for p in psis]
    kw = dict(randomized=True, target_rank=chi, oversampling=6, power_iterations=2, det_crossover=40, seed=23)
    ops = [np.kron(Mdl.SZ, np.eye(2))] + [np.kron(np.diag(np.arange(d)), np.eye(d)).astype(complex)] * n_chain
    for rm, dm, rd, dd in run_both(ref, dims2, lterms, 0.1, 3, chi, kw, locals_, chunks=3):
        assert dd.max_bond_dim == rd["max_bond_dim"]
        assert abs(dd.kept_fraction - rd["kept_fraction"]) < 1e-10
        compare(rm, dm, ops)
    assert any(u["backend"] == "rrsvd" for u in dd.updates)
