"""CPU tests: the oracle is pinned before it is trusted.

- oracle/port.py (numpy restatement) vs the golden vectors produced by the compiled reference
  (tests/golden/golden.npz, tests/golden/make_golden.py);
- the compiled reference (oracle/_ref) reproduces its own goldens (when it is built);
- the C-ABI library loads and exports every symbol include/rrsvd_b200.h declares.
"""
import os

import numpy as np
import pytest

from oracle import port

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


def test_port_gaussian_stream_matches_reference():
    """randomized.cpp:17-45: mt19937_64 draws bit-exact; Box–Muller within a few ulps (numpy's
    log/sin/cos vs glibc)."""
    for i in range(3):
        n, l, seed = (int(x) for x in GOLD[f"omega{i}_args"])
        got = port.gaussian_test_matrix(n, l, seed)
        want = GOLD[f"omega{i}"]
        assert np.max(np.abs(got - want)) <= 4e-15 * np.max(np.abs(want))


def test_port_fixed_rank_and_sketch():
    u, s, v, w = port.rrsvd_fixed_rank(GOLD["fr_a"], 16, 6, 2, 7)
    assert np.max(np.abs(s - GOLD["fr_sigma"]) / GOLD["fr_sigma"]) < 1e-12
    assert abs(w - float(GOLD["fr_w"])) < 1e-14
    assert np.linalg.norm((u * s) @ v.conj().T - GOLD["fr_proj"]) < 1e-12
    _, s2, _, w2 = port.rrsvd_sketched_svd(GOLD["sk_a"], 20, 1, 3)
    assert np.max(np.abs(s2 - GOLD["sk_sigma"])) < 1e-12 * GOLD["sk_sigma"][0]
    assert abs(w2 - float(GOLD["sk_w"])) < 1e-14


def test_port_fixed_precision_matches_reference(ref):
    """port.rrsvd_fixed_precision (randomized.cpp:124-176) against the compiled reference: the same
    final width and certificate for growth_block 0 / 1 / 3 / 5 / 7 / 50 — including a basis grown
    past the rank of a rank-6 matrix — and σ, w to rounding."""
    lf, rf = ref.gaussian_test_matrix(120, 6, 4), ref.gaussian_test_matrix(80, 6, 5)
    low = lf @ rf.conj().T
    for g in (0, 1, 3, 5):
        for l0 in (1, 2, 5, 8):
            _, s_r, _, _, c_r = ref.fixed_precision(low, 1e-8, 4, l0, 1, 11, growth_block=g)
            _, s_p, _, _, c_p = port.rrsvd_fixed_precision(low, 1e-8, 4, l0, 1, 11, growth_block=g)
            assert (len(s_p), c_p) == (len(s_r), c_r), (g, l0)
            assert np.max(np.abs(s_p[:6] - s_r[:6])) <= 1e-12 * s_r[0]
    a = ref.structured_matrix(0.97 ** np.arange(400), 400, 5, 6)
    for g in (0, 7, 50):
        _, s_r, _, w_r, c_r = ref.fixed_precision(a, 1e-3, 10, 20, 2, 17, growth_block=g)
        _, s_p, _, w_p, c_p = port.rrsvd_fixed_precision(a, 1e-3, 10, 20, 2, 17, growth_block=g)
        assert (len(s_p), c_p) == (len(s_r), c_r)
        assert np.max(np.abs(s_p - s_r)) <= 1e-12 * s_r[0] and abs(w_p - w_r) <= 1e-13


def test_port_theta_gate_decimate():
    lam = GOLD["tb_lam"]
    th = port.build_theta(GOLD["tb_g1"], GOLD["tb_g2"], lam, lam, lam)
    assert np.max(np.abs(th - GOLD["tb_theta"])) < 1e-14
    th2 = port.apply_gate(th, GOLD["tb_gate"])
    assert np.max(np.abs(th2 - GOLD["tb_theta_gated"])) < 1e-14
    for tag, kw in [("det", {}), ("rnd", dict(randomized=True, target_rank=4, oversampling=4, det_crossover=0,
                                              seed=9))]:
        gl, lm, gr, w, chi, rnd, pinv = port.decimate(th2, lam, lam, 4, 0.0, **kw)
        assert chi == int(GOLD[f"dec_{tag}_chi"]) and rnd == (tag == "rnd")
        assert np.max(np.abs(lm - GOLD[f"dec_{tag}_lambda"])) < 1e-12
        assert abs(w - float(GOLD[f"dec_{tag}_w"])) < 1e-13
        cl, d1, k = gl.shape
        left = gl.reshape(cl * d1, k) * np.repeat(lam, d1)[:, None]
        right = gr.reshape(k, -1) * np.tile(lam, gr.shape[1])[None, :]
        assert np.linalg.norm((left * lm) @ right - GOLD[f"dec_{tag}_recon"]) < 1e-12


def test_port_decimate_edge_cases():
    bell = np.zeros((2, 2, 1, 1), complex)
    bell[0, 0] = bell[1, 1] = 1 / np.sqrt(2)
    _, lm, _, _, chi, _, _ = port.decimate(bell, None, None, 4, 0.0)
    assert chi == 2 and np.allclose(lm, 1 / np.sqrt(2))
    with pytest.raises(ValueError):
        port.decimate(np.zeros((2, 2, 1, 1), complex), None, None, 4, 0.0)
    bad = bell.copy()
    bad[0, 1, 0, 0] = np.inf
    with pytest.raises(ValueError):
        port.decimate(bad, None, None, 4, 0.0)


def test_models_match_golden_chain():
    from paper_1504_00992_b200 import models as M
    t0, om, hop = M.ohmic_chain(12, 2001)
    assert abs(t0 - float(GOLD["chain_t0"])) < 1e-14
    assert np.max(np.abs(om - GOLD["chain_omegas"])) < 1e-12
    assert np.max(np.abs(hop - GOLD["chain_hoppings"])) < 1e-12


def test_reference_reproduces_its_goldens(ref):
    for i in range(3):
        n, l, seed = (int(x) for x in GOLD[f"omega{i}_args"])
        assert np.array_equal(ref.gaussian_test_matrix(n, l, seed), GOLD[f"omega{i}"])
    _, s, _, w = ref.fixed_rank(GOLD["fr_a"], 16, 6, 2, 7)
    assert np.max(np.abs(s - GOLD["fr_sigma"]) / GOLD["fr_sigma"]) < 1e-13


def test_abi_library_exports_every_header_symbol():
    """The drop-in boundary: librrsvd_b200.so loads (no GPU needed) and exports each entry point
    of include/rrsvd_b200.h."""
    import paper_1504_00992_b200 as P
    from paper_1504_00992_b200._lib import header_symbols
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(P.lib(), s), s
    assert b"sm_100a" in P.lib().rrsvd_b200_version()


def test_no_cpu_fallback_without_gpu():
    """Without a device the context refuses to open — the product path never falls back."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1504_00992_b200 as P
    with pytest.raises(P.CudaError):
        P.Context(0)
