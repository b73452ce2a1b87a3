"""The kernel variants behind the environment switches, each in its own process
(the switches are read once per process): every variant must meet the same parity bar as the
default, so an A/B switch can never hide a wrong result.

  * zgemm: 3M (default on the 64x56 tile) vs 4M, 3M on the 64x64 tile, TMA staging (default)
    vs the cp.async ring, and the shapes that fall back to cp.async (odd N; odd M under op C) —
    vs numpy, the reference's cblas_zgemm contract (linalg.cpp:20-40);
  * block Jacobi: the persistent sweep kernel (forced with RRSVD_B200_BJ_S=1) vs one launch per
    tournament step — singular values vs LAPACK (the reference's svd_full, linalg.cpp:67-88);
  * the RRSVD A-products: FP64 DMMA only (RRSVD_B200_OZAKI=0), the INT8 emulation with 15
    (default), 14 or 16 moduli, with the last two products on DMMA (RRSVD_B200_OZAKI_TAIL=2), and
    the span-only schedule for the power iteration's bases (RRSVD_B200_SPAN_PASSES=1) — the
    headline decimation vs the reference's decimate (tebd.cpp:141-237).
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

GEMM_SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, %(root)r)
import paper_1504_00992_b200 as P
rng = np.random.default_rng(5)
out = {}
for (m, k, n, adj) in [(2000, 2000, 110, False), (2000, 1500, 110, True), (400, 300, 256, False), (333, 100, 2000, False),
                       (250, 301, 111, False), (201, 173, 90, True), (64, 7, 56, False)]:
    a = rng.standard_normal((k, m) if adj else (m, k)) + 1j * rng.standard_normal((k, m) if adj else (m, k))
    b = rng.standard_normal((k, n)) + 1j * rng.standard_normal((k, n))
    c = P.gemm(a, adj, b)
    want = (a.conj().T if adj else a) @ b
    bound = np.abs(a.conj().T if adj else a) @ np.abs(b)
    out["%%d_%%d_%%d_%%d" %% (m, k, n, adj)] = float(np.max(np.abs(c - want) / bound))
print(json.dumps(out))
"""

SVD_SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, %(root)r)
import paper_1504_00992_b200 as P
rng = np.random.default_rng(11)
out = {}
for (m, n) in [(600, 500), (256, 256), (300, 420)]:
    s_true = 0.8 ** np.arange(min(m, n))
    u, _ = np.linalg.qr(rng.standard_normal((m, min(m, n))) + 1j * rng.standard_normal((m, min(m, n))))
    v, _ = np.linalg.qr(rng.standard_normal((n, min(m, n))) + 1j * rng.standard_normal((n, min(m, n))))
    a = (u * s_true) @ v.conj().T
    U, s, V = P.svd_full(a)
    sref = np.linalg.svd(a, compute_uv=False)
    recon = np.linalg.norm((U * s) @ V.conj().T - a) / np.linalg.norm(a)
    orth = np.linalg.norm(U.conj().T @ U - np.eye(U.shape[1]))
    out["%%dx%%d" %% (m, n)] = [float(np.max(np.abs(s - sref)) / sref[0]), float(recon), float(orth)]
print(json.dumps(out))
"""


DEC_SCRIPT = r"""
import ctypes as C, json, sys
import numpy as np
sys.path.insert(0, %(root)r)
import paper_1504_00992_b200 as P
from oracle import ref
from tests.conftest import cplx_randn
from tests.test_gpu_parity import random_fragment
ctx = P.Context(0)
ctx.check(P.lib().rrsvd_b200_set_gemm_timing(ctx.h, 1))
out = {}
for seed in (2000, 2001):
    rng = np.random.default_rng(seed)
    g1, g2, ll, lm, lr = random_fragment(rng, 100, 20, 100, 20, 100, decay=0.85)
    gate, _ = np.linalg.qr(cplx_randn(rng, 400, 400))
    theta = ref.apply_gate(ref.build_theta(g1, g2, ll, lm, lr), gate)
    kw = dict(randomized=True, target_rank=100, oversampling=10, power_iterations=2, det_crossover=256, seed=77)
    got = P.decimate(theta, ll, lr, 100, 0.0, P.DecimationBackend(**kw), ctx=ctx)
    want = ref.decimate(theta, ll, lr, 100, 0.0, ref.Backend(**kw))
    out[str(seed)] = [int(got.chi), int(want.chi), float(np.max(np.abs(np.asarray(got.lam) - want.lam))),
                      float(abs(got.discarded - want.discarded))]
vals = [C.c_double() for _ in range(3)] + [C.c_uint64()] + [C.c_double() for _ in range(2)]
ctx.check(P.lib().rrsvd_b200_ozaki_stats(ctx.h, *[C.byref(v) for v in vals]))
out["oz_calls"] = int(vals[3].value)
print(json.dumps(out))
"""


def run_variant(script, env_extra):
    env = dict(os.environ)
    env.update(env_extra)
    r = subprocess.run([sys.executable, "-c", script % {"root": ROOT}], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("env", [{"RRSVD_B200_GEMM_3M": "1"}, {"RRSVD_B200_GEMM_3M": "0"},
                                 {"RRSVD_B200_GEMM_3M": "1", "RRSVD_B200_GEMM_3M64": "1"},
                                 {"RRSVD_B200_GEMM_CFG": "56"}, {"RRSVD_B200_GEMM_CFG": "64"},
                                 {"RRSVD_B200_GEMM_TMA": "0"}, {"RRSVD_B200_GEMM_TMA": "0", "RRSVD_B200_GEMM_3M": "0"}])
def test_zgemm_variants_componentwise(env):
    """Every tile / complex-product form: |C - AB| <= 1e-13 |A||B| elementwise (FP64 GEMM error
    bound class; 3M's imaginary-part bound is a small constant times 4M's)."""
    res = run_variant(GEMM_SCRIPT, env)
    for shape, err in res.items():
        assert err <= 1e-13, (env, shape, err)


@pytest.mark.parametrize("env", [{}, {"RRSVD_B200_BJ_S": "1"}, {"RRSVD_B200_BJ_S": "1", "RRSVD_B200_BJ_PER_STEP": "1"},
                                 {"RRSVD_B200_BJ_MIN_C": "64"}, {"RRSVD_B200_BJ_CROSS": "0"}])
def test_block_jacobi_variants(env):
    """Persistent sweep kernel, per-step kernel and the block path for narrow problems:
    σ within 1e-13·σ1 of LAPACK, reconstruction and orthonormality at 1e-12."""
    res = run_variant(SVD_SCRIPT, env)
    for shape, (ds, recon, orth) in res.items():
        assert ds <= 1e-13 and recon <= 1e-12 and orth <= 1e-12, (env, shape, ds, recon, orth)


@pytest.mark.parametrize("env", [{"RRSVD_B200_OZAKI": "0"}, {}, {"RRSVD_B200_OZAKI": "16"}, {"RRSVD_B200_OZAKI": "14"},
                                 {"RRSVD_B200_OZAKI_TAIL": "2"}, {"RRSVD_B200_SPAN_PASSES": "1"},
                                 {"RRSVD_B200_OZAKI_PERSISTENT": "0"}, {"RRSVD_B200_OZAKI_GRID": "37"}])
def test_rrsvd_a_product_paths(env):
    """The headline decimation (2000 x 2000 Θ, RRSVD k = 100, p = 10, q = 2, reference Ω) with the
    A-products on the DMMA zgemm or on the INT8 emulation: chi equal, λ and w within 1e-10 of the
    reference; the emulation really ran unless switched off."""
    res = run_variant(DEC_SCRIPT, {"RRSVD_B200_OZAKI_MIN_WORK": "0", **env})  # (a single 2000^2 decimation)
    calls = res.pop("oz_calls")
    assert (calls == 0) == (env.get("RRSVD_B200_OZAKI") == "0"), (env, calls)
    for seed, (chi, rchi, dlam, dw) in res.items():
        assert chi == rchi == 100 and dlam < 1e-10 and dw < 1e-10, (env, seed, chi, rchi, dlam, dw)


@pytest.mark.parametrize("env", [{"RRSVD_B200_OZAKI_MIN": "256", "RRSVD_B200_OZAKI_MIN_WORK": "0"},
                                 {"RRSVD_B200_OZAKI_MIN": "256", "RRSVD_B200_OZAKI_MIN_WORK": "0", "RRSVD_B200_OZAKI": "16"}])
def test_emulated_products_on_every_bond_shape(env):
    """The d = 20 TEDOPA chain's evolve trace (tests/test_gpu_headline.py) with the emulated
    A-products lowered to every bond with both sides >= 256 (400 x 400 up to 2000 x 2000 Θ):
    chi profile, kept fraction and observables as the reference's."""
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_headline.py"), "-k", "tedopa_d20 or decimate_headline"],
                       env=e, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-2000:])
