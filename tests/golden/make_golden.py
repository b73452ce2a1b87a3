"""Generates tests/golden/golden.npz by running the REFERENCE implementation (oracle/_ref, the
unmodified /root/reference core compiled by oracle/Makefile) single-threaded on fixed seeds.

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py

The reference ships no golden vectors for this path, so these fixtures are the
pin for both the numpy restatement (oracle/port.py) and the device path.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
from oracle import ref  # noqa: E402


def main():
    ref.set_threads(1)
    g = {}
    # 1. Ω: gaussian_test_matrix (randomized.cpp:79-86)
    for i, (n, l, seed) in enumerate([(7, 3, 5), (64, 10, 123456789), (300, 20, 7)]):
        g[f"omega{i}"] = ref.gaussian_test_matrix(n, l, seed)
        g[f"omega{i}_args"] = np.array([n, l, seed], np.uint64)
    # 2. fixed rank on a config-1-style matrix (σ_i = e^{-i/10}), smaller n
    n = 128
    sig = np.exp(-np.arange(n) / 10.0)
    a = ref.structured_matrix(sig, n, 1, 2)
    u, s, v, w = ref.fixed_rank(a, 16, 6, 2, 7)
    g.update(fr_a=a, fr_sigma=s, fr_w=np.array(w), fr_proj=(u * s) @ v.conj().T)
    # 3. sketched SVD
    rng = np.random.default_rng(3)
    b = rng.standard_normal((64, 48)) + 1j * rng.standard_normal((64, 48))
    u, s, v, w = ref.sketched_svd(b, 20, 1, 3)
    g.update(sk_a=b, sk_sigma=s, sk_w=np.array(w))
    # 4. build_theta + apply_gate + decimate on a fragment (det + randomized)
    cl, d1, cm, d2, cr = 6, 2, 6, 2, 6
    g1 = (rng.standard_normal((cl, d1, cm)) + 1j * rng.standard_normal((cl, d1, cm))) / np.sqrt(cl * d1)
    g2 = (rng.standard_normal((cm, d2, cr)) + 1j * rng.standard_normal((cm, d2, cr))) / np.sqrt(cm * d2)
    lam = 0.6 ** np.arange(6)
    lam /= np.linalg.norm(lam)
    gate = np.linalg.qr(rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4)))[0]
    th = ref.build_theta(g1, g2, lam, lam, lam)
    th2 = ref.apply_gate(th, gate)
    g.update(tb_g1=g1, tb_g2=g2, tb_lam=lam, tb_gate=gate, tb_theta=th, tb_theta_gated=th2)
    for tag, be in [("det", ref.Backend()),
                    ("rnd", ref.Backend(randomized=True, target_rank=4, oversampling=4, det_crossover=0, seed=9))]:
        d = ref.decimate(th2, lam, lam, 4, 0.0, be)
        g[f"dec_{tag}_lambda"] = d.lam
        g[f"dec_{tag}_w"] = np.array(d.discarded)
        g[f"dec_{tag}_chi"] = np.array(d.chi)
        left = d.gamma_left.reshape(cl * d1, d.chi) * np.repeat(lam, d1)[:, None]
        right = d.gamma_right.reshape(d.chi, d2 * cr) * np.tile(lam, d2)[None, :]
        g[f"dec_{tag}_recon"] = (left * d.lam) @ right
    # 5. evolve: Ising L=8, χ=8, dt=0.05, 10 steps, deterministic, from all-up
    nsite = 8
    terms = {b_: t for b_, t in enumerate(ref.ising_terms(nsite, 1.0, 1.0))}
    mps = ref.RefMps([2] * nsite, [np.array([1, 0], complex)] * nsite, 8, 0.0)
    be = ref.Backend()
    diag = mps.evolve(terms, 0.05, 10, be)
    sz = np.diag([1.0, -1.0]).astype(complex)
    g["ev_sz"] = np.array([mps.expectation_local(s_, sz).real for s_ in range(nsite)])
    g["ev_entropy"] = np.array([mps.schmidt_entropy(b_) for b_ in range(nsite - 1)])
    g["ev_kept_fraction"] = np.array(diag["kept_fraction"])
    # 6. TEDOPA chain map (chainmap.cpp:58-68,108-153), h²(x)=x on [0,1]
    x = np.linspace(0.0, 1.0, 2001)
    t0, om, hop = ref.stieltjes(x, x.copy(), 12)
    g.update(chain_t0=np.array(t0), chain_omegas=om, chain_hoppings=hop)
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
    np.savez_compressed(out, **g)
    print("wrote", out, os.path.getsize(out), "bytes")


if __name__ == "__main__":
    main()
