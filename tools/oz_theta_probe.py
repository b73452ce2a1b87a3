"""Diagnose the emulated A-products on the Θ of the d = 20 TEDOPA parity chain (bond 2, after one
step): exact spectrum tail, product errors (DMMA vs emulated vs numpy), and a numpy RRSVD
(k = 100, p = 10, q = 2) whose A-products go through either path."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_1504_00992_b200 as P  # noqa: E402
from oracle import ref  # noqa: E402
from paper_1504_00992_b200 import models as Mdl  # noqa: E402
from paper_1504_00992_b200.tebd import DeviceMps, evolve  # noqa: E402
from tests.test_gpu_headline import HEADLINE_KW, TEDOPA_DT, tedopa_d20  # noqa: E402

ctx = P.Context(0)
dims, terms, locals_ = tedopa_d20()
rm = ref.RefMps(dims, locals_, 100, 0.0)
rbe = ref.Backend(**HEADLINE_KW)
rm.evolve(dict(enumerate(terms)), TEDOPA_DT, 1, rbe)
print("ref bond dims after 1 step", [s[2] for s in rm.shapes()[:-1]])
for b in (2, 4):
    g1, g2 = rm.gamma(b), rm.gamma(b + 1)
    ll, lm, lr = rm.lam(b - 1), rm.lam(b), rm.lam(b + 1)
    gate = Mdl.bond_gate(terms[b], TEDOPA_DT)
    th = ref.apply_gate(ref.build_theta(g1, g2, ll, lm, lr), gate)
    a = th.reshape(th.shape[0] * th.shape[1], -1) if th.ndim == 2 else np.transpose(th, (2, 0, 1, 3)).reshape(th.shape[2] * th.shape[0], th.shape[1] * th.shape[3])
    print(f"bond {b}: theta {th.shape} -> A {a.shape}, max|A| {np.max(np.abs(a)):.3e}")
    s = np.linalg.svd(a, compute_uv=False)
    print("  exact sigma[88:104]/s1:", np.array2string(s[88:104] / s[0], precision=2))
    rng = np.random.default_rng(0)
    om = (rng.standard_normal((a.shape[1], 110)) + 1j * rng.standard_normal((a.shape[1], 110))) / np.sqrt(2)
    want = a @ om
    scale = np.abs(a) @ np.abs(om)
    for name, got in (("dmma", P.gemm(a, False, om, ctx=ctx)), ("oz16", P.ozaki_gemm(a, False, om, 16, ctx=ctx)),
                      ("oz14", P.ozaki_gemm(a, False, om, 14, ctx=ctx))):
        print(f"  Y=A.Om {name}: max|err|/(|A||Om|) {np.max(np.abs(got - want) / scale):.2e}  normwise {np.linalg.norm(got - want) / np.linalg.norm(want):.2e}")

    def rr(prod, prodh):
        y = prod(om)
        q, _ = np.linalg.qr(y)
        for _ in range(2):
            z = prodh(q)
            qt, _ = np.linalg.qr(z)
            y = prod(qt)
            q, _ = np.linalg.qr(y)
        bh = prodh(q)
        return np.linalg.svd(bh, compute_uv=False)

    for name, pr, ph in (("numpy", lambda x: a @ x, lambda x: a.conj().T @ x),
                         ("dmma", lambda x: P.gemm(a, False, x, ctx=ctx), lambda x: P.gemm(a, True, x, ctx=ctx)),
                         ("oz16", lambda x: P.ozaki_gemm(a, False, x, 16, ctx=ctx), lambda x: P.ozaki_gemm(a, True, x, 16, ctx=ctx)),
                         ("oz16+dmmaB", lambda x: P.ozaki_gemm(a, False, x, 16, ctx=ctx), lambda x: P.gemm(a, True, x, ctx=ctx))):
        sr = rr(pr, ph)
        print(f"  rrsvd[{name:10s}] sigma[88:104]/s1:", np.array2string(sr[88:104] / sr[0], precision=2))
