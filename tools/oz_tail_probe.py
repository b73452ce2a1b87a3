"""The Θ of the d = 20 TEDOPA chain's even bonds in the middle sweep of step 1 (the decimations where
the emulated final products cut chi below the reference's): exact spectrum tail vs a numpy RRSVD
(k = 100, p = 10, q = 2, the reference's Omega) whose A-products run on the DMMA zgemm or the INT8
emulation — is the emulation less accurate there, or only different at the noise floor?"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_1504_00992_b200 as P  # noqa: E402
from oracle import ref  # noqa: E402
from paper_1504_00992_b200 import models as Mdl  # noqa: E402
from tests.test_gpu_headline import HEADLINE_KW, TEDOPA_DT, tedopa_d20  # noqa: E402

ctx = P.Context(0)
dims, terms, locals_ = tedopa_d20()
n = len(dims)
G = [np.asarray(v, complex).reshape(1, -1, 1) for v in locals_]
L = [np.ones(1) for _ in range(n - 1)]
be = ref.Backend(**HEADLINE_KW)


def lam(b):
    return L[b] if 0 <= b < n - 1 else np.ones(1)


def theta_of(b, dt):
    gate = Mdl.bond_gate(terms[b], dt)
    ll = L[b - 1] if b > 0 else np.ones(G[b].shape[0])
    lr = L[b + 1] if b + 1 < n - 1 else np.ones(G[b + 1].shape[2])
    th = ref.apply_gate(ref.build_theta(G[b], G[b + 1], ll, L[b], lr), gate)
    return th, ll, lr


def update(b, dt):
    th, ll, lr = theta_of(b, dt)
    r = ref.decimate(th, ll, lr, 100, 0.0, be)
    G[b], G[b + 1], L[b] = r.gamma_left, r.gamma_right, np.asarray(r.lam)


for b in range(1, n - 1, 2):
    update(b, 0.5 * TEDOPA_DT)
for b in range(0, n - 1, 2):
    if b in (2, 4):
        th, ll, lr = theta_of(b, TEDOPA_DT)
        a = np.transpose(th, (2, 0, 1, 3)).reshape(th.shape[2] * th.shape[0], th.shape[1] * th.shape[3])
        s = np.linalg.svd(a, compute_uv=False)
        print(f"bond {b}: A {a.shape}; exact sigma[90:104]/s1:", np.array2string(s[90:104] / s[0], precision=2))
        om = ref.gaussian_test_matrix(a.shape[1], 110, 12345)
        import os
        kw = dict(HEADLINE_KW, seed=be.seed)
        got = P.decimate(th, ll, lr, 100, 0.0, P.DecimationBackend(**kw), ctx=ctx)
        want = ref.decimate(th, ll, lr, 100, 0.0, ref.Backend(**kw))
        print(f"  decimate (OZAKI={os.environ.get('RRSVD_B200_OZAKI')}, TAIL={os.environ.get('RRSVD_B200_OZAKI_TAIL')}):"
              f" chi dev {got.chi} ref {want.chi}; lam tail dev {np.asarray(got.lam)[-3:]} ref {want.lam[-3:]}")
        if os.environ.get("QUICK"):
            update(b, TEDOPA_DT)
            continue

        def rr(prod, prodh):
            y = prod(om)
            q, _ = np.linalg.qr(y)
            for _ in range(2):
                qt, _ = np.linalg.qr(prodh(q))
                q, _ = np.linalg.qr(prod(qt))
            return np.linalg.svd(prodh(q), compute_uv=False)

        for name, pr, ph in (
                ("numpy", lambda x: a @ x, lambda x: a.conj().T @ x),
                ("dmma", lambda x: P.gemm(a, False, x, ctx=ctx), lambda x: P.gemm(a, True, x, ctx=ctx)),
                ("oz14", lambda x: P.ozaki_gemm(a, False, x, 14, ctx=ctx), lambda x: P.ozaki_gemm(a, True, x, 14, ctx=ctx)),
                ("oz16", lambda x: P.ozaki_gemm(a, False, x, 16, ctx=ctx), lambda x: P.ozaki_gemm(a, True, x, 16, ctx=ctx))):
            sr = rr(pr, ph)
            print(f"  rrsvd[{name:5s}] sigma[90:104]/s1:", np.array2string(sr[90:104] / sr[0], precision=2))
    update(b, TEDOPA_DT)
