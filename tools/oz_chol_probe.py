"""Why the device's final CholeskyQR loses tail directions of an emulated Y = A Q~ (and not of a DMMA
one): numpy restatement of the device orth (shifted CholeskyQR, dead pivot <= 0 zeroed;
full schedule shifted | [ill] shifted, plain | plain) on the same Θ (tools/oz_tail_probe.py)."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_1504_00992_b200 as P  # noqa: E402
from oracle import ref  # noqa: E402
from paper_1504_00992_b200 import models as Mdl  # noqa: E402
from tests.test_gpu_headline import HEADLINE_KW, TEDOPA_DT, tedopa_d20  # noqa: E402

U = 2.0 ** -53


def chol_pass(y, shift_scale):
    g = y.conj().T @ y
    l = g.shape[0]
    s = shift_scale * U * np.trace(g).real
    a = g + s * np.eye(l)
    r = np.zeros_like(a)
    dead = np.zeros(l, bool)
    ill = False
    for i in range(l):
        d = (a[i, i] - np.sum(np.abs(r[:i, i]) ** 2)).real
        if not d > 0:
            dead[i] = True
            ill = True
            continue
        if shift_scale > 0 and d < 100 * s:
            ill = True
        r[i, i] = np.sqrt(d)
        for j in range(i + 1, l):
            r[i, j] = (a[i, j] - r[:i, i].conj() @ r[:i, j]) / r[i, i]
    t = np.zeros_like(r)
    live = ~dead
    t[np.ix_(live, live)] = np.linalg.inv(r[np.ix_(live, live)])
    return y @ t, ill, dead


def orth_full(y, m):
    sh = 10.0 * (m + y.shape[1])
    y, ill, d1 = chol_pass(y, sh)
    if ill:
        y, _, _ = chol_pass(y, sh)
        y, _, _ = chol_pass(y, 0.0)
    y, _, d4 = chol_pass(y, 0.0)
    return y, int(d1.sum()), int(d4.sum())


ctx = P.Context(0)
dims, terms, locals_ = tedopa_d20()
n = len(dims)
G = [np.asarray(v, complex).reshape(1, -1, 1) for v in locals_]
L = [np.ones(1) for _ in range(n - 1)]
be = ref.Backend(**HEADLINE_KW)


def theta_of(b, dt):
    gate = Mdl.bond_gate(terms[b], dt)
    ll = L[b - 1] if b > 0 else np.ones(G[b].shape[0])
    lr = L[b + 1] if b + 1 < n - 1 else np.ones(G[b + 1].shape[2])
    return ref.apply_gate(ref.build_theta(G[b], G[b + 1], ll, L[b], lr), gate), ll, lr


def update(b, dt):
    th, ll, lr = theta_of(b, dt)
    r = ref.decimate(th, ll, lr, 100, 0.0, be)
    G[b], G[b + 1], L[b] = r.gamma_left, r.gamma_right, np.asarray(r.lam)


for b in range(1, n - 1, 2):
    update(b, 0.5 * TEDOPA_DT)
th, ll, lr = theta_of(2, TEDOPA_DT)
a = np.transpose(th, (2, 0, 1, 3)).reshape(th.shape[2] * th.shape[0], th.shape[1] * th.shape[3])
m = a.shape[0]
om = ref.gaussian_test_matrix(a.shape[1], 110, 777)
for name, pr, ph in (("numpy", lambda x: a @ x, lambda x: a.conj().T @ x),
                     ("dmma", lambda x: P.gemm(a, False, x, ctx=ctx), lambda x: P.gemm(a, True, x, ctx=ctx)),
                     ("oz16", lambda x: P.ozaki_gemm(a, False, x, 16, ctx=ctx), lambda x: P.ozaki_gemm(a, True, x, 16, ctx=ctx))):
    y = pr(om)
    q, d1, d4 = orth_full(y, m)
    for _ in range(2):
        qt, _, _ = orth_full(ph(q), a.shape[1])
        y = pr(qt)
        q, d1, d4 = orth_full(y, m)
    sy = np.linalg.svd(y, compute_uv=False)
    s = np.linalg.svd(ph(q), compute_uv=False)
    print(f"{name:6s} final-Y sigma[95:110]/s1 {np.array2string(sy[95:110] / sy[0], precision=1)}")
    print(f"       dead first/last pass {d1}/{d4}; sigma(B)[88:101]/s1 {np.array2string(s[88:101] / s[0], precision=2)}")
r = P.rrsvd_fixed_rank(a, 100, 10, 2, 777, ctx=ctx)
s = np.asarray(r.sigma)
print("device fixed_rank sigma[88:100]/s1", np.array2string(s[88:100] / s[0], precision=2))


def dev_pass(y, shift_scale):
    g = P.gemm(y, True, y, ctx=ctx)
    t, nd, ill = P.chol_inv(g, shift_scale, ctx=ctx, flags=True)
    return P.gemm(y, False, t, ctx=ctx), nd, ill


# the device passes on a Y from the numpy power iteration, final product DMMA vs emulated
qt = None
y = a @ om
q, _ = np.linalg.qr(y)
for _ in range(2):
    qt, _ = np.linalg.qr(a.conj().T @ q)
    q, _ = np.linalg.qr(a @ qt)
for name, y in (("dmma", P.gemm(a, False, qt, ctx=ctx)), ("oz14", P.ozaki_gemm(a, False, qt, 14, ctx=ctx)),
                ("oz16", P.ozaki_gemm(a, False, qt, 16, ctx=ctx)), ("numpy", a @ qt)):
    sh = 10.0 * (m + 110)
    y1, n1, i1 = dev_pass(y, sh)
    y2, n2, i2 = dev_pass(y1, sh)
    y3, n3, _ = dev_pass(y2, 0.0)
    y4, n4, _ = dev_pass(y3, 0.0)
    print(f"device passes on Y[{name}]: dead {n1} {n2} {n3} {n4}, ill {i1} {i2}; cond(y2) {np.linalg.cond(y2):.2e}")


def span_orth(y, rows):
    sh = 10.0 * (rows + 110)
    y1, _, ill = dev_pass(y, sh)
    if ill:
        y1, _, _ = dev_pass(y1, sh)
    return y1


def full_orth(y, rows):
    sh = 10.0 * (rows + 110)
    y1, n1, ill = dev_pass(y, sh)
    if ill:
        y1, n2, _ = dev_pass(y1, sh)
        y1, n3, _ = dev_pass(y1, 0.0)
    y1, n4, _ = dev_pass(y1, 0.0)
    return y1, (n1, n4)


oz = lambda x: P.ozaki_gemm(a, False, x, 14, ctx=ctx)  # noqa: E731
ozh = lambda x: P.ozaki_gemm(a, True, x, 14, ctx=ctx)  # noqa: E731
dm = lambda x: P.gemm(a, False, x, ctx=ctx)  # noqa: E731
q = span_orth(oz(om), m)
for j in range(2):
    qt = span_orth(ozh(q), a.shape[1])
    print(f"  Q~ (span orth) cond {np.linalg.cond(qt):.2e}")
    if j == 1:
        for name, f in (("dmma", dm), ("oz14", oz), ("numpy", lambda x: a @ x)):
            qf, nd = full_orth(f(qt), m)
            s = np.linalg.svd(P.gemm(a, True, qf, ctx=ctx), compute_uv=False)
            print(f"device-pipeline final Y[{name}]: dead {nd}, sigma(B)[90:100]/s1 {np.array2string(s[90:100] / s[0], precision=2)}")
    q = span_orth(oz(qt), m)

print("--- intermediate bases with the full schedule")
q, _ = full_orth(oz(om), m)
for j in range(2):
    qt, _ = full_orth(ozh(q), a.shape[1])
    print(f"  Q~ (full orth) cond {np.linalg.cond(qt):.2e}")
    if j == 1:
        for name, f, fh in (("dmma", dm, lambda x: P.gemm(a, True, x, ctx=ctx)), ("oz14", oz, ozh),
                            ("oz16", lambda x: P.ozaki_gemm(a, False, x, 16, ctx=ctx), lambda x: P.ozaki_gemm(a, True, x, 16, ctx=ctx))):
            qf, nd = full_orth(f(qt), m)
            s = np.linalg.svd(fh(qf), compute_uv=False)
            print(f"full-orth pipeline final Y+B[{name}]: dead {nd}, sigma(B)[90:100]/s1 {np.array2string(s[90:100] / s[0], precision=2)}")
    q, _ = full_orth(oz(qt), m)
