"""TEST INFRASTRUCTURE: numpy primitives for paper_1504_00992_b200.sharded.ShardedRrsvd, so the
row-sharded host logic (reduction order, replicated steps, the CholeskyQR schedule) runs on CPU
with gloo and is compared with the unsharded computation and with the reference."""
import numpy as np

from oracle import port

U = 2.0 ** -53


def chol_inv(g, shift_scale, flags=False):
    """Shifted Cholesky + triangular inverse (the device chol_inv's contract, smallla.cuh); with
    flags, also whether some pivot fell below 1e4 x the shift or died (kIllRatio)."""
    g = np.triu(np.asarray(g))
    g = g + np.triu(g, 1).conj().T
    l = g.shape[0]
    d = np.real(np.diag(g)).copy()
    s = shift_scale * U * float(np.sum(d))
    a = g + s * np.eye(l)
    r = np.zeros_like(a)
    dead = np.zeros(l, bool)
    ill = False
    for j in range(l):
        piv = a[j, j].real
        ill = ill or not piv >= 1e4 * s
        if not piv > 0.0:
            dead[j] = True
            ill = True
            continue
        rj = np.sqrt(piv)
        r[j, j] = rj
        r[j, j + 1:] = a[j, j + 1:] / rj
        a[j + 1:, j + 1:] -= np.outer(r[j, j + 1:].conj(), r[j, j + 1:])
    rp = r.copy()
    rp[dead, dead] = 1.0
    t = np.triu(np.linalg.inv(rp))
    t[:, dead] = 0.0
    t[dead, :] = 0.0
    return (t, ill) if flags else t


class NumpyOps:
    def gemm(self, a, adj_a, b):
        return (a.conj().T if adj_a else a) @ b

    def chol_inv(self, g, shift_scale):
        return chol_inv(g, shift_scale, flags=True)

    def svd(self, a):
        u, s, vh = np.linalg.svd(a, full_matrices=False)
        return u, s, vh.conj().T

    def omega(self, n, l, seed, mode):
        return port.gaussian_test_matrix(n, l, seed)

    def sumsq(self, a):
        return float(np.vdot(a, a).real)

    def zeros_like(self, a):
        return np.zeros_like(a)

    def add(self, a, b):
        return a + b
