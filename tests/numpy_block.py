"""TEST INFRASTRUCTURE: a chain block whose local compute is the numpy restatement of the
reference (oracle/port.py).  It lets the multi-rank host logic of parallel.py (partitioning, ghost
refresh, boundary return, global seed bookkeeping) run on CPU with gloo, and be compared with the
unpartitioned chain."""
import numpy as np

from oracle import port


def _np(x):
    if x is None:
        return None
    if hasattr(x, "detach"):
        return x.detach().cpu().numpy()
    return np.asarray(x)


class Diag:
    def __init__(self, kept):
        self.kept_fraction = kept


class NumpyBlock:
    def __init__(self, spec, gammas, lambdas, chi_max, backend_kwargs):
        self.spec = spec
        sites = spec.local_sites
        self.g = [np.array(gammas[s]) for s in sites]
        nb_local = len(sites) - 1
        self.lam = [np.array(lambdas[spec.a + i]) for i in range(nb_local)]
        n = spec.n_global
        self.edges = [np.array(lambdas[spec.a - 1]) if spec.a > 0 else None,
                      np.array(lambdas[sites[-1]]) if sites[-1] + 1 < n else None]
        self.chi_max = chi_max
        self.kw = backend_kwargs

    def get_gamma(self, i):
        return self.g[i].copy()

    def get_lambda(self, i):
        return self.lam[i].copy()

    def set_gamma(self, i, g, lam=None):
        self.g[i] = _np(g).copy()
        if lam is not None and i < len(self.lam):
            self.lam[i] = _np(lam).copy()

    def set_edges(self, left, right):
        self.edges = [_np(left), _np(right)]

    def sweep(self, parity, gates, dt, backend, seed):
        kept = 1.0
        nloc = len(self.g)
        for gb in sorted(gates):
            i = gb - self.spec.a
            ll = self.lam[i - 1] if i > 0 else self.edges[0]
            lr = self.lam[i + 1] if i + 2 < nloc else self.edges[1]
            th = port.apply_gate(port.build_theta(self.g[i], self.g[i + 1], ll, self.lam[i], lr), gates[gb])
            gl, lm, gr, w, chi, _, _ = port.decimate(th, ll, lr, self.chi_max, 0.0, seed=seed, **self.kw)
            seed += 1
            self.g[i], self.lam[i], self.g[i + 1] = gl, lm, gr
            kept *= 1.0 - w
        return Diag(kept)
