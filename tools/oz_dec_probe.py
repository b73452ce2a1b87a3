"""Decimations of the d = 20 TEDOPA chain's bonds (after one reference step) through the library
(env RRSVD_B200_OZAKI selects the A-product path) vs the reference decimate."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_1504_00992_b200 as P  # noqa: E402
from oracle import ref  # noqa: E402
from paper_1504_00992_b200 import models as Mdl  # noqa: E402
from tests.test_gpu_headline import HEADLINE_KW, TEDOPA_DT, tedopa_d20  # noqa: E402

ctx = P.Context(0)
dims, terms, locals_ = tedopa_d20()
rm = ref.RefMps(dims, locals_, 100, 0.0)
rbe = ref.Backend(**HEADLINE_KW)
rm.evolve(dict(enumerate(terms)), TEDOPA_DT, 1, rbe)
for b in range(1, len(dims) - 2):
    g1, g2 = rm.gamma(b), rm.gamma(b + 1)
    ll, lm, lr = rm.lam(b - 1), rm.lam(b), rm.lam(b + 1)
    gate = Mdl.bond_gate(terms[b], TEDOPA_DT)
    th = ref.apply_gate(ref.build_theta(g1, g2, ll, lm, lr), gate)
    kw = dict(HEADLINE_KW, seed=5)
    got = P.decimate(th, ll, lr, 100, 0.0, P.DecimationBackend(**kw), ctx=ctx)
    want = ref.decimate(th, ll, lr, 100, 0.0, ref.Backend(**kw))
    d = np.max(np.abs(np.asarray(got.lam)[:min(got.chi, want.chi)] - want.lam[:min(got.chi, want.chi)]))
    print(f"bond {b}: theta {th.shape} chi dev {got.chi} ref {want.chi} max|dlam| {d:.2e} rr {got.randomized_path}")
