"""Probe: χ profile of a short d=20 TEDOPA chain (spin + 10 bosons, χ_max=100) after 1 and 2
Trotter steps from random local boson states, for a few dt — picks the parity-test setting in
which the interior bonds reach the C3 shape (χ_l = χ_r = 100, n = 2000) within 2 steps."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1504_00992_b200 as P  # noqa: E402
from paper_1504_00992_b200 import models as Mdl  # noqa: E402
from paper_1504_00992_b200.tebd import DeviceMps, evolve  # noqa: E402

n_chain, d, chi = 10, 20, 100
t0, om, hop = Mdl.ohmic_chain(n_chain, 2001)
dims, terms = Mdl.build_chain_terms(t0, om, hop, d, 0.5 * Mdl.SZ + 0.5 * Mdl.SX, Mdl.SZ)
rng = np.random.default_rng(7)
locals_ = [np.array([1, 0], complex)] + [v / np.linalg.norm(v) for v in
                                          (rng.standard_normal((n_chain, d)) + 1j * rng.standard_normal((n_chain, d)))]
for dt in (0.05, 0.1, 0.2, 0.4, 0.8):
    dm = DeviceMps(dims, chi)
    for s, v in enumerate(locals_):
        dm.set_site(s, v.reshape(1, -1, 1), np.ones(1) if s < len(dims) - 1 else None)
    be = P.DecimationBackend(randomized=True, target_rank=chi, oversampling=10, power_iterations=2, seed=1)
    tmap = dict(enumerate(terms))
    for step in range(2):
        t = time.time()
        dd = evolve(dm, tmap, dt, 1, be)
        print(f"dt={dt} step={step + 1} bonds={dm.bond_dims()} rrsvd={sum(u['backend'] == 'rrsvd' for u in dd.updates)}"
              f" t={time.time() - t:.2f}s", flush=True)
