"""Debug: step-by-step device evolve vs the reference evolve (prints per-step divergence)."""
import sys

import numpy as np

sys.path.insert(0, '.')
import paper_1504_00992_b200 as P  # noqa: E402
from oracle import ref  # noqa: E402
from paper_1504_00992_b200 import models as Mdl  # noqa: E402
from paper_1504_00992_b200.tebd import DeviceMps, evolve  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else 'ising'
if which == 'ising':
    n, chi = 8, 8
    site_dims = [2] * n
    terms = {b: t for b, t in enumerate(Mdl.ising_terms(n, 1.0, 0.7))}
    kw = dict(randomized=True, target_rank=8, oversampling=8, power_iterations=2, det_crossover=0, seed=5)
else:
    n_chain, d, chi = 5, 4, 12
    t0, om, hop = Mdl.ohmic_chain(n_chain, 2001)
    site_dims, tl = Mdl.build_chain_terms(t0, om, hop, d, 0.5 * Mdl.SZ + 0.5 * Mdl.SX, Mdl.SZ)
    terms = {b: t for b, t in enumerate(tl)}
    n = len(site_dims)
    kw = dict(randomized=True, target_rank=chi, oversampling=4, power_iterations=2, det_crossover=8, seed=11)
dt = 0.05
for det in [False, True]:
    kk = {} if det else dict(kw)
    rm = ref.RefMps(site_dims, [np.eye(d_, dtype=complex)[0] for d_ in site_dims], chi, 0.0)
    dm = DeviceMps(site_dims, chi, 0.0)
    rbe, dbe = ref.Backend(**kk), P.DecimationBackend(**kk)
    print('det' if det else 'rnd')
    for step in range(12):
        rd = rm.evolve(terms, dt, 1, rbe)
        dd = evolve(dm, terms, dt, 1, dbe)
        ent = max(abs(rm.schmidt_entropy(b) - dm.schmidt_entropy(b)) for b in range(n - 1))
        lam = max(np.max(np.abs(rm.lam(b) - dm.lam(b))) if len(rm.lam(b)) == len(dm.lam(b)) else 99
                  for b in range(n - 1))
        print(step, f"ent {ent:.2e} lam {lam:.2e} kf {abs(rd['kept_fraction'] - dd.kept_fraction):.2e}",
              [len(rm.lam(b)) for b in range(n - 1)], [len(dm.lam(b)) for b in range(n - 1)],
              f"{rd['kept_fraction']:.3e}", flush=True)
