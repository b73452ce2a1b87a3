"""One C3 interior bond update (Θ → gate → RRSVD decimate) on the device, repeated; used as the
ncu target (launch list / full capture) and for per-stage timing.

  python tools/profile_update.py [--reps R] [--chi 100] [--d 20] [--p 10]
"""
import argparse
import sys
import time

import numpy as np

sys.path.insert(0, '.')
import torch  # noqa: E402

import paper_1504_00992_b200 as P  # noqa: E402
from paper_1504_00992_b200 import models as M  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--chi", type=int, default=100)
ap.add_argument("--d", type=int, default=20)
ap.add_argument("--p", type=int, default=10)
ap.add_argument("--q", type=int, default=2)
args = ap.parse_args()

chi, d = args.chi, args.d
rng = np.random.default_rng(0)
dev = "cuda"


def t(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(dev)


g1 = t((rng.standard_normal((chi, d, chi)) + 1j * rng.standard_normal((chi, d, chi))) / np.sqrt(chi * d))
g2 = t((rng.standard_normal((chi, d, chi)) + 1j * rng.standard_normal((chi, d, chi))) / np.sqrt(chi * d))
lam = 0.9 ** np.arange(chi)
lam = t(lam / np.linalg.norm(lam))
h = rng.standard_normal((d * d, d * d)) + 1j * rng.standard_normal((d * d, d * d))
gate = t(M.bond_gate(h + h.conj().T, 0.01))
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = P.Context(0, stream=stream.cuda_stream)
be = P.DecimationBackend(randomized=True, target_rank=chi, oversampling=args.p, power_iterations=args.q,
                         omega_mode=P.OMEGA_PHILOX)
for r in range(args.reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    m = P.build_theta_unfolded(g1, g2, lam, lam, lam, ctx=ctx)
    m2 = P.apply_gate_unfolded(gate, m, d, d, ctx=ctx)
    res = P.decimate_unfolded(m2, d, d, lam, lam, chi, 0.0, be, ctx=ctx)
    torch.cuda.synchronize()
    print(f"rep {r}: {1e3 * (time.perf_counter() - t0):.2f} ms  chi={res.chi} launches={ctx.launches}", flush=True)
