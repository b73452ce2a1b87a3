"""Noise floor of the RRSVD sketch on an exactly rank-deficient A (rank r < l): the singular
values beyond r that the decimation's numerically-zero cutoff (sigma <= 1e-15 sigma_1,
tebd.cpp:193) tests — device (DMMA or emulated A-products, per RRSVD_B200_OZAKI) vs the reference."""
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_1504_00992_b200 as P  # noqa: E402
from oracle import ref  # noqa: E402

m = n = int(os.environ.get("N", "2000"))
r = int(os.environ.get("R", "92"))
rng = np.random.default_rng(1)
u, _ = np.linalg.qr(rng.standard_normal((m, r)) + 1j * rng.standard_normal((m, r)))
v, _ = np.linalg.qr(rng.standard_normal((n, r)) + 1j * rng.standard_normal((n, r)))
s = np.exp(-np.arange(r) / 10.0)
a = (u * s) @ v.conj().T
ctx = P.Context(0)
for tag, fn in (("device", lambda: P.rrsvd_fixed_rank(a, 100, 10, 2, 11, ctx=ctx)),):
    out = fn()
    sig = np.asarray(out[1] if isinstance(out, tuple) else out.sigma)
    print(tag, os.environ.get("RRSVD_B200_OZAKI", "0"), "sigma[r-2:r+8]/sigma1:", np.array2string(sig[r - 2:r + 8] / sig[0], precision=2))
if ref.available() and os.environ.get("REF", "1") == "1":
    res = ref.fixed_rank(a, 100, 10, 2, 11, vectors=False)
    sig = np.asarray(res[1] if isinstance(res, tuple) else res["sigma"])
    print("reference", "sigma[r-2:r+8]/sigma1:", np.array2string(sig[r - 2:r + 8] / sig[0], precision=2))
