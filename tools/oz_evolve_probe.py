"""Device evolve (RRSVD_B200_OZAKI from the env) vs the reference evolve on the d = 20 TEDOPA chain:
per-bond chi and lambda differences after each of `steps` single steps."""
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from tests.test_gpu_headline import HEADLINE_KW, TEDOPA_DT, run_both, tedopa_d20  # noqa: E402
from oracle import ref  # noqa: E402

dims, terms, locals_ = tedopa_d20()
steps = int(os.environ.get("STEPS", "1"))
for rm, dm, rd, dd in run_both(ref, dims, terms, TEDOPA_DT, steps, 100, HEADLINE_KW, locals_, chunks=steps):
    rb = [s[2] for s in rm.shapes()[:-1]]
    print("ref chi", rb)
    print("dev chi", dm.bond_dims())
    for b in range(len(dims) - 1):
        lr, ld = np.asarray(rm.lam(b)), np.asarray(dm.lam(b))
        k = min(len(lr), len(ld))
        print(f"  bond {b}: chi {len(lr)}/{len(ld)} max|dlam| {np.max(np.abs(lr[:k] - ld[:k])):.2e} lam_min ref {lr[-1]:.2e} dev {ld[-1]:.2e}")
