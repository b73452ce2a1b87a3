"""Full-SVD timing probe across sizes (single problems): python tools/jac_probe.py [sizes...]"""
import sys
import time

sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1504_00992_b200 as P  # noqa: E402

ctx = P.Context(0)
rng = np.random.default_rng(0)
for m in [int(x) for x in sys.argv[1:]] or [110, 256]:
    a = torch.from_numpy(rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))).cuda()
    P.svd_full(a, ctx=ctx)
    torch.cuda.synchronize()
    reps = 5 if m <= 512 else 1
    t0 = time.perf_counter()
    for _ in range(reps):
        P.svd_full(a, ctx=ctx)
    torch.cuda.synchronize()
    print(m, "svd_full ms", round((time.perf_counter() - t0) / reps * 1e3, 2), flush=True)
