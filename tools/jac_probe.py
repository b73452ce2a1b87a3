import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1504_00992_b200 as P
ctx = P.Context(0)
rng = np.random.default_rng(0)
for m in [110, 256]:
    a = torch.from_numpy(rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))).cuda()
    P.svd_full(a, ctx=ctx); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5): P.svd_full(a, ctx=ctx)
    torch.cuda.synchronize()
    print(m, "svd_full ms", (time.perf_counter() - t0) / 5 * 1e3, flush=True)
