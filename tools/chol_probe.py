"""chol_inv latency probe: python tools/chol_probe.py [widths...] (single problems, device-resident)."""
import sys

sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1504_00992_b200 as P  # noqa: E402

ctx = P.Context(0)
rng = np.random.default_rng(0)
for l in [int(x) for x in sys.argv[1:]] or [32, 64, 110, 128, 168, 256]:
    a = rng.standard_normal((4 * l, l)) + 1j * rng.standard_normal((4 * l, l))
    g = torch.from_numpy(a.conj().T @ a).cuda()
    P.chol_inv(g, 10.0, ctx=ctx)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        P.chol_inv(g, 10.0, ctx=ctx)
    e1.record()
    torch.cuda.synchronize()
    print(f"chol_inv l={l}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us per call (incl. host)", flush=True)
