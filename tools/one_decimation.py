"""One single-matrix RRSVD decimation (config-5 shape, default n=1000, k=100, p=10, q=2) after a
warm-up, for per-kernel launch lists:

  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/one.csv python tools/one_decimation.py --skip-warm
"""
import argparse
import sys

import numpy as np

sys.path.insert(0, '.')
import torch  # noqa: E402

import paper_1504_00992_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1000)
ap.add_argument("--k", type=int, default=100)
ap.add_argument("--p", type=int, default=10)
ap.add_argument("--reps", type=int, default=20)
args = ap.parse_args()

stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = P.Context(0, stream=stream.cuda_stream)
n, r = args.n, 300
G1 = torch.randn(n, r, dtype=torch.complex128, device="cuda") * torch.tensor(0.95 ** np.arange(r), device="cuda")
A = P.gemm(G1, False, torch.randn(r, n, dtype=torch.complex128, device="cuda"), ctx=ctx)
run = lambda: P.rrsvd_fixed_rank(A, args.k, args.p, 2, 3, mode=P.OMEGA_PHILOX, vectors=True, ctx=ctx)  # noqa: E731
run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(args.reps):
    run()
e1.record(stream)
e1.synchronize()
print(f"n={n} k={args.k} p={args.p}: {e0.elapsed_time(e1) / args.reps:.3f} ms per decimation, "
      f"{ctx.launch_count() if hasattr(ctx, 'launch_count') else '?'} launches total")
