"""One TEBD step of a bench workload (default c2) after a warm-up step, for ncu launch lists:

  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file out.csv \
      python tools/one_step.py --workload c2
"""
import argparse
import sys

sys.path.insert(0, '.')
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1504_00992_b200 as P  # noqa: E402
from paper_1504_00992_b200 import models as M  # noqa: E402
from paper_1504_00992_b200.tebd import DeviceMps, PreparedGates, build_gates, evolve  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2")
ap.add_argument("--serial", action="store_true", help="lanes off (one stream)")
args = ap.parse_args()
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = P.Context(0, stream=stream.cuda_stream)
if args.serial:
    ctx.check(P.lib().rrsvd_b200_set_overlap(ctx.h, 0))
wl = bench.workload(args.workload)
plan, gh = build_gates(wl["site_dims"], wl["terms"], wl["dt"])
gates = PreparedGates(gh, ctx)
g, l = M.synthetic_saturated_mps(wl["site_dims"], wl["chi"], seed=1)
mps = DeviceMps(wl["site_dims"], wl["chi"], 0.0, ctx=ctx)
be = P.DecimationBackend(omega_mode=P.OMEGA_PHILOX, **wl["backend"])
for _ in range(2):
    mps.load(g, l)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    evolve(mps, wl["terms"], wl["dt"], 1, be, record_updates=False, gates=gates, plan=plan)
    e1.record(stream)
    e1.synchronize()
    print(f"{args.workload}: {e0.elapsed_time(e1):.2f} ms per step")
