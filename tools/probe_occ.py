"""DMMA throughput vs residency (warps/SM) and ILP (independent accumulators per warp)."""
import sys

sys.path.insert(0, '.')
import paper_1504_00992_b200 as P  # noqa: E402

ctx = P.Context(0)
for w in (4, 8, 12, 16, 24, 32):
    print(w, "warps/SM:", " ".join(f"chains={c}: {P.probe_peak(100 + w * 10 + c, ctx=ctx):6.2f}" for c in (1, 2, 4, 8)),
          flush=True)
