"""DMMA throughput vs residency: one CTA per SM with W warps, C independent accumulator chains per
warp (rrsvd_b200_probe_peak code 100 + 10 W + C) — how many warps / chains the FP64 tensor pipe
needs to saturate."""
import sys
sys.path.insert(0, ".")
import paper_1504_00992_b200 as P  # noqa: E402

ctx = P.Context(0)
print("warps/SM  chains:   1      2      4      8   (TF/s)")
for w in (2, 4, 8, 12, 16):
    row = [P.probe_peak(100 + 10 * w + c, ctx=ctx) for c in (1, 2, 4, 8)]
    print(f"{w:8d}        " + " ".join(f"{x:6.2f}" for x in row), flush=True)
