"""FP64 pipes on this B200: DMMA alone, DFMA alone, and both issued together (8 DMMA chains +
8/16/32 DFMA chains per iteration) — does the vector pipe add throughput beside the tensor pipe?"""
import sys
sys.path.insert(0, ".")
import paper_1504_00992_b200 as P  # noqa: E402

ctx = P.Context(0)
for what, name in [(0, "dmma"), (1, "dfma"), (2, "dmma+8dfma"), (3, "dmma+16dfma"), (4, "dmma+32dfma")]:
    print(f"{name:14s} {P.probe_peak(what, ctx=ctx):7.2f} TF/s", flush=True)
