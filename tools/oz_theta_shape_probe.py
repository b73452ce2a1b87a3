import sys, time
sys.path.insert(0, ".")
import torch
import paper_1504_00992_b200 as P
ctx = P.Context(0)
g = torch.Generator(device="cuda").manual_seed(0)
a = torch.randn(2000, 100, dtype=torch.complex128, device="cuda", generator=g)
x = torch.randn(100, 2000, dtype=torch.complex128, device="cuda", generator=g)
for name, f in (("dmma", lambda: P.gemm(a, False, x, ctx=ctx)), ("oz15", lambda: P.ozaki_gemm(a, False, x, 15, ctx=ctx))):
    f(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(20):
        c = f()
    torch.cuda.synchronize()
    print(name, (time.perf_counter() - t) / 20 * 1e3, "ms", float(torch.max(torch.abs(c - a @ x))))
