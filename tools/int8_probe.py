"""Feasibility probe: INT8 tensor-core GEMM throughput at the RRSVD A-product shapes."""
import torch
dev = "cuda"
def t(fn, it=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / it
for (m, k, n) in [(4000, 2000, 224), (4000, 2000, 256), (2000, 4000, 224), (16000, 8192, 224), (8192, 8192, 8192), (4000*16, 2000, 224)]:
    a = torch.randint(-127, 127, (m, k), dtype=torch.int8, device=dev)
    b = torch.randint(-127, 127, (n, k), dtype=torch.int8, device=dev).t()
    ms = t(lambda: torch._int_mm(a, b))
    print(f"int_mm {m}x{k}x{n}: {ms*1e3:.1f} us  {2*m*k*n/ms/1e9:.1f} TOPS")
    ab, bb = a.to(torch.bfloat16), b.to(torch.bfloat16)
    ms = t(lambda: ab @ bb)
    print(f"bf16   {m}x{k}x{n}: {ms*1e3:.1f} us  {2*m*k*n/ms/1e9:.1f} TF/s")
a = torch.randint(-127, 127, (16, 4000, 2000), dtype=torch.int8, device=dev)
b = torch.randint(-127, 127, (16, 224, 2000), dtype=torch.int8, device=dev)
for i in range(1):
    ms = t(lambda: [torch._int_mm(a[j], b[j].t()) for j in range(16)])
    print(f"16 x int_mm 4000x2000x224: {ms*1e3:.1f} us  {16*2*4000*2000*224/ms/1e9:.1f} TOPS")
