import numpy as np, paper_1504_00992_b200 as P
ctx = P.Context(0)
rng = np.random.default_rng(0)
for (m, n) in [(64,64),(128,128),(200,200),(256,256),(256,128)]:
    r = min(m,n); s_true = np.logspace(0,-12,r)
    uq,_ = np.linalg.qr(rng.standard_normal((m,r))+1j*rng.standard_normal((m,r)))
    vq,_ = np.linalg.qr(rng.standard_normal((n,r))+1j*rng.standard_normal((n,r)))
    a = (uq*s_true)@vq.conj().T
    u,s,v = P.svd_full(a, ctx=ctx)
    print(m, n, np.max(np.abs(s-s_true)), flush=True)
