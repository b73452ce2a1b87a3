"""Secondary measurements of the BASELINE.json configs beside the bench.py headline (config 3):

  config 1 — RRSVD of a 512² matrix, σ_i = e^{-i/10}, k=64, p=10, q=2: single-call latency
             (device-resident and through host buffers) and batched decimations/s, with the
             reference (oracle/_ref) timed on the host cores and σ parity to it;
  config 5 — RRSVD sweep n = 1000…16000, k=100, p=10, q=2 (exponentially decaying synthetic
             spectrum), device time per decimation vs the reference on the host (n ≤ 4000).

  python tools/measure_configs.py [--quick] > profiles/r01_configs.json
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, '.')
import torch  # noqa: E402

import paper_1504_00992_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--quick", action="store_true")
args = ap.parse_args()

stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = P.Context(0, stream=stream.cuda_stream)
try:
    from oracle import ref
    have_ref = ref.available()
    if have_ref:
        ref.set_threads(os.cpu_count() or 1)
except Exception:
    have_ref = False


def dev_time(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps


def cpu_time(fn, reps):
    fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t0) / reps


rng = np.random.default_rng(0)


def structured(n, sigma):
    u, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    return np.ascontiguousarray((u * sigma) @ v.conj().T)


# ---------------------------------------------------------------- config 1
n = 512
sig = np.exp(-np.arange(n) / 10.0)
A = structured(n, sig)
Ad = torch.from_numpy(A).cuda()
k, p, q = 64, 10, 2
lat_dev = dev_time(lambda: P.rrsvd_fixed_rank(Ad, k, p, q, 7, mode=P.OMEGA_PHILOX, ctx=ctx), 20)
lat_ref_mode = dev_time(lambda: P.rrsvd_fixed_rank(Ad, k, p, q, 7, ctx=ctx), 10)
t0 = time.perf_counter()
for _ in range(10):
    P.rrsvd_fixed_rank(A, k, p, q, 7, ctx=ctx)  # host buffers: H2D/D2H inside
lat_e2e = (time.perf_counter() - t0) / 10
batch = 64
As = [torch.from_numpy(structured(n, sig) if i < 2 else A).cuda() for i in range(batch)]
seeds = list(range(batch))
bt = dev_time(lambda: P.rrsvd_fixed_rank_batch(As, k, p, q, seeds, ctx=ctx), 3)
line = {"config": "c1_rrsvd_512_k64_p10_q2", "device_latency_ms": round(1e3 * lat_dev, 3),
        "device_latency_ms_reference_omega_stream": round(1e3 * lat_ref_mode, 3),
        "e2e_latency_ms_host_buffers": round(1e3 * lat_e2e, 3),
        "batched_decimations_per_s": round(batch / bt, 1), "batch": batch}
if have_ref:
    tr = cpu_time(lambda: ref.fixed_rank(A, k, p, q, 7), 3)
    _, s_ref, _, w_ref = ref.fixed_rank(A, k, p, q, 7)
    res = P.rrsvd_fixed_rank(A, k, p, q, 7, ctx=ctx)  # reference Ω stream regenerated on device
    line.update({"reference_s_per_call": round(tr, 4), "reference_decimations_per_s": round(1 / tr, 2),
                 "reference_cores": os.cpu_count(),
                 "sigma_max_rel_err_vs_reference": float(np.max(np.abs(res.sigma - s_ref) / s_ref)),
                 "w_abs_err_vs_reference": abs(res.discarded_weight - w_ref)})
print(json.dumps(line), flush=True)

# ---------------------------------------------------------------- config 5
ns = [1000, 2000, 4000] if args.quick else [1000, 2000, 4000, 8000, 16000]
for n in ns:
    r = 300
    G1 = torch.randn(n, r, dtype=torch.complex128, device="cuda") * torch.tensor(0.95 ** np.arange(r), device="cuda")
    G2h = torch.randn(r, n, dtype=torch.complex128, device="cuda")
    Ad = P.gemm(G1, False, G2h, ctx=ctx)
    reps = 5 if n <= 4000 else 2
    t = dev_time(lambda: P.rrsvd_fixed_rank(Ad, 100, 10, 2, 3, mode=P.OMEGA_PHILOX, vectors=True, ctx=ctx), reps)
    flops = 8.0 * 6 * n * n * 110
    line = {"config": f"c5_rrsvd_n{n}_k100_p10_q2", "device_s_per_decimation": round(t, 5),
            "decimations_per_s": round(1 / t, 2), "rrsvd_gemm_tflops": round(flops / t / 1e12, 2)}
    if have_ref and n <= (2000 if args.quick else 4000):
        Ah = Ad.cpu().numpy()
        tr = cpu_time(lambda: ref.fixed_rank(Ah, 100, 10, 2, 3, vectors=True), 1)
        line.update({"reference_s_per_decimation": round(tr, 3), "speedup_vs_reference": round(tr / t, 1),
                     "reference_cores": os.cpu_count()})
    print(json.dumps(line), flush=True)
    del Ad, G1, G2h
    torch.cuda.empty_cache()

# ---------------------------------------------------------------- config 5, deterministic arm
# (BASELINE configs[4]: "vs reference CPU RRSVD and deterministic SVD"): full SVD of a graded
# full-rank n x n matrix (column scales 0.99^i), device vs the reference's svd_full (zgesdd)
if not args.quick:
    for n in [1000, 4000]:
        G1 = torch.randn(n, n, dtype=torch.complex128, device="cuda") * torch.tensor(0.99 ** np.arange(n), device="cuda")
        Ad = P.gemm(G1, False, torch.randn(n, n, dtype=torch.complex128, device="cuda"), ctx=ctx)
        t = dev_time(lambda: P.svd_full(Ad, ctx=ctx), 2 if n <= 1000 else 1)
        line = {"config": f"c5_full_svd_{n}x{n}", "device_s_per_svd": round(t, 4)}
        if have_ref:
            Ah = Ad.cpu().numpy()
            tr = cpu_time(lambda: ref.svd_full(Ah), 1)
            _, s_r, _ = ref.svd_full(Ah)
            _, s_d, _ = P.svd_full(Ad, ctx=ctx)
            line.update({"reference_s_per_svd": round(tr, 3), "speedup_vs_reference": round(tr / t, 2),
                         "reference_cores": os.cpu_count(),
                         "sigma_max_abs_err_over_s1": float(np.max(np.abs(s_d.cpu().numpy() - s_r)) / s_r[0])})
        print(json.dumps(line), flush=True)
        del Ad, G1
        torch.cuda.empty_cache()

# ---------------------------------------------------------------- config 3, full-SVD arm (A13)
if not args.quick:
    n = 2000
    G1 = torch.randn(n, n, dtype=torch.complex128, device="cuda") * torch.tensor(0.99 ** np.arange(n), device="cuda")
    Ad = P.gemm(G1, False, torch.randn(n, n, dtype=torch.complex128, device="cuda"), ctx=ctx)
    t = dev_time(lambda: P.svd_full(Ad, ctx=ctx), 1)
    line = {"config": "c3_full_svd_2000x2000", "device_s_per_svd": round(t, 4)}
    if have_ref:
        Ah = Ad.cpu().numpy()
        tr = cpu_time(lambda: ref.svd_full(Ah), 1)
        _, s_r, _ = ref.svd_full(Ah)
        _, s_d, _ = P.svd_full(Ad, ctx=ctx)
        line.update({"reference_s_per_svd": round(tr, 3), "speedup_vs_reference": round(tr / t, 2),
                     "reference_cores": os.cpu_count(),
                     "sigma_max_abs_err_over_s1": float(np.max(np.abs(s_d.cpu().numpy() - s_r)) / s_r[0])})
    print(json.dumps(line), flush=True)
