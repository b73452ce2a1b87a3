#!/usr/bin/env python
"""Benchmark of the B200-native TEBD two-site decimation path (BASELINE.json metric).

Headline workload (north star, BASELINE.json configs[2]): TEDOPA spin-boson chain, spin + 100
oscillators (d=20), χ=100 (n = d·χ = 2000 at interior bonds), RRSVD decimation p=10, q=2,
3rd-order Trotter (150 two-site updates per step).  A "step" is one TEBD step on a χ-saturated
synthetic MPS (Gaussian Γ, λ ∝ 0.9^i) held in HBM; the gates are the real
TEDOPA bond gates.  Inputs are larger than L2 (MPS ≈ 320 MB > 126 MB) so no L2 flush is needed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload c3|c3p100|c3det|c2|c5|c4]

Under torchrun (N > 1) the chain is partitioned into contiguous site blocks, one per rank (weak
scaling: 100 oscillator sites per rank, boundary Γ/λ exchanged by NCCL send/recv), and rank 0
prints the max-over-ranks timing.  Only the JSON line goes to stdout (library and NCCL chatter is
redirected to stderr).  `--impl reference` times the reference C++ core (oracle/_ref, built
from /root/reference) on the host cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

_JSON_FD = None  # the process's original stdout: the JSON line only (see main)


def emit(obj) -> None:
    line = json.dumps(obj) + "\n"
    if _JSON_FD is None:
        sys.stdout.write(line)
        sys.stdout.flush()
    else:
        os.write(_JSON_FD, line.encode())

METRIC = "TEBD steps/s at n=d·χ (RRSVD decimation; FP64 tensor-core roofline of the zgemm stages)"


# ----------------------------------------------------------------------------- workloads

def workload(name: str):
    from paper_1504_00992_b200 import models as M
    if name == "c3":
        site_dims, terms = M.tedopa_system(n_chain=100, boson_dim=20)
        return dict(name="tedopa_spin_boson_101sites_d20_chi100", site_dims=site_dims,
                    terms={b: t for b, t in enumerate(terms)}, chi=100, dt=0.01,
                    backend=dict(randomized=True, target_rank=0, oversampling=10, power_iterations=2,
                                 det_crossover=256, seed=7),
                    desc="TEDOPA spin-boson, spin + 100 bosons (d=20), chi=100, n=2000, RRSVD p=10 q=2")
    if name == "c3p100":  # config 3 with the paper's oversampling p = k (l = 200)
        site_dims, terms = M.tedopa_system(n_chain=100, boson_dim=20)
        return dict(name="tedopa_spin_boson_101sites_d20_chi100_p100", site_dims=site_dims,
                    terms={b: t for b, t in enumerate(terms)}, chi=100, dt=0.01,
                    backend=dict(randomized=True, target_rank=0, oversampling=100, power_iterations=2,
                                 det_crossover=256, seed=7),
                    desc="TEDOPA spin-boson, spin + 100 bosons (d=20), chi=100, n=2000, RRSVD p=100 q=2")
    if name == "c3det":  # config 3's "vs full SVD" arm: deterministic decimation (tebd.cpp:185)
        site_dims, terms = M.tedopa_system(n_chain=100, boson_dim=20)
        return dict(name="tedopa_spin_boson_101sites_d20_chi100_fullsvd", site_dims=site_dims,
                    terms={b: t for b, t in enumerate(terms)}, chi=100, dt=0.01,
                    backend=dict(randomized=False, det_crossover=256, seed=7),
                    desc="TEDOPA spin-boson, spin + 100 bosons (d=20), chi=100, n=2000, full SVD decimation")
    if name == "c2":
        n = 64
        return dict(name="ising_L64_d2_chi128", site_dims=[2] * n,
                    terms={b: t for b, t in enumerate(M.ising_terms(n, 1.0, 1.0))}, chi=128, dt=0.01,
                    backend=dict(randomized=False, det_crossover=256, seed=7),
                    desc="Ising L=64, d=2, chi=128 (n=256), deterministic (reference default crossover)")
    if name == "c4mpdo":  # config 4 at a feasible d: the mixed-state TEDOPA chain as an MPDO
        site_dims, terms = M.tedopa_system(n_chain=100, boson_dim=4)
        dims2, lterms = M.mpdo_terms(site_dims, terms)
        return dict(name="mpdo_tedopa_101sites_d4sq16_chi200", site_dims=dims2,
                    terms={b: t for b, t in enumerate(lterms)}, chi=200, dt=0.01,
                    backend=dict(randomized=True, target_rank=0, oversampling=10, power_iterations=2,
                                 det_crossover=256, seed=7),
                    desc="MPDO TEDOPA (vec rho, sites d^2 = 16: oscillators d = 4), chi = 200, n = 3200, "
                         "Liouvillian gates U (x) U*, RRSVD p=10 q=2 (config 4; d^2 = 400 would make one "
                         "Theta 102 GB)")
    if name == "c2rr":  # config 2's RRSVD arm: randomized decimation forced (tebd.cpp:167-186)
        n = 64
        return dict(name="ising_L64_d2_chi128_rrsvd", site_dims=[2] * n,
                    terms={b: t for b, t in enumerate(M.ising_terms(n, 1.0, 1.0))}, chi=128, dt=0.01,
                    backend=dict(randomized=True, target_rank=0, oversampling=10, power_iterations=2,
                                 det_crossover=0, seed=7),
                    desc="Ising L=64, d=2, chi=128 (n=256), RRSVD p=10 q=2 forced (det_crossover=0)")
    raise SystemExit(f"unknown workload {name}")


def measured_hbm_peak():
    """HBM copy bandwidth from MEASURED_PEAKS.json (driver-written), else the profiling guide's
    fallback (6.65 TB/s)."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "MEASURED_PEAKS.json")) as f:
            v = float(json.load(f)["hbm_gbs"])
        return v, "MEASURED_PEAKS.json hbm_gbs (copy bandwidth, read+write bytes)"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md; MEASURED_PEAKS.json absent)"


def emulated_entry(flops, ms, nbytes, calls, prep_ms, prep_bytes, gemm_ms=0.0, gemm_bytes=0.0) -> dict:
    """The RRSVD A-products on the INT8 tensor cores (csrc/ozaki.cuh), from the serial roofline pass:
    kept out of the DMMA roofline above (its `frac` covers the FP64 zgemm launches only)."""
    moduli = int(os.environ.get("RRSVD_B200_OZAKI", "15") or 0)
    tail = int(os.environ.get("RRSVD_B200_OZAKI_TAIL", "0") or 0)
    if ms <= 0:
        return {"enabled": False, "moduli": moduli}
    return {"enabled": True, "moduli": moduli,
            "scheme": "Chinese-remainder (Ozaki-II) emulation of the complex-FP64 product: A and the panel "
                      "equilibrated by powers of two, int8 residues, tcgen05.mma kind::i8 into TMEM, 96-bit "
                      "fixed-point CRT to FP64",
            "products": ("all 2q+2 = 6 A-products per decimation (Y = A Omega, the power iteration, B^H = A^H Q)"
                         if tail == 0 else f"all but the last {tail} of the 2q+2 A-products per decimation (those on "
                                           "the FP64 DMMA zgemm, RRSVD_B200_OZAKI_TAIL)"),
            "ms_per_step": round(ms, 3), "fp64_equivalent_tflops": round(flops / (ms * 1e-3) / 1e12, 2),
            "algorithmic_GBps": round(nbytes / (ms * 1e-3) / 1e9, 1), "launch_groups": int(calls),
            "int8_gemm_roofline": ({"bound": "hbm", "kernel": "oz_gemm_persistent_kernel (tcgen05.mma kind::i8)",
                                    "achieved": round(gemm_bytes / (gemm_ms * 1e-3) / 1e9, 1),
                                    "peak": measured_hbm_peak()[0], "unit": "GB/s",
                                    "frac": round(gemm_bytes / (gemm_ms * 1e-3) / 1e9 / measured_hbm_peak()[0], 4),
                                    "peak_source": measured_hbm_peak()[1],
                                    "traffic_note": "achieved counts the algorithmic bytes (A residue tiles + panel "
                                                    "read, residue products written) over the event-timed launches; "
                                                    "ncu DRAM bytes in profiles/r02_ozaki_summary.md",
                                    "ms_per_step": round(gemm_ms, 3)} if gemm_ms > 0 else None),
            "a_preparation_ms_per_step": round(prep_ms, 3),
            "a_preparation_GBps": round(prep_bytes / (prep_ms * 1e-3) / 1e9, 1) if prep_ms > 0 else None,
            "note": "ms are event-timed per launch group (residue panel + INT8 GEMM + CRT) in the serial pass; "
                    "fp64_equivalent_tflops counts 8 m n k per complex product; the INT8 GEMM kernel's own "
                    "roofline (HBM-bound) is in profiles/r02_ozaki_summary.md"}


def bench_config(wl, ups, world) -> dict:
    """The `config` object — identical in both arms (ours and --impl reference)."""
    from paper_1504_00992_b200 import models as M
    dims = M.saturated_bond_dims(wl["site_dims"], wl["chi"])
    sd = wl["site_dims"]
    mps_bytes = sum(16 * (1 if s == 0 else dims[s - 1]) * sd[s] * (1 if s == len(sd) - 1 else dims[s])
                    for s in range(len(sd))) + 8 * sum(dims)
    return {"workload": wl["name"], "desc": wl["desc"], "sites": len(sd), "chi": wl["chi"],
            "updates_per_step": ups, "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
            "l2": ("inputs larger than L2 (MPS %.0f MB > 126 MB)" % (mps_bytes / 1e6)) if mps_bytes > 126e6 else
                  ("MPS %.0f MB fits L2; no flush: consecutive TEBD steps rewrite the whole state, which is "
                   "the workload" % (mps_bytes / 1e6))}


def updates_per_step(site_dims, terms):
    nb = len(site_dims) - 1
    return sum(1 for par, _ in [(1, .5), (0, 1.), (1, .5)] for b in range(par, nb, 2) if b in terms)


def state_bytes(gammas, lambdas):
    return int(sum(g.size * 16 for g in gammas) + sum(l.size * 8 for l in lambdas))


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- multi-GPU arm

def run_partitioned(args, rank, world, local_rank):
    """N > 1: chain-block partition over N GPUs, weak scaling.  The TEDOPA chain
    grows with N — spin + 100·N oscillators, chain coefficients of config 3 repeated per block —
    and rank r owns one config-3-sized block (rank 0: spin + 100 bosons; rank r ≥ 1: 100
    bosons).  Boundary Γ/λ travel by NCCL send/recv (torch.distributed P2P) around every sweep."""
    import torch
    import torch.distributed as dist

    import paper_1504_00992_b200 as P
    from paper_1504_00992_b200 import models as M
    from paper_1504_00992_b200.parallel import BlockSpec, ChainPartition, DeviceBlock, TorchComm

    # RRSVD_B200_BENCH_GLOO=1: gloo with host-staged exchanges and every rank on GPU
    # local_rank % device_count — a protocol check of this N > 1 driver on a one-GPU box (ranks
    # never wait on each other's kernels); never a measurement.
    gloo = os.environ.get("RRSVD_B200_BENCH_GLOO", "0") not in ("", "0")
    if gloo:
        local_rank %= torch.cuda.device_count()
    red = "cpu" if gloo else "cuda"  # where the reductions' tensors live
    torch.cuda.set_device(local_rank)
    if "RANK" not in os.environ:  # --force-partition without torchrun: a one-rank group on 127.0.0.1
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # rank / transport lines on stderr for the driver
    if gloo:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = P.Context(local_rank, stream=stream.cuda_stream)
    peak_dmma = P.probe_peak(0, ctx=ctx)
    t0c, om, hop = M.ohmic_chain(100)
    nb = 100 * world
    om_x = np.tile(om, world)
    hop_x = np.tile(np.append(hop, hop[-1]), world)[:nb - 1]
    mpdo = args.workload == "c4mpdo"
    boson = 4 if mpdo else 20
    site_dims, terms_l = M.build_chain_terms(t0c, om_x, hop_x, boson, 0.5 * M.SZ + 0.5 * M.SX, M.SZ)
    if mpdo:  # config 4: the mixed-state chain as an MPDO (Liouvillian terms, d^2 sites)
        site_dims, terms_l = M.mpdo_terms(site_dims, terms_l)
    n = len(site_dims)
    chi, dt = (200 if mpdo else 100), 0.01
    bounds = [0] + [1 + 100 * (r + 1) for r in range(world)]
    a, b = bounds[rank], bounds[rank + 1]
    spec = BlockSpec(rank, world, a, b, n)
    bonds_dims = M.saturated_bond_dims(site_dims, chi)
    plan = M.trotter_plan_3rd(dt)
    gates = {}
    for s, (p, c) in enumerate(plan):
        for j in spec.local_bonds:
            if j % 2 == p:
                gates[(s, j)] = M.bond_gate(terms_l[j], c * dt)
    from paper_1504_00992_b200.tebd import PreparedGates
    gates = PreparedGates(gates, ctx)  # resident on the device, block structure analysed once

    def site_gamma(gs):  # deterministic per global site, so ghost copies equal the owner's
        rng = np.random.default_rng(1000 + gs)
        cl = 1 if gs == 0 else bonds_dims[gs - 1]
        cr = 1 if gs == n - 1 else bonds_dims[gs]
        g = rng.standard_normal((cl, site_dims[gs], cr)) + 1j * rng.standard_normal((cl, site_dims[gs], cr))
        return g / np.sqrt(cl * site_dims[gs])

    def lam(j):
        v = 0.9 ** np.arange(bonds_dims[j])
        return v / np.linalg.norm(v)

    blk = DeviceBlock(spec, site_dims, chi, ctx=ctx)
    local = spec.local_sites

    def load_state():
        blk.set_edges(lam(a - 1) if a > 0 else None, lam(local[-1]) if local[-1] + 1 < n else None)
        for i, gs in enumerate(local):
            blk.set_gamma(i, site_gamma(gs), lam(gs) if i + 1 < len(local) else None)

    load_state()
    # the data plane: rrsvd_b200_evolve_partitioned over NCCL behind the C ABI (default), or the
    # Python driver over torch.distributed P2P (RRSVD_B200_PARTITION=python; gloo protocol checks)
    native = not gloo and os.environ.get("RRSVD_B200_PARTITION", "native") != "python"
    if native:
        from paper_1504_00992_b200.parallel import NativeComm, evolve_partitioned
        uid = [NativeComm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = NativeComm.nccl(ctx, world, rank, uid[0])
        local_gates = {(s_, j - a): h for (s_, j), h in gates.items()}

        class _Native:
            def evolve(self, gates_, plan_, dt_, n_steps_, be_, base_, step0=0):
                be_.seed = base_
                evolve_partitioned(blk.mps, comm, a, n, local_gates, plan_, list(range(n - 1)), n_steps_, be_,
                                   step0=step0)
        part = _Native()
    else:
        part = ChainPartition(blk, TorchComm(red), list(range(n - 1)))
    be = P.DecimationBackend(omega_mode=P.OMEGA_PHILOX, randomized=True, target_rank=0, oversampling=10,
                             power_iterations=2, det_crossover=256, seed=7)
    dist.barrier()  # a collective on the whole group before the first batched P2P exchange (NCCL)
    for w in range(args.warmup):
        part.evolve(gates, plan, dt, 1, be, 7, step0=w)
        load_state()
    dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = ctx.launches
    with ClockSampler(local_rank) as clk:
        ev0.record(stream)
        part.evolve(gates, plan, dt, args.steps, be, 7)
        ev1.record(stream)
        ev1.synchronize()
    elapsed = ev0.elapsed_time(ev1) / 1e3
    gpu_launches = ctx.launches - launches0
    t = torch.tensor([elapsed], device=red)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed = float(t.item())
    ups_rank = sum(1 for p, _ in plan for j in spec.local_bonds if j % 2 == p)
    ups = torch.tensor([ups_rank], device=red, dtype=torch.float64)
    dist.all_reduce(ups)

    # ---- end-to-end: every step each rank uploads its block from pinned host memory through the
    # C ABI, steps, and downloads its owned sites back; max over ranks of the wall time
    import ctypes as C
    pin_g = [torch.from_numpy(site_gamma(gs)).pin_memory() for gs in local]
    pin_l = [torch.from_numpy(lam(gs)).pin_memory() if i + 1 < len(local) else None for i, gs in enumerate(local)]
    own = b - a
    e2e_steps = max(1, min(args.steps, 2))
    out_bufs = [torch.empty(blk.mps.dims(i), dtype=torch.complex128).pin_memory() for i in range(own)]
    dist.barrier()
    torch.cuda.synchronize()
    te0 = time.perf_counter()
    h2d = d2h = 0
    for st in range(e2e_steps):
        blk.set_edges(lam(a - 1) if a > 0 else None, lam(local[-1]) if local[-1] + 1 < n else None)
        for i in range(len(local)):
            blk.set_gamma(i, pin_g[i], pin_l[i])
        h2d = sum(t.numel() * 16 for t in pin_g) + sum(t.numel() * 8 for t in pin_l if t is not None)
        part.evolve(gates, plan, dt, 1, be, 7, step0=st)
        d2h = 0
        for i in range(own):
            if tuple(out_bufs[i].shape) != blk.mps.dims(i):  # (saturated state: never)
                out_bufs[i] = torch.empty(blk.mps.dims(i), dtype=torch.complex128).pin_memory()
            buf = out_bufs[i]
            ctx.check(P.lib().rrsvd_b200_mps_get_site(blk.mps.h, i, None, C.c_void_p(buf.data_ptr()), None))
            d2h += buf.numel() * 16
    torch.cuda.synchronize()
    te = torch.tensor([time.perf_counter() - te0], device=red)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e = world * e2e_steps / float(te.item())
    if rank == 0:
        emit({
            "metric": METRIC, "value": round(world * args.steps / elapsed, 6), "unit": "steps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * elapsed / args.steps, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "c128 (fp64)",
            "data": "synthetic χ-saturated MPS + TEDOPA bond gates (config-3 chain coefficients repeated per block)",
            "config": {"workload": (f"mpdo_tedopa_{n}sites_d4sq16_chi200_chain_blocks" if mpdo else
                                    f"tedopa_spin_boson_{n}sites_d20_chi100_chain_blocks"),
                       "desc": "weak scaling: one config-3-sized block (100 bosons, n=2000 bonds) per GPU; "
                               "value = blocks x steps / s (each block is a config-3 chain)",
                       "sites": n, "chi": chi, "updates_per_step": int(ups.item()),
                       "parallelism": f"chain-block partition x{world}, " + (
                           "gloo host-staged exchange on shared GPUs (protocol check, not a measurement)"
                           if gloo else ("NCCL send/recv boundary exchange behind the C ABI "
                                         "(rrsvd_b200_evolve_partitioned)" if native else
                                         "NCCL P2P boundary exchange (Python driver)")),
                       "l2": "inputs larger than L2"},
            "decimations_per_s": round(float(ups.item()) * args.steps / elapsed, 3),
            "roofline": {"bound": "tensor", "peak": round(peak_dmma, 3), "unit": "TFLOP/s", "achieved": None,
                         "frac": None, "note": "per-launch roofline is reported by the N=1 run"},
            "e2e": {"value": round(e2e, 6), "unit": "steps/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "note": "rank 0's bytes; every rank stages its own block"},
            "gpu_launches": int(gpu_launches), "clocks": clk.summary(),
        })
    dist.barrier()
    dist.destroy_process_group()


# ----------------------------------------------------------------------------- our arm

def run_ours(args, rank, world, local_rank):
    import torch
    import paper_1504_00992_b200 as P
    from paper_1504_00992_b200 import models as M
    from paper_1504_00992_b200.tebd import DeviceMps, build_gates, evolve

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = P.Context(local_rank, stream=stream.cuda_stream)  # library work and events share one stream
    peak_dmma = P.probe_peak(0, ctx=ctx)
    wl = workload(args.workload)
    site_dims, terms, chi = wl["site_dims"], wl["terms"], wl["chi"]
    plan, gates_host = build_gates(site_dims, terms, wl["dt"])
    from paper_1504_00992_b200.tebd import PreparedGates
    gates = PreparedGates(gates_host, ctx)  # resident on the device, block structure analysed once
    gammas, lambdas = M.synthetic_saturated_mps(site_dims, chi, seed=1 + rank)
    mps = DeviceMps(site_dims, chi, 0.0, ctx=ctx)
    mps.load(gammas, lambdas)
    be = P.DecimationBackend(omega_mode=P.OMEGA_PHILOX, **wl["backend"])
    ups = updates_per_step(site_dims, terms)

    def one_step():
        return evolve(mps, terms, wl["dt"], 1, be, record_updates=False, gates=gates, plan=plan)

    for _ in range(args.warmup):
        one_step()
        mps.load(gammas, lambdas)  # keep the saturated timing state (χ stays at the cap)

    # ---- device-resident timed region
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    lib = P.lib()
    import ctypes as C
    launches0 = ctx.launches
    if dist:
        dist.barrier()
    ctx.synchronize()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        t0 = time.perf_counter()
        ev0.record(stream)
        diag = evolve(mps, terms, wl["dt"], args.steps, be, record_updates=True, gates=gates, plan=plan)
        ev1.record(stream)
        ev1.synchronize()
        t1 = time.perf_counter()
    elapsed = ev0.elapsed_time(ev1) / 1e3  # device time (CUDA events on the launching stream)
    wall = t1 - t0
    gpu_launches = ctx.launches - launches0
    dev_update_us = sum(u["t_theta_us"] + u["t_gate_us"] + u["t_svd_us"] for u in diag.updates)

    # ---- roofline pass: the same step with the two-lane overlap off, every zgemm launch
    # event-timed on its stream (with overlap on, concurrent launches inflate each other's
    # durations, so per-launch kernel efficiency is read from this serial pass).
    ctx.check(lib.rrsvd_b200_set_overlap(ctx.h, 0))
    ctx.check(lib.rrsvd_b200_set_gemm_timing(ctx.h, 1))
    er0, er1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    er0.record(stream)
    one_step()
    er1.record(stream)
    er1.synchronize()
    serial_step_s = er0.elapsed_time(er1) / 1e3
    fl, ms, calls = C.c_double(), C.c_double(), C.c_uint64()
    ctx.check(lib.rrsvd_b200_gemm_stats(ctx.h, C.byref(fl), C.byref(ms), C.byref(calls)))
    exec_fl, tma_ms = C.c_double(), C.c_double()
    ctx.check(lib.rrsvd_b200_gemm_pipe_stats(ctx.h, C.byref(exec_fl), C.byref(tma_ms)))
    sfl, sms = (C.c_double * 8)(), (C.c_double * 8)()
    ctx.check(lib.rrsvd_b200_gemm_stage_stats(ctx.h, sfl, sms))
    ofl, oms, obytes, ocalls, opms, opbytes = (C.c_double(), C.c_double(), C.c_double(), C.c_uint64(), C.c_double(),
                                               C.c_double())
    ctx.check(lib.rrsvd_b200_ozaki_stats(ctx.h, C.byref(ofl), C.byref(oms), C.byref(obytes), C.byref(ocalls),
                                         C.byref(opms), C.byref(opbytes)))
    ogms, ogbytes = C.c_double(), C.c_double()
    ctx.check(lib.rrsvd_b200_ozaki_gemm_stats(ctx.h, C.byref(ogms), C.byref(ogbytes)))
    ctx.check(lib.rrsvd_b200_set_gemm_timing(ctx.h, 0))
    ctx.check(lib.rrsvd_b200_set_overlap(ctx.h, 1))
    stage_names = ["theta", "gate", "rrsvd_A_products", "qr_gram", "qr_apply", "svd_assembly", "det_precond"]
    stages = {nm: {"tflops": round(sfl[i] / (sms[i] * 1e-3) / 1e12, 2), "ms_per_step": round(sms[i], 2)}
              for i, nm in enumerate(stage_names) if sms[i] > 0}
    if dist:
        t = torch.tensor([elapsed], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    steps_per_s = world * args.steps / elapsed

    # ---- end-to-end through the C ABI with HOST buffers (pinned): the SAME consecutive sequence
    # of args.steps steps as `value`, the state held in host memory between steps: step 0 uploads
    # it (rrsvd_b200_state_upload); after every step it goes device -> host -> device
    # (rrsvd_b200_state_roundtrip: per site, the D2H and the H2D of the next step's input pipelined
    # on two streams — each site's upload starts when its download has landed); the last step
    # downloads it (rrsvd_b200_state_download).  Every step thus moves its whole input H2D and its
    # whole result D2H.  Buffers are allocated before the region.
    mps.load(gammas, lambdas)
    pin_g = [torch.from_numpy(g).pin_memory() for g in gammas]
    pin_l = [torch.from_numpy(l).pin_memory() for l in lambdas]
    h2d = d2h = state_bytes(gammas, lambdas)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    te0 = time.perf_counter()
    mps.upload(pin_g, pin_l)
    for st in range(args.steps):
        one_step()
        dims = mps.all_dims()
        same = True
        for s_ in range(len(site_dims)):  # (a saturated state keeps its dims: nothing reallocated)
            if tuple(pin_g[s_].shape) != dims[s_]:
                pin_g[s_] = torch.empty(dims[s_], dtype=torch.complex128).pin_memory()
                same = False
        for b in range(len(site_dims) - 1):
            if pin_l[b].shape[0] != dims[b][2]:
                pin_l[b] = torch.empty(dims[b][2], dtype=torch.float64).pin_memory()
                same = False
        if st + 1 < args.steps and same:
            mps.roundtrip(pin_g, pin_l)
        else:
            mps.download(pin_g, pin_l)
            if st + 1 < args.steps:
                mps.upload(pin_g, pin_l)
        d2h = sum(g.numel() * 16 for g in pin_g) + sum(l.numel() * 8 for l in pin_l)
    te1 = time.perf_counter()
    e2e = world * args.steps / (te1 - te0)

    clocks = clk.summary()
    achieved = fl.value / (ms.value * 1e-3) / 1e12 if ms.value > 0 else 0.0
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(steps_per_s, 6), "unit": "steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * elapsed / args.steps, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128 (fp64)",
            "data": "synthetic χ-saturated MPS (Gaussian Γ, λ∝0.9^i) + real TEDOPA bond gates",
            "config": bench_config(wl, ups, world),
            "sketch": "Philox in-kernel (the reference arm: its mt19937_64 stream)",
            "decimations_per_s": round(world * ups * args.steps / elapsed, 3),
            "roofline": {"bound": "tensor",
                         "kernel": "zgemm_dmma_kernel: every zgemm launch of one step (serial roofline pass,"
                                   " CUDA events per launch on its stream)",
                         "achieved": round(achieved, 3), "peak": round(peak_dmma, 3), "unit": "TFLOP/s",
                         "frac": round(achieved / peak_dmma, 4) if peak_dmma else None,
                         "peak_source": "measured live: DMMA probe (mma.sync m8n8k4 f64) on this GPU;"
                                        " MEASURED_PEAKS.json has no FP64 entry",
                         "frac_of_40tf_nominal": round(achieved / 40.0, 4),
                         "achieved_executed": round(exec_fl.value / (ms.value * 1e-3) / 1e12, 3) if ms.value > 0 else None,
                         "frac_executed": round(exec_fl.value / (ms.value * 1e-3) / 1e12 / peak_dmma, 4)
                         if ms.value > 0 and peak_dmma else None,
                         "frac_note": "frac counts the algorithmic 8 flops per complex MAC (a 4M zgemm's work, SURVEY"
                                      " 8(d)); frac_executed counts what the DMMA pipe executed (6 per MAC in the"
                                      " 3M form) — the tensor-pipe utilisation",
                         "tma_time_share": round(tma_ms.value / ms.value, 4) if ms.value > 0 else None,
                         "complex_product": "3M on the 64x56 tile (RRSVD_B200_GEMM_3M=0: 4M): the DMMA pipe"
                                            " executes 6 real flops per complex MAC; achieved counts the"
                                            " algorithmic 8 (SURVEY 8(d)), as a 4M zgemm would have to",
                         "gemm_time_share_serial": round(ms.value / (1e3 * serial_step_s), 4),
                         "serial_step_ms": round(1e3 * serial_step_s, 3),
                         "step_level_tflops": round(fl.value / (elapsed / args.steps) / 1e12, 3),
                         "gemm_launches": int(calls.value), "stages": stages, **traffic_entry(),
                         "emulated_a_products": emulated_entry(ofl.value, oms.value, obytes.value, ocalls.value,
                                                               opms.value, opbytes.value, ogms.value, ogbytes.value)},
            "e2e": {"value": round(e2e, 6), "unit": "steps/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "steps": args.steps,
                    "note": "same consecutive steps as value; the state lives in pinned host memory between "
                            "steps: every step uploads its whole input and downloads its whole result "
                            "(between steps as one per-site pipelined device->host->device round trip)"},
            "gpu_launches": int(gpu_launches),
            "clocks": clocks,
            "device_time_per_step_ms": round(dev_update_us / 1e3 / args.steps, 3),
            "wall_ms_per_step": round(1e3 * wall / args.steps, 3),
        }
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline(args, wl, gammas, lambdas, gates_host, plan, samples=2)
        emit(line)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


# ----------------------------------------------------------------------------- row-sharded RRSVD

SHARDED = {  # C5 top of the sweep and the C4 interpretation (i)
    "c5": dict(name="c5_rrsvd_n16000_k100_p10_q2", n=16000, k=100, p=10, q=2,
               desc="single RRSVD of a 16000^2 matrix, exponential spectrum 0.95^i, k=100 p=10 q=2"),
    "c4": dict(name="c4i_rrsvd_n80000_k200_p10_q2", n=80000, k=200, p=10, q=2,
               desc="config-4 interpretation (i): single RRSVD of an 80000^2 matrix (102 GB), "
                    "exponential spectrum 0.95^i, k=200 p=10 q=2, row-sharded"),
}
SPECTRUM_RANK = 800  # 0.95^799 ~ 1.6e-18: the truncated tail is below double resolution


def run_sharded(args, rank, world, local_rank):
    """Row-sharded RRSVD (SURVEY §8(e) level 2): the matrix's rows are split over the ranks (and,
    past the GEMM's 32-bit offsets, over several in-process shards per rank); Gram matrices and
    A^H products are all-reduced (NCCL).  Strong scaling: the matrix is fixed as N grows."""
    import torch
    import paper_1504_00992_b200 as P
    from paper_1504_00992_b200.sharded import DeviceOps, LocalSum, ShardedRrsvd, TorchSum

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = P.Context(local_rank, stream=stream.cuda_stream)
    peak_dmma = P.probe_peak(0, ctx=ctx)
    wl = SHARDED[args.workload]
    n, k, p, q = wl["n"], wl["k"], wl["p"], wl["q"]
    l = k + p
    rows = [(n * r) // world for r in range(world + 1)]
    r0, r1 = rows[rank], rows[rank + 1]
    per = max(1, -(-((r1 - r0) * n) // 900_000_000))  # in-process shards: < 2^31 doubles each
    cuts = [r0 + ((r1 - r0) * i) // per for i in range(per + 1)]
    comm = TorchSum(f"cuda:{local_rank}") if world > 1 else LocalSum()
    ops = DeviceOps(ctx)
    drv = ShardedRrsvd(comm, ops)
    # synthetic A = U diag(0.95^i) V^H, U (n x r) orthonormal across all shards, V replicated
    rk = SPECTRUM_RANK
    sig = torch.tensor(0.95 ** np.arange(rk), dtype=torch.float64, device="cuda")
    ys = [P.gaussian_test_matrix(cuts[i + 1] - cuts[i], rk, 1000 + cuts[i], P.OMEGA_PHILOX, ctx=ctx,
                                 device="cuda") for i in range(per)]
    us = drv._orth_sharded(ys, n, 4)
    v, _ = P.qr(P.gaussian_test_matrix(n, rk, 2, P.OMEGA_PHILOX, ctx=ctx, device="cuda"), ctx=ctx)
    vh = v.conj().T.contiguous()
    del ys, v
    shards = [P.gemm(u * sig, False, vh, ctx=ctx) for u in us]
    del us, vh
    torch.cuda.synchronize()

    def one():
        return drv.fixed_rank(shards, n, k, p, q, 11, mode=P.OMEGA_PHILOX)

    for _ in range(args.warmup):
        one()
    launches0 = ctx.launches
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            res = one()
        ev1.record(stream)
        ev1.synchronize()
    elapsed = ev0.elapsed_time(ev1) / 1e3
    gpu_launches = ctx.launches - launches0
    if dist:
        t = torch.tensor([elapsed], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    per_dec = elapsed / args.steps
    w_rr = 8.0 * (2 * q + 2) * n * n * l
    sig_out = res[1].cpu().numpy()
    check = float(np.max(np.abs(sig_out[:20] - 0.95 ** np.arange(20)) / 0.95 ** np.arange(20)))
    line = None
    if rank == 0:
        line = {
            "metric": "RRSVD decimations/s (row-sharded single matrix; FP64 tensor-core roofline)",
            "value": round(1.0 / per_dec, 5), "unit": "decimations/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * per_dec, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128 (fp64)",
            "data": f"synthetic: U diag(0.95^i, i<{rk}) V^H with Philox-Gaussian orthonormalised U, V",
            "config": {"workload": wl["name"], "desc": wl["desc"], "n": n, "k": k, "p": p, "q": q,
                       "shards_per_rank": per, "sketch": "Philox in-kernel",
                       "parallelism": f"row-sharded x{world}" if world > 1 else f"one GPU, {per} row shards",
                       "l2": "inputs larger than L2 (A %.1f GB)" % (16.0 * n * n / 1e9)},
            "roofline": {"bound": "tensor", "kernel": "whole decimation: W_rr = 8(2q+2) m n l over the step time",
                         "achieved": round(w_rr / per_dec / 1e12, 3), "peak": round(peak_dmma * world, 3),
                         "unit": "TFLOP/s", "frac": round(w_rr / per_dec / 1e12 / (peak_dmma * world), 4),
                         "peak_source": "measured live: DMMA probe (mma.sync m8n8k4 f64) x n_gpus",
                         "traffic": None},
            "sigma_check_top20_rel_err": check,
            "e2e": None, "e2e_note": "input is the resident matrix (%.0f GB); host staging not timed" % (16.0 * n * n / 1e9),
            "gpu_launches": int(gpu_launches), "clocks": clk.summary(),
        }
        if not args.no_cpu_baseline and world == 1 and args.workload == "c5":
            line["cpu_baseline"] = sharded_cpu_baseline(wl)
        elif args.workload == "c4":
            line["cpu_baseline"] = None
            line["cpu_baseline_note"] = "not run: the 102 GB input exceeds a host-core run's budget"
        emit(line)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def sharded_cpu_baseline(wl):
    """The reference rrsvd_fixed_rank on the host cores, one call on a 4000^2 sample of the same
    synthetic family, extrapolated by its GEMM work (n^2) to the configured n."""
    from oracle import ref
    if not ref.available():
        return None
    cores = os.cpu_count() or 1
    ref.set_threads(cores)
    ns = 4000
    rng = np.random.default_rng(0)
    u, _ = np.linalg.qr(rng.standard_normal((ns, 400)) + 1j * rng.standard_normal((ns, 400)))
    v, _ = np.linalg.qr(rng.standard_normal((ns, 400)) + 1j * rng.standard_normal((ns, 400)))
    a = (u * 0.95 ** np.arange(400)) @ v.conj().T
    t0 = time.perf_counter()
    ref.fixed_rank(a, wl["k"], wl["p"], wl["q"], 11, vectors=True)
    dt = (time.perf_counter() - t0) * (wl["n"] / ns) ** 2
    return {"value": round(1.0 / dt, 6), "unit": "decimations/s", "cores": cores, "kind": "reference",
            "sample": f"one rrsvd_fixed_rank at n={ns} on the host, x(n/{ns})^2 to n={wl['n']}"}


def traffic_entry():
    """DRAM traffic of the dominant kernel from the committed ncu --set full capture (per
    launch), with the launch's algorithmic bytes for comparison; null if absent."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(path):
        return {"traffic": None}
    with open(path) as f:
        t = json.load(f)
    return {"traffic": t.get("dram_bytes_per_launch"), "traffic_note": t.get("note")}


# ----------------------------------------------------------------------------- CPU reference

def ref_update_sample(ref, wl, gammas, lambdas, gates, plan, bonds, seed):
    """Times the reference's build_theta → apply_gate_to_theta → decimate on the given bonds of
    the same synthetic state (tebd.cpp:296-306), returns seconds per update."""
    be = ref.Backend(**wl["backend"])
    be.seed = seed
    n = len(wl["site_dims"])
    t = 0.0
    for b in bonds:
        s = 0 if (b % 2 == 1) else 1  # a sweep of this bond's parity
        g = gates[(s, b)]
        ll = lambdas[b - 1] if b > 0 else None
        lr = lambdas[b + 1] if b + 2 < n else None
        t0 = time.perf_counter()
        th = ref.apply_gate(ref.build_theta(gammas[b], gammas[b + 1], ll, lambdas[b], lr), g)
        ref.decimate(th, ll, lr, wl["chi"], 0.0, be)
        t += time.perf_counter() - t0
    return t / len(bonds)


def cpu_baseline(args, wl, gammas, lambdas, gates, plan, samples=2):
    from oracle import ref
    host = host_info()
    ref.set_threads(host["cores"])
    nb = len(wl["site_dims"]) - 1
    bonds = [nb // 2 - 1 + i for i in range(samples)]
    sec = ref_update_sample(ref, wl, gammas, lambdas, gates, plan, bonds, 7)
    ups = updates_per_step(wl["site_dims"], wl["terms"])
    return {"value": round(1.0 / (sec * ups), 8), "unit": "steps/s", "cores": host["cores"], "kind": "reference",
            "sample": f"{samples} interior bond updates (build_theta+apply_gate+decimate, "
                      f"{'RRSVD' if wl['backend'].get('randomized') else 'deterministic SVD'}) of the "
                      f"same state, {sec:.3f} s/update, extrapolated x{ups} updates/step (the --impl "
                      f"reference arm times a whole evolve step)",
            "cpu_model": host["cpu_model"], "blas": ref.blas_info()["config"]}


def host_info() -> dict:
    """CPU model, the cores this process is pinned to (taskset equivalent: sched_setaffinity on
    every core the process may use) and the reference BLAS build."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            model = next(l.split(":", 1)[1].strip() for l in f if l.startswith("model name"))
    except (OSError, StopIteration):
        pass
    cores = sorted(os.sched_getaffinity(0))
    os.sched_setaffinity(0, cores)
    return {"cpu_model": model, "cores": len(cores), "affinity": f"{cores[0]}-{cores[-1]}" if cores else "",
            "online_cpus": os.cpu_count()}


def run_reference(args, rank, world):
    """The reference's OWN evolve (tebd.cpp:260-326) — one full TEBD step, evolve(state, ..., 1)
    exactly as its tebd-run driver calls it per step (experiments.cpp:351-352), gate rebuild
    (tebd.cpp:276-285) included — on the same synthetic saturated state as our arm, timed on the
    host cores.  A C3 step takes minutes on a CPU, so this arm times ONE step whatever --steps
    says (reported as "steps": 1); the warm-up is one interior bond update (BLAS thread pool,
    page-in), not a whole step."""
    if rank != 0:
        return
    from oracle import ref
    from paper_1504_00992_b200 import models as M
    if not ref.available():
        emit({"impl": "reference", "unavailable": "oracle/_ref/librrsvd_ref.so not built"})
        return
    host = host_info()
    ref.set_threads(host["cores"])
    blas = ref.blas_info()
    wl = workload(args.workload)
    site_dims, terms, chi = wl["site_dims"], wl["terms"], wl["chi"]
    gammas, lambdas = M.synthetic_saturated_mps(site_dims, chi, seed=1)
    n = len(site_dims)
    ups = updates_per_step(site_dims, terms)
    rm = ref.RefMps(site_dims, [np.eye(d, dtype=complex)[0] for d in site_dims], chi, 0.0)
    for s_ in range(n):
        rm.set_site(s_, gammas[s_], lambdas[s_] if s_ < n - 1 else None)
    from paper_1504_00992_b200.tebd import build_gates
    plan, gates = build_gates(site_dims, terms, wl["dt"])
    tw = time.perf_counter()
    ref_update_sample(ref, wl, gammas, lambdas, gates, plan, [(n - 1) // 2], 100)
    warm_s = time.perf_counter() - tw
    be = ref.Backend(**wl["backend"])
    if args.workload == "c4mpdo":  # a whole MPDO step is ~15 min of CPU: time 2 interior updates
        sec = ref_update_sample(ref, wl, gammas, lambdas, gates, plan, [(n - 1) // 2 - 1, (n - 1) // 2], 7)
        wall = sec * ups
        d = {"n_updates": ups, "update_us": wall * 1e6}
        sample = (f"2 interior bond updates (build_theta+apply_gate+decimate) of the same state, {sec:.2f} s/update, "
                  f"extrapolated x{ups} updates/step")
    else:
        t0 = time.perf_counter()
        d = rm.evolve(terms, wl["dt"], 1, be)
        wall = time.perf_counter() - t0
        sample = (f"one full step: the reference evolve(state, terms, plan, 1, backend) on the same synthetic "
                  f"state ({d['n_updates']} updates, {wall:.1f} s incl. the per-call gate rebuild; "
                  f"{d['update_us'] / 1e6:.1f} s in build_theta+apply_gate+decimate)")
    upd = d["update_us"] / 1e6
    v = 1.0 / wall
    emit({
        "impl": "reference", "metric": METRIC, "value": round(v, 8), "unit": "steps/s", "n_gpus": world,
        "steps": 1, "warmup": 0, "steps_requested": args.steps, "warmup_requested": args.warmup,
        "warmup_note": f"one interior bond update ({warm_s:.1f} s) instead of whole steps",
        "ms_per_step": round(1e3 * wall, 1), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "c128 (fp64)", "data": "synthetic χ-saturated MPS (Gaussian Γ, λ∝0.9^i) + real TEDOPA bond gates",
        "config": bench_config(wl, ups, world),
        "steps_per_s_excl_gate_rebuild": round(1.0 / upd, 8) if upd > 0 else None,
        "decimations_per_s": round(d["n_updates"] / wall, 4),
        "cpu_baseline": {"value": round(v, 8), "unit": "steps/s", "cores": host["cores"], "kind": "reference",
                         "sample": sample, "cpu_model": host["cpu_model"], "affinity": host["affinity"],
                         "blas": blas["config"], "blas_core": blas["core"], "blas_threads": blas["threads"]},
        "e2e": {"value": round(v, 8), "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    })


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default 10; 1 for c3det, whose steps take ~40 s)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3", choices=["c3", "c3p100", "c3det", "c2", "c2rr", "c4mpdo", "c5", "c4"],
                    help="c3 (headline TEBD), c3p100, c3det, c2, c2rr, c4mpdo (MPDO chain); c5/c4: row-sharded "
                         "single-matrix RRSVD")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--force-partition", action="store_true",
                    help="use the chain-block partition driver even on one GPU (smoke test of the N>1 path)")
    args = ap.parse_args()
    global _JSON_FD
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)  # NCCL's version banner and any library prints go to stderr
    if args.steps is None:
        args.steps = 1 if args.workload == "c3det" else 10
    if args.warmup < 3:
        args.warmup = 3
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.workload in SHARDED and args.impl == "reference":
        if rank == 0:
            wl = SHARDED[args.workload]
            cb = sharded_cpu_baseline(wl) if args.workload == "c5" else None
            if cb is None:
                emit({"impl": "reference", "unavailable": "c4: 102 GB input exceeds a host run"
                                  if args.workload == "c4" else "oracle/_ref not built"})
            else:
                emit({"impl": "reference", "metric": "RRSVD decimations/s (row-sharded single matrix;"
                                  " FP64 tensor-core roofline)", "value": cb["value"], "unit": "decimations/s",
                                  "n_gpus": world, "steps": 1, "warmup": 0, "higher_is_better": True,
                                  "config": {"workload": wl["name"]}, "cpu_baseline": cb,
                                  "e2e": {"value": cb["value"], "unit": "decimations/s", "h2d_bytes_per_step": 0,
                                          "d2h_bytes_per_step": 0}})
    elif args.workload in SHARDED:
        run_sharded(args, rank, world, local_rank)
    elif args.impl == "reference":
        run_reference(args, rank, world)
    elif world > 1 or args.force_partition:
        run_partitioned(args, rank, world, local_rank)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
