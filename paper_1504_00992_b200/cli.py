"""Command line of the reference's experiment drivers on the B200 path:
the same subcommands, flags, CSV schemas and exit codes as proj/tools (main.cpp,
experiments.cpp) — `tebd-run` and `svd-bench` run their decimations through librrsvd_b200.

  python -m paper_1504_00992_b200.cli tebd-run --model ising --sites 8 --chi 16 --steps 20 \
      --backend rrsvd --out diag.csv --observables-out obs.csv --state-out state.rrmp
  python -m paper_1504_00992_b200.cli svd-bench --sizes 900,1600 --k 100 --p 100 --out bench.csv

Exit codes (experiments.hpp:16-19): 0 ok, 2 usage, 3 simulation abort (discarded-weight budget),
4 recurrence breakdown.  CSV numbers are written as std::to_chars(general, 17).
"""
from __future__ import annotations

import argparse
import sys
import time

import numpy as np

EXIT_OK, EXIT_USAGE, EXIT_ABORT, EXIT_BREAKDOWN = 0, 2, 3, 4


class CsvWriter:
    """tools/src/csv.hpp: fixed header, one row per end_row, general/17 doubles."""

    def __init__(self, path: str, header: list[str]):
        self.f = open(path, "w")
        self.n = len(header)
        self.f.write(",".join(header) + "\n")

    def row(self, *fields):
        if len(fields) != self.n:
            raise RuntimeError("CSV row has wrong number of fields")
        out = []
        for v in fields:
            if isinstance(v, float):
                out.append(format(v, ".17g"))
            else:
                out.append(str(v))
        self.f.write(",".join(out) + "\n")

    def close(self):
        self.f.close()


def mix_seed(base: int, salt: int) -> int:
    """experiments.cpp:38-40."""
    return (base + 0x9e3779b97f4a7c15 * (salt + 1)) % (1 << 64)


def parse_spectrum(text: str, n: int) -> np.ndarray:
    """experiments.cpp parse_spectrum + matgen.cpp spectrum_* (normalised exponential)."""
    from .io import read_value_lines
    if text == "power":
        return 1.0 / np.arange(1, n + 1, dtype=float)
    if text.startswith("exp:"):
        ratio = float(text[4:])
        if not 0.0 < ratio < 1.0:
            raise ValueError("spectrum_exponential: ratio must be in (0, 1)")
        s = ratio ** np.arange(n, dtype=float)
        return s / np.sqrt(np.sum(s * s))
    if text.startswith("file:"):
        v = read_value_lines(text[5:])
        if len(v) < n:
            raise ValueError("spectrum file has fewer values than requested")
        return np.asarray(v[:n])
    raise ValueError(f"unknown spectrum spec: {text} (expected exp:RATIO, power, or file:PATH)")


# ------------------------------------------------------------------------------- tebd-run

def run_tebd(a) -> int:
    """experiments.cpp run_tebd: product-state quench, one evolve(…, 1) per step, per-update
    diagnostics CSV, optional observables CSV and final RRMP state."""
    from . import api, models as M
    from .io import read_coefficients_file, write_rrmp
    from .tebd import DeviceMps, PreparedGates, build_gates, evolve

    if a.model in ("ising", "heisenberg"):
        if a.sites < 2:
            print("tebd-run: need at least two sites", file=sys.stderr)
            return EXIT_USAGE
        site_dims = [2] * a.sites
        terms = M.ising_terms(a.sites, a.coupling, a.field) if a.model == "ising" else \
            M.heisenberg_terms(a.sites, a.coupling)
        observables = [M.SZ] * a.sites
        locals_ = [np.array([1, 0], complex) if (a.model == "ising" or s % 2 == 0) else np.array([0, 1], complex)
                   for s in range(a.sites)]
    elif a.model == "tedopa-chain":
        if not a.coeffs:
            print("tebd-run: --coeffs required for tedopa-chain", file=sys.stderr)
            return EXIT_USAGE
        try:
            t0, om, hop = read_coefficients_file(a.coeffs)
        except Exception as e:  # noqa: BLE001 — the reference maps every reader error to usage
            print(f"tebd-run: {e}", file=sys.stderr)
            return EXIT_USAGE
        if a.sites >= 2 and a.sites - 1 < len(om):
            om, hop = om[:a.sites - 1], hop[:a.sites - 2]
        h_sys = np.array([[0.5 * a.sys_epsilon, 0.5 * a.sys_delta], [0.5 * a.sys_delta, -0.5 * a.sys_epsilon]],
                         complex)
        site_dims, terms = M.build_chain_terms(t0, om, hop, a.boson_dim, h_sys, M.SZ)
        num = np.diag(np.arange(a.boson_dim, dtype=float)).astype(complex)
        observables = [M.SZ] + [num] * (len(site_dims) - 1)
        vac = np.zeros(a.boson_dim, complex)
        vac[0] = 1.0
        locals_ = [np.array([1, 0], complex)] + [vac] * (len(site_dims) - 1)
    else:
        print(f"tebd-run: unknown model {a.model}", file=sys.stderr)
        return EXIT_USAGE
    if a.backend == "rrsvd":
        be = api.DecimationBackend(randomized=True, target_rank=a.chi, oversampling=a.oversampling,
                                   power_iterations=a.q, det_crossover=a.crossover, seed=a.seed,
                                   accuracy_check=a.epsilon > 0.0, epsilon=a.epsilon if a.epsilon > 0 else 1e-3)
    elif a.backend == "det":
        be = api.DecimationBackend()  # the reference leaves the deterministic backend's seed at 0
    else:
        print(f"tebd-run: unknown backend {a.backend}", file=sys.stderr)
        return EXIT_USAGE

    n = len(site_dims)
    mps = DeviceMps(site_dims, a.chi, a.trunc_tolerance)
    for s, v in enumerate(locals_):
        if not np.allclose(v, np.eye(site_dims[s])[0]):
            mps.set_site(s, v.reshape(1, -1, 1), np.ones(1) if s < n - 1 else None)
    tmap = {b: t for b, t in enumerate(terms)}
    plan, gh = build_gates(site_dims, tmap, a.dt)
    gates = PreparedGates(gh, mps.ctx)
    diag_csv = CsvWriter(a.out, ["step", "bond", "chi", "discarded_weight", "t_theta_us", "t_gate_us",
                                 "t_svd_us", "backend"])
    obs_csv = CsvWriter(a.observables_out, ["step", "site", "value_re", "value_im"]) if a.observables_out else None

    def emit(step):
        if obs_csv:
            for s in range(n):
                v = mps.expectation_local(s, observables[s])
                obs_csv.row(step, s, float(v.real), float(v.imag))

    emit(0)
    aborted, abort_step, cumulative = False, 0, 1.0
    step = 0
    while step < a.steps and not aborted:
        d = evolve(mps, tmap, a.dt, 1, be, abort_discarded_threshold=a.abort_threshold, gates=gates, plan=plan)
        for r in d.updates:
            diag_csv.row(step, r["bond"], r["chi"], float(r["discarded_weight"]), float(r["t_theta_us"]),
                         float(r["t_gate_us"]), float(r["t_svd_us"]), r["backend"])
        cumulative *= d.kept_fraction
        if d.aborted or 1.0 - cumulative > a.abort_threshold:
            aborted, abort_step = True, step
        emit(step + 1)
        step += 1
    diag_csv.close()
    if obs_csv:
        obs_csv.close()
    if a.state_out:
        write_rrmp(a.state_out, mps)
    if aborted:
        print(f"tebd-run: discarded-weight budget exceeded at step {abort_step}", file=sys.stderr)
        return EXIT_ABORT
    return EXIT_OK


# ------------------------------------------------------------------------------- svd-bench

def structured_matrix(sigma, m: int, u_seed: int, v_seed: int, ctx):
    """matgen.cpp:27-35 on the device: U (m x n), V (n x n) orthonormalised Gaussians (reference
    Ω stream), A = U diag(σ) V^H.  (The reference's Householder Q and this CholeskyQR Q span the
    same spaces; the instance matrices therefore differ by column phases, the spectrum is exact.)"""
    import torch

    from . import api
    n = len(sigma)
    u, _ = api.qr(api.gaussian_test_matrix(m, n, u_seed, ctx=ctx, device="cuda"), ctx=ctx)
    v, _ = api.qr(api.gaussian_test_matrix(n, n, v_seed, ctx=ctx, device="cuda"), ctx=ctx)
    us = u * torch.from_numpy(np.asarray(sigma)).cuda()
    return api.gemm(us, False, v.conj().T.contiguous(), ctx=ctx)


def run_svd_bench(a) -> int:
    """experiments.cpp run_svd_bench: deterministic vs randomized timings per size, median
    speedup summary rows.  Wall times include the device synchronisation of every call."""
    import torch

    from . import api
    if not a.out:
        print("svd-bench: --out required", file=sys.stderr)
        return EXIT_USAGE
    sizes = [(a.rows, a.cols)] if a.rows and a.cols else [(s, s) for s in a.sizes]
    if not sizes or a.trials < 1:
        print("svd-bench: need sizes and at least one trial", file=sys.stderr)
        return EXIT_USAGE
    for rows, cols in sizes:
        if cols < a.k + a.p or rows < cols:
            print("svd-bench: size too small for k + p", file=sys.stderr)
            return EXIT_USAGE
    ctx = api.default_context()
    csv = CsvWriter(a.out, ["record", "experiment", "rows", "cols", "k", "p", "q", "trial", "seed", "threads",
                            "algo", "wall_seconds", "max_abs_sv_error", "residual_fro", "speedup"])
    for rows, cols in sizes:
        try:
            sigma = parse_spectrum(a.spectrum, cols)
            m = structured_matrix(sigma, rows, mix_seed(a.seed, rows), mix_seed(a.seed, rows + 1), ctx)
        except torch.cuda.OutOfMemoryError:
            csv.row("skipped", "svd-bench", rows, cols, a.k, a.p, 0, 0, a.seed, a.threads, "alloc-failure",
                    0.0, 0.0, 0.0, 0.0)
            continue
        a_norm = api.frobenius_norm(m, ctx=ctx)
        det_walls = []
        for trial in range(a.trials):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _, s, _ = api.svd_full(m, ctx=ctx)
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
            det_walls.append(wall)
            s = s.cpu().numpy()
            err = float(np.max(np.abs(s[:a.k] - sigma[:a.k])))
            res = float(np.sqrt(np.sum(s[a.k:] ** 2)))
            csv.row("trial", "svd-bench", rows, cols, a.k, a.p, 0, trial, a.seed, a.threads, "det", wall,
                    err, res, 0.0)
        for q in a.qs:
            rr_walls = []
            for trial in range(a.trials):
                seed = mix_seed(a.seed, 1000 + 7 * trial + q)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                rr = api.rrsvd_fixed_rank(m, a.k, a.p, q, seed, vectors=True, ctx=ctx)
                torch.cuda.synchronize()
                wall = time.perf_counter() - t0
                rr_walls.append(wall)
                s = rr.sigma.cpu().numpy()
                err = float(np.max(np.abs(s - sigma[:a.k])))
                res = float(np.sqrt(rr.discarded_weight) * a_norm)
                csv.row("trial", "svd-bench", rows, cols, a.k, a.p, q, trial, seed, a.threads, "rrsvd", wall,
                        err, res, 0.0)
            speedup = float(np.median(det_walls) / np.median(rr_walls))
            csv.row("summary", "svd-bench", rows, cols, a.k, a.p, q, 0, a.seed, a.threads, "median_speedup",
                    float(np.median(rr_walls)), 0.0, 0.0, speedup)
        del m
    csv.close()
    return EXIT_OK


# ------------------------------------------------------------------------------- main

def _ints(text: str) -> list[int]:
    return [int(x) for x in text.split(",") if x]


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="rrsvd-b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    t = sub.add_parser("tebd-run", help="Time-evolve a chain and profile updates")
    t.add_argument("--model", default="ising")
    t.add_argument("--coeffs", default="")
    t.add_argument("--sites", type=int, default=6)
    t.add_argument("--chi", type=int, default=32)
    t.add_argument("--dt", type=float, default=1e-3)
    t.add_argument("--steps", type=int, default=100)
    t.add_argument("--backend", default="det")
    t.add_argument("--epsilon", type=float, default=0.0)
    t.add_argument("--q", type=int, default=2)
    t.add_argument("--oversampling", type=int, default=0)
    t.add_argument("--crossover", type=int, default=256)
    t.add_argument("--coupling", type=float, default=1.0)
    t.add_argument("--field", type=float, default=1.0)
    t.add_argument("--trunc-tolerance", dest="trunc_tolerance", type=float, default=0.0)
    t.add_argument("--abort-threshold", dest="abort_threshold", type=float, default=1.0)
    t.add_argument("--boson-dim", dest="boson_dim", type=int, default=4)
    t.add_argument("--sys-epsilon", dest="sys_epsilon", type=float, default=1.0)
    t.add_argument("--sys-delta", dest="sys_delta", type=float, default=1.0)
    t.add_argument("--seed", type=int, default=1)
    t.add_argument("--threads", type=int, default=0)
    t.add_argument("--out", required=True)
    t.add_argument("--observables-out", dest="observables_out", default="")
    t.add_argument("--state-out", dest="state_out", default="")
    s = sub.add_parser("svd-bench", help="Deterministic vs randomized SVD timings")
    s.add_argument("--sizes", type=_ints, default=[900, 1600, 2500, 3600, 4900])
    s.add_argument("--rows", type=int, default=0)
    s.add_argument("--cols", type=int, default=0)
    s.add_argument("--k", type=int, default=100)
    s.add_argument("--p", type=int, default=100)
    s.add_argument("--qs", type=_ints, default=[2])
    s.add_argument("--trials", type=int, default=5)
    s.add_argument("--spectrum", default="exp:0.95")
    s.add_argument("--seed", type=int, default=1)
    s.add_argument("--threads", type=int, default=0)
    s.add_argument("--out", required=True)
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:  # argparse usage errors exit 2, like CLI11
        return int(e.code or 0)
    if args.cmd == "tebd-run":
        return run_tebd(args)
    return run_svd_bench(args)


if __name__ == "__main__":
    sys.exit(main())
