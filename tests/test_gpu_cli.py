"""The CLI's tebd-run against the reference's own run_tebd
(experiments.cpp:241-372, compiled into oracle/_ref): same CSV schemas, rows, χ profile,
discarded weights, observables, final state λ (RRMP v1) and exit codes."""
import csv

import numpy as np
import pytest

from paper_1504_00992_b200 import io as fio
from paper_1504_00992_b200 import models as M
from paper_1504_00992_b200.cli import EXIT_ABORT, main

pytestmark = pytest.mark.gpu


def rows(path):
    with open(path) as f:
        r = list(csv.reader(f))
    return r[0], r[1:]


def compare_runs(tmp_path, ref, args: dict, expect_rc=0):
    mine = {k: str(tmp_path / f"m_{k}") for k in ("out", "obs", "state")}
    theirs = {k: str(tmp_path / f"r_{k}") for k in ("out", "obs", "state")}
    argv = ["tebd-run"]
    for k, v in args.items():
        argv += ["--" + k.replace("_", "-"), str(v)]
    rc = main(argv + ["--out", mine["out"], "--observables-out", mine["obs"], "--state-out", mine["state"]])
    rc_ref = ref.run_tebd(theirs["out"], observables_out=theirs["obs"], state_out=theirs["state"], **args)
    assert rc == rc_ref == expect_rc
    h1, d1 = rows(mine["out"])
    h2, d2 = rows(theirs["out"])
    assert h1 == h2 == ["step", "bond", "chi", "discarded_weight", "t_theta_us", "t_gate_us", "t_svd_us", "backend"]
    assert len(d1) == len(d2)
    for a, b in zip(d1, d2):
        assert a[:3] == b[:3] and a[7] == b[7]                  # step, bond, chi, backend
        assert abs(float(a[3]) - float(b[3])) < 1e-10            # discarded weight
    h1, o1 = rows(mine["obs"])
    h2, o2 = rows(theirs["obs"])
    assert h1 == h2 == ["step", "site", "value_re", "value_im"] and len(o1) == len(o2)
    for a, b in zip(o1, o2):
        assert a[:2] == b[:2]
        assert abs(float(a[2]) - float(b[2])) < 1e-8 and abs(float(a[3]) - float(b[3])) < 1e-8
    _, _, lm = fio.read_rrmp_arrays(mine["state"])
    _, _, lr = fio.read_rrmp_arrays(theirs["state"])
    assert [len(x) for x in lm] == [len(x) for x in lr]
    for x, y in zip(lm, lr):
        assert np.max(np.abs(x - y)) < 1e-8


def test_tebd_run_ising_rrsvd(tmp_path, ref):
    compare_runs(tmp_path, ref, dict(model="ising", sites=8, chi=8, dt=0.05, steps=8, backend="rrsvd",
                                     oversampling=4, crossover=0, field=0.7, seed=3))


def test_tebd_run_heisenberg_det(tmp_path, ref):
    compare_runs(tmp_path, ref, dict(model="heisenberg", sites=6, chi=8, dt=0.05, steps=6, backend="det"))


def test_tebd_run_tedopa_chain(tmp_path, ref):
    t0, om, hop = M.ohmic_chain(8)
    cf = str(tmp_path / "coeffs.txt")
    ref.write_coefficients(cf, t0, om, hop)
    compare_runs(tmp_path, ref, dict(model="tedopa-chain", coeffs=cf, sites=6, chi=12, dt=0.05, steps=4,
                                     boson_dim=4, backend="det"))


def test_tebd_run_abort_exit_code(tmp_path, ref):
    compare_runs(tmp_path, ref, dict(model="ising", sites=8, chi=2, dt=0.1, steps=6, backend="det",
                                     abort_threshold=1e-6), expect_rc=EXIT_ABORT)


def test_svd_bench_schema(tmp_path):
    out = str(tmp_path / "b.csv")
    assert main(["svd-bench", "--sizes", "300,400", "--k", "20", "--p", "20", "--qs", "1,2", "--trials", "2",
                 "--out", out]) == 0
    h, d = rows(out)
    assert h == ["record", "experiment", "rows", "cols", "k", "p", "q", "trial", "seed", "threads", "algo",
                 "wall_seconds", "max_abs_sv_error", "residual_fro", "speedup"]
    # per size: trials det rows + per q (trials rrsvd rows + 1 summary)
    assert len(d) == 2 * (2 + 2 * (2 + 1))
    for r in d:  # max |σ_i − σ_i^exact|, i < k: roundoff for det, approximation error for rrsvd
        if r[10] == "det":
            assert float(r[12]) < 1e-12
        elif r[10] == "rrsvd":
            assert float(r[12]) < 5e-2
