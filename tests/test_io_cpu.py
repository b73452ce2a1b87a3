"""File formats are byte-compatible with the reference's writers, and the
CLI (row 4) validates its arguments with the reference's exit codes (no GPU needed)."""
import os

import numpy as np
import pytest

from paper_1504_00992_b200 import io as fio
from paper_1504_00992_b200.cli import EXIT_USAGE, main
from tests.conftest import cplx_randn


def test_rrsm_bytes_match_reference(ref, tmp_path):
    a = cplx_randn(np.random.default_rng(1), 7, 5)
    ours, theirs = str(tmp_path / "a.rrsm"), str(tmp_path / "b.rrsm")
    fio.write_rrsm(ours, a)
    ref.write_rrsm(theirs, a)
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    assert np.array_equal(fio.read_rrsm(theirs), a)
    assert np.array_equal(ref.read_rrsm(ours), a)


def test_rrsm_reader_rejects_bad_files(tmp_path):
    p = str(tmp_path / "x.rrsm")
    fio.write_rrsm(p, np.ones((3, 3), complex))
    raw = open(p, "rb").read()
    for bad in (b"XXSM" + raw[4:], raw[:20], raw[:-16]):
        open(p, "wb").write(bad)
        with pytest.raises(fio.FormatError):
            fio.read_rrsm(p)
    a = np.ones((2, 2), complex)
    a[1, 1] = np.nan
    fio.write_rrsm(p, a)
    with pytest.raises(fio.FormatError):
        fio.read_rrsm(p)


def test_value_lines_and_coefficients_bytes_match_reference(ref, tmp_path):
    v = np.array([1.0, 0.1, 1e-5, 1.0 / 3.0, 2.0 ** -40, 123456.789])
    fio.write_value_lines(str(tmp_path / "o"), v)
    ref.write_value_lines(str(tmp_path / "r"), v)
    assert open(tmp_path / "o").read() == open(tmp_path / "r").read()
    assert fio.read_value_lines(str(tmp_path / "r")) == list(v)
    from paper_1504_00992_b200 import models as M
    t0, om, hop = M.ohmic_chain(12)
    fio.write_coefficients_file(str(tmp_path / "co"), t0, om, hop)
    ref.write_coefficients(str(tmp_path / "cr"), t0, om, hop)
    assert open(tmp_path / "co").read() == open(tmp_path / "cr").read()
    t0b, omb, hopb = fio.read_coefficients_file(str(tmp_path / "cr"))
    assert t0b == t0 and np.array_equal(omb, om) and np.array_equal(hopb, hop)


def test_rrmp_round_trip_of_reference_state(ref, tmp_path):
    """The reference's tebd-run writes RRMP v1 (experiments.cpp:400-425); we parse it and write
    the identical bytes back."""
    theirs = str(tmp_path / "ref.rrmp")
    rc = ref.run_tebd(str(tmp_path / "d.csv"), model="heisenberg", sites=6, chi=8, dt=0.05, steps=5,
                      state_out=theirs)
    assert rc == 0
    dims, g, lam = fio.read_rrmp_arrays(theirs)
    assert dims == [2] * 6 and len(g) == 6 and len(lam) == 5
    assert all(abs(np.sum(l_ ** 2) - 1.0) < 1e-12 for l_ in lam)
    ours = str(tmp_path / "ours.rrmp")
    fio.write_rrmp_arrays(ours, g, lam)
    assert open(ours, "rb").read() == open(theirs, "rb").read()


def test_cli_usage_exit_codes(tmp_path):
    out = str(tmp_path / "d.csv")
    assert main(["tebd-run", "--model", "nope", "--out", out]) == EXIT_USAGE
    assert main(["tebd-run", "--model", "tedopa-chain", "--out", out]) == EXIT_USAGE
    assert main(["tebd-run", "--model", "ising", "--sites", "1", "--out", out]) == EXIT_USAGE
    assert main(["tebd-run", "--model", "ising"]) == EXIT_USAGE  # --out required
    assert main(["svd-bench", "--sizes", "50", "--k", "40", "--p", "20", "--out", out]) == EXIT_USAGE
    assert not os.path.exists(str(tmp_path / "never"))
