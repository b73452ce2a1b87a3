"""The reference's OWN test programs — its acceptance suite (proj/tests/acceptance.cpp) and its
doctest unit suites for the hot path (test_linalg, test_randomized, test_mps, test_tebd) plus
test_matgen (whose Haar generators call the drop-in's qr / gemm) — compiled unmodified against
the drop-in (tests/cpp/Makefile; symbol provenance checked in tests/test_refsuite_cpu.py) and run
on the B200.  Every hot-path call lands in librrsvd_b200.so."""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "build", "refsuite")


def _run(prog, *args, timeout=1200):
    exe = os.path.join(OUT, prog)
    if not os.path.exists(exe):
        pytest.skip(f"{prog} not built (make -C tests/cpp, needs /root/reference)")
    res = subprocess.run([exe, *args], capture_output=True, text=True, timeout=timeout)
    print(res.stdout[-4000:])
    return res


@pytest.mark.parametrize("suite", ["test_linalg", "test_randomized", "test_mps", "test_tebd", "test_matgen"])
def test_reference_unit_suite(suite):
    res = _run(suite)
    assert res.returncode == 0, res.stdout[-6000:] + res.stderr[-2000:]
    assert re.search(r"failed: 0 ", res.stdout)


# criteria whose statement is numerical (accuracy, parity, certificates); 8 and 9 compare CPU
# wall-clock shapes (RRSVD vs zgesdd speed-up growing with n; decimate share of a CPU update) and
# are run and reported by test_acceptance_timing_criteria
NUMERIC = [1, 2, 3, 4, 5, 6, 7, 10]


@pytest.mark.parametrize("criterion", NUMERIC)
def test_reference_acceptance_criterion(criterion):
    res = _run("acceptance", "--only", str(criterion), timeout=2400)
    line = next((l for l in res.stdout.splitlines() if f"criterion {criterion}:" in l), "")
    assert res.returncode == 0 and line.startswith("PASS"), res.stdout[-4000:] + res.stderr[-2000:]
