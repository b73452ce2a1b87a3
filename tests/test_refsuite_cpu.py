"""The reference's own test programs linked against the drop-in (tests/cpp/Makefile): build them
(here, where /root/reference exists) and prove from the link maps that EVERY function the drop-in
defines resolved to the drop-in's strong copy (shim_strong.o), not to the reference core's
weakened objects — i.e. every hot-path call of those programs goes to librrsvd_b200.so.
(The programs themselves run on the B200: tests/test_refsuite_gpu.py.)"""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "build", "refsuite")
PROGRAMS = ["acceptance", "test_linalg", "test_randomized", "test_mps", "test_tebd", "test_matgen"]


@pytest.fixture(scope="module")
def built():
    if os.path.isdir("/root/reference/proj/tests"):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "tests", "cpp")], check=True,
                       capture_output=True)
    missing = [p for p in PROGRAMS if not os.path.exists(os.path.join(OUT, p))]
    if missing:
        pytest.skip(f"reference test programs not built (no /root/reference here): {missing}")
    return OUT


def _sections(mapfile):
    """(start, size, object) of every input section in the link map."""
    out = []
    pat = re.compile(r"^\s+(0x[0-9a-f]+)\s+(0x[0-9a-f]+)\s+(\S+\.o)\s*$")
    pat1 = re.compile(r"^\s*\.\S+\s+(0x[0-9a-f]+)\s+(0x[0-9a-f]+)\s+(\S+\.o)\s*$")
    with open(mapfile) as f:
        for line in f:
            m = pat.match(line) or pat1.match(line)
            if m:
                out.append((int(m.group(1), 16), int(m.group(2), 16), m.group(3)))
    return out


def _nm(path, defined_only=True):
    args = ["nm"] + (["--defined-only"] if defined_only else []) + [path]
    res = subprocess.run(args, check=True, capture_output=True, text=True).stdout
    syms = {}
    for line in res.splitlines():
        parts = line.split()
        if len(parts) == 3:
            syms.setdefault(parts[2], (parts[1], int(parts[0], 16)))
    return syms


def test_dropin_symbols_resolve_to_the_shim(built):
    shim = _nm(os.path.join(built, "shim_strong.o"))
    ours = sorted(s for s, (t, _) in shim.items() if t == "T")
    assert len(ours) >= 30
    ref_weak = set()
    for o in os.listdir(os.path.join(built, "ref")):
        ref_weak |= {s for s, (t, _) in _nm(os.path.join(built, "ref", o)).items() if t == "W"}
    overridden = [s for s in ours if s in ref_weak]
    # the reference core defines (weakly, after objcopy) the hot path the drop-in replaces
    for must in ("_ZN5rrsvd2qrERKNS_11DenseMatrixE", "_ZN5rrsvd4gemmERKNS_11DenseMatrixEbS2_b"):
        assert must in overridden
    for prog in PROGRAMS:
        exe = os.path.join(built, prog)
        secs = _sections(exe + ".map")
        syms = _nm(exe)
        for s in ours:
            if s not in syms:
                continue  # not linked into this program
            addr = syms[s][1]
            owner = [o for (a, n, o) in secs if a <= addr < a + max(n, 1)]
            assert owner and owner[0].endswith("shim_strong.o"), (prog, s, owner)
        ldd = subprocess.run(["ldd", exe], capture_output=True, text=True).stdout
        assert "librrsvd_b200.so" in ldd, prog


def test_reference_sources_are_unmodified_inputs(built):
    """The test programs are compiled from /root/reference in place (never copied into the repo)."""
    here = subprocess.run(["git", "-C", ROOT, "ls-files"], capture_output=True, text=True).stdout.split()
    assert not any(os.path.basename(p) in {"acceptance.cpp", "test_linalg.cpp", "test_tebd.cpp"} for p in here)
