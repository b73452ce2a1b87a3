"""The header-only C++ drop-in (include/rrsvd_b200/rrsvd.hpp): reference-style C++ test bodies
compile against it unchanged (CPU) and pass on the device (GPU)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1504_00992_b200", "lib")


def build(tmp_path) -> str:
    exe = str(tmp_path / "shim_test")
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{ROOT}/include", f"{ROOT}/tests/cpp/shim_test.cpp",
                    f"-L{LIBDIR}", "-lrrsvd_b200", f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_shim_compiles_and_links(tmp_path):
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
def test_shim_runs_reference_style_tests(tmp_path):
    out = subprocess.run([build(tmp_path)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "shim_test passed" in out.stdout
