"""File formats of the reference, byte-compatible.

* RRSM v1 — one complex128 matrix (proj/core/src/matrix_io.cpp:36-73): "RRSM", uint32 version 1,
  uint8 dtype 0 (complex double), uint64 rows, uint64 cols, then the row-major interleaved payload;
  little-endian, no padding (25-byte header).  Readers reject bad magic/version/dtype, truncation
  and non-finite entries, as the reference does.
* value lines — one double per line formatted "%.17g" (matrix_io.cpp:76-103, std::to_chars
  general/17), blank lines skipped.
* RRMP v1 — an MPS state (proj/tools/src/experiments.cpp:400-459): "RRMP", uint32 version 1,
  uint64 n_sites; per site uint64 (dim_left, dim_phys, dim_right) + the Γ payload (α, i, β)
  row-major complex128; per bond uint64 χ + χ doubles (λ).
* chain coefficients — text "n ω_n t_n" per line, t_0 then the hoppings
  (proj/core/src/chainmap.cpp:270-301).

`read_rrmp`/`write_rrmp` exchange device-resident states (tebd.DeviceMps) through the C ABI;
`*_arrays` variants work on host lists of Γ and λ.
"""
from __future__ import annotations

import struct

import numpy as np

from ._lib import ContractViolation

_RRSM = b"RRSM"
_RRMP = b"RRMP"


class FormatError(RuntimeError):
    """io_error / std::runtime_error of the reference readers."""


# ------------------------------------------------------------------------------- RRSM v1

def write_rrsm(path: str, a) -> None:
    a = np.ascontiguousarray(np.asarray(a), dtype=np.complex128)
    if a.ndim != 2:
        raise ContractViolation("write_rrsm: a matrix is required")
    with open(path, "wb") as f:
        f.write(_RRSM + struct.pack("<IBQQ", 1, 0, a.shape[0], a.shape[1]))
        f.write(a.astype("<c16", copy=False).tobytes())


def read_rrsm(path: str) -> np.ndarray:
    with open(path, "rb") as f:
        head = f.read(25)
        if len(head) < 25:
            raise FormatError(f"truncated header: {path}")
        if head[:4] != _RRSM:
            raise FormatError(f"bad magic: {path}")
        version, dtype, rows, cols = struct.unpack("<IBQQ", head[4:])
        if version != 1:
            raise FormatError(f"unsupported version: {path}")
        if dtype != 0:
            raise FormatError(f"unsupported dtype: {path}")
        payload = f.read(rows * cols * 16)
    if len(payload) < rows * cols * 16:
        raise FormatError(f"truncated payload: {path}")
    a = np.frombuffer(payload, dtype="<c16").astype(np.complex128).reshape(rows, cols)
    if not np.all(np.isfinite(a)):
        raise FormatError(f"non-finite entries: {path}")
    return a


# ------------------------------------------------------------------------------- value lines

def format_double(v: float) -> str:
    """std::to_chars(..., std::chars_format::general, 17)."""
    return format(float(v), ".17g")


def write_value_lines(path: str, values) -> None:
    with open(path, "w") as f:
        for v in values:
            f.write(format_double(v) + "\n")


def read_value_lines(path: str) -> list[float]:
    out = []
    with open(path) as f:
        for line in f:
            line = line.strip()
            if line:
                try:
                    out.append(float(line))
                except ValueError:
                    raise FormatError(f"bad value line: {line}") from None
    return out


# ------------------------------------------------------------------------------- RRMP v1

def write_rrmp_arrays(path: str, gammas, lambdas) -> None:
    n = len(gammas)
    with open(path, "wb") as f:
        f.write(_RRMP + struct.pack("<IQ", 1, n))
        for g in gammas:
            g = np.ascontiguousarray(g, dtype=np.complex128)
            f.write(struct.pack("<QQQ", *g.shape))
            f.write(g.astype("<c16", copy=False).tobytes())
        for b in range(n - 1):
            lam = np.ascontiguousarray(lambdas[b], dtype=np.float64)
            f.write(struct.pack("<Q", lam.size))
            f.write(lam.astype("<f8", copy=False).tobytes())


def read_rrmp_arrays(path: str):
    """-> (site_dims, gammas (χ_l, d, χ_r), lambdas)."""
    with open(path, "rb") as f:
        data = f.read()
    if len(data) < 16 or data[:4] != _RRMP or struct.unpack_from("<I", data, 4)[0] != 1:
        raise FormatError(f"bad state file: {path}")
    n = struct.unpack_from("<Q", data, 8)[0]
    off = 16
    gammas, dims, lambdas = [], [], []
    try:
        for _ in range(n):
            dl, d, dr = struct.unpack_from("<QQQ", data, off)
            off += 24
            cnt = dl * d * dr
            if off + 16 * cnt > len(data):
                raise FormatError(f"truncated state file: {path}")
            gammas.append(np.frombuffer(data, "<c16", cnt, off).astype(np.complex128).reshape(dl, d, dr))
            dims.append(int(d))
            off += 16 * cnt
        for _ in range(max(n - 1, 0)):
            (chi,) = struct.unpack_from("<Q", data, off)
            off += 8
            if off + 8 * chi > len(data):
                raise FormatError(f"truncated state file: {path}")
            lambdas.append(np.frombuffer(data, "<f8", chi, off).astype(np.float64))
            off += 8 * chi
    except struct.error:
        raise FormatError(f"truncated state file: {path}") from None
    return dims, gammas, lambdas


def write_rrmp(path: str, mps) -> None:
    """Download a tebd.DeviceMps and write it as RRMP v1."""
    n = mps.n_sites
    write_rrmp_arrays(path, [mps.gamma(s) for s in range(n)], [mps.lam(b) for b in range(n - 1)])


def read_rrmp(path: str, chi_max: int = 0, trunc_tolerance: float = 0.0, ctx=None):
    """Read RRMP v1 into a new device-resident tebd.DeviceMps."""
    from .tebd import DeviceMps
    dims, gammas, lambdas = read_rrmp_arrays(path)
    mps = DeviceMps(dims, chi_max, trunc_tolerance, ctx=ctx)
    mps.load(gammas, lambdas)
    return mps


# ------------------------------------------------------------------------------- chain files

def read_coefficients_file(path: str):
    """-> (t0, omegas, hoppings) (chainmap.cpp:280-301)."""
    omegas, ts = [], []
    with open(path) as f:
        for line in f:
            if not line.strip() or line.startswith("#"):
                continue
            parts = line.split()
            try:
                n, om, t = int(parts[0]), float(parts[1]), float(parts[2])
            except (ValueError, IndexError):
                raise ContractViolation(f"bad coefficients line: {line.rstrip()}") from None
            if n != len(omegas):
                raise ContractViolation(f"coefficients file rows out of order: {path}")
            omegas.append(om)
            ts.append(t)
    if not omegas:
        raise ContractViolation(f"empty coefficients file: {path}")
    return ts[0], np.array(omegas), np.array(ts[1:])


def write_coefficients_file(path: str, t0: float, omegas, hoppings) -> None:
    with open(path, "w") as f:
        for n, om in enumerate(omegas):
            t = t0 if n == 0 else hoppings[n - 1]
            f.write(f"{n} {format_double(om)} {format_double(t)}\n")
