"""The arithmetic of the INT8 emulated A-products (csrc/ozaki.cuh), restated in Python integers and
checked on the CPU: moduli, exponent budget, symmetric residues, the epilogue's (D mod m)·w mod m,
the 96-bit fixed-point CRT, and the power-of-two equilibration of A and the panel.  The device
kernels are checked against numpy / the reference in tests/test_gpu_ozaki.py and
tests/test_gpu_variants.py; this file pins the scheme itself (exactness up to the stated bounds)."""
import math

import numpy as np
import pytest

MODULI = [256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193]  # ozaki.cu kModuli


def consts(T):
    ms = MODULI[:T]
    M = math.prod(ms)
    bits = M.bit_length() - 1
    w = [pow(M // m % m, -1, m) for m in ms]
    c = [((1 << 128) - 1) // m for m in ms]
    c3 = [[(x >> 32) & 0xFFFFFFFF, (x >> 64) & 0xFFFFFFFF, (x >> 96) & 0xFFFFFFFF] for x in c]
    return ms, M, bits, w, c3


def total_bits(bits, K):
    return bits - 2 - math.ceil(math.log2(2 * K))


def sym_res(v, m):
    r = v % m
    return r - m if r > m - 1 - m // 2 else r


def crt96(ts, ms, M, c3):
    a = [0, 0, 0]
    for t, limbs in zip(ts, c3):
        for i in range(3):
            a[i] += t * limbs[i]
    F = ((a[0] << 32) + (a[1] << 64) + (a[2] << 96)) % (1 << 128)
    if F >= 1 << 127:
        F -= 1 << 128
    return (F * M + (1 << 127)) >> 128  # exact integer rounding (the kernel rounds once to FP64)


def test_moduli_pairwise_coprime_and_budget():
    for i, a in enumerate(MODULI):
        for b in MODULI[:i]:
            assert math.gcd(a, b) == 1
    for T, want in ((14, 96), (16, 111)):
        _, M, bits, _, _ = consts(T)
        assert total_bits(bits, 2000) == want  # kA + kX at K = 2000 (C3): 48 + 48 / 56 + 55
    # int32 accumulators: 2K products of |r| <= 128 each stay below 2^31 up to K = 32768
    assert 2 * 32768 * 128 * 128 <= 2 ** 31


@pytest.mark.parametrize("T", [14, 16])
def test_residue_gemm_and_crt_are_exact(T):
    """D = A'X' (integers at the full kA / kX budget) from T residue products, the epilogue's
    t = (D mod m)·w mod m, and the 96-bit CRT: |CRT - D| <= 2^(bits - 82), i.e. exact far below
    one unit of the scaled inputs' rounding."""
    ms, M, bits, w, c3 = consts(T)
    rng = np.random.default_rng(T)
    K = 64
    tot = total_bits(bits, K)
    kA = (tot + 1) // 2
    kX = tot - kA
    A = [[int(x) for x in row] for row in rng.integers(-(2 ** 62), 2 ** 62, (6, K), dtype=np.int64) >> (62 - kA)]
    X = [[int(x) for x in row] for row in rng.integers(-(2 ** 62), 2 ** 62, (K, 5), dtype=np.int64) >> (62 - kX)]
    A[0] = [2 ** kA] * K  # the extremes
    X = [[2 ** kX if j == 0 else x for j, x in enumerate(row)] for row in X]
    for i in range(6):
        for j in range(5):
            D = sum(A[i][k] * X[k][j] for k in range(K))
            assert abs(D) < M // 2
            ts = []
            for m, wt in zip(ms, w):
                acc = sum(sym_res(A[i][k], m) * sym_res(X[k][j], m) for k in range(K))
                assert abs(acc) < 2 ** 31
                x = acc % m
                ts.append(x * wt % m)
            assert abs(crt96(ts, ms, M, c3) - D) <= 2 ** (bits - 82)


def test_complex_product_as_one_real_gemm():
    """op N: [Y_re | Y_im] = [A_re A_im]·[[X_re, X_im], [-X_im, X_re]]; op C: [Z_re | Z_im] =
    [A_re A_im]^T·[[X_re, X_im], [X_im, -X_re]] (the B' panel layout of oz_resid_b)."""
    rng = np.random.default_rng(0)
    a = rng.integers(-50, 50, (7, 9)) + 1j * rng.integers(-50, 50, (7, 9))
    x = rng.integers(-50, 50, (9, 4)) + 1j * rng.integers(-50, 50, (9, 4))
    lhs = np.hstack([a.real, a.imag])
    for sg, prod in ((-1, a @ x), (+1, None)):
        if sg > 0:
            q = rng.integers(-50, 50, (7, 4)) + 1j * rng.integers(-50, 50, (7, 4))
            prod = a.conj().T @ q
            rhs = np.vstack([np.hstack([q.real, q.imag]), np.hstack([q.imag, -q.real])])
            d = np.vstack([a.real, a.imag]).T @ rhs
        else:
            rhs = np.vstack([np.hstack([x.real, x.imag]), np.hstack([-x.imag, x.real])])
            d = lhs @ rhs
        n = d.shape[1] // 2
        assert np.array_equal(d[:, :n] + 1j * d[:, n:], prod)


def test_two_sided_equilibration_bounds():
    """A' = rint(A·2^(kA - e_i - f_k)): e_i = exponent of row i's max, f_k = max_i e(|A_ik|) - e_i <= 0;
    every |A'| <= 2^kA, and a λ-graded Θ keeps ~kA significant bits in every entry."""
    rng = np.random.default_rng(3)
    kA = 48
    lam_l = 0.7 ** np.arange(40)
    lam_r = 0.6 ** np.arange(30)
    a = (rng.standard_normal((40, 30)) + 1j * rng.standard_normal((40, 30))) * lam_l[:, None] * lam_r[None, :]
    mag = np.maximum(np.abs(a.real), np.abs(a.imag))
    e_el = np.frexp(mag)[1]  # mag in [2^(e-1), 2^e)
    e_row = e_el.max(axis=1)
    f_col = (e_el - e_row[:, None]).max(axis=0)
    assert np.all(f_col <= 0)
    scale = np.ldexp(1.0, (kA - e_row[:, None] - f_col[None, :]))
    ap_re, ap_im = np.rint(a.real * scale), np.rint(a.imag * scale)
    assert np.max(np.abs(ap_re)) <= 2 ** kA and np.max(np.abs(ap_im)) <= 2 ** kA
    back = (ap_re + 1j * ap_im) / scale
    rel = np.abs(back - a) / mag
    # relative rounding of each entry against its own magnitude: the grading costs no precision
    # beyond the row/column spread of a rank-1-scaled matrix (a few bits here)
    assert np.max(rel) < 2.0 ** (-kA + 12)
    # a single global scale would lose ~log2(max/min) bits on the small entries
    g = np.ldexp(1.0, kA - int(e_el.max()))
    glob = (np.rint(a.real * g) + 1j * np.rint(a.imag * g)) / g
    assert np.max(np.abs(glob - a) / mag) > 1e3 * np.max(rel)


def _f32(x):
    return np.float32(x)


@pytest.mark.parametrize("T", [14, 15, 16])
def test_paired_residues(T):
    """oz_store8_pair: r = v mod m_a·m_b by a shifter-rounded FP64 quotient and an exact remainder,
    then each residue's quotient from an FP32 shifter (fmaf rounds once: emulated here by an FP64
    sum rounded to FP32) and the byte from the integer remainder — the symmetric residue of v for
    every modulus of the pair."""
    rng = np.random.default_rng(T)
    sh64 = 6755399441055744.0
    sh32 = np.float32(12582912.0)
    vals = [float(x) for x in rng.integers(-(2 ** 52), 2 ** 52, 4000, dtype=np.int64)]
    vals += [0.0, 2.0 ** 52, -(2.0 ** 52), 32640.0, -32640.0, 65280.0 * 12345 + 32640, -(65280.0 * 777 + 32640)]
    for t in range(0, T - 1, 2):
        ma, mb = MODULI[t], MODULI[t + 1]
        P = float(ma * mb)
        for v in vals:
            q = (v * (1.0 / P) + sh64) - sh64          # |v/P| < 2^37: the FP64 product's rounding is below 2^-15
            r = v - q * P                              # exact (an FMA on the device)
            assert abs(r) <= P / 2 + 1
            f = np.float32(r)
            ri = int(r)
            for m in (ma, mb):
                # q from the FP32 shifter's bits (fmaf rounds once), the byte from ri - q·m
                shifted = _f32(np.float64(f) * np.float64(np.float32(1.0 / m)) + np.float64(sh32))
                qq = int(shifted - sh32)
                rr = ri - qq * m
                assert abs(rr) <= m / 2
                byte = rr & 0xFF
                want = sym_res(int(v), m) & 0xFF
                assert byte == want, (v, m, rr, sym_res(int(v), m))
                # the kernel's single IMAD: the low byte of ri - bits·m, bits the shifter's FP32 bit
                # pattern (= q + 0x4B400000, and 0x4B400000·m = 0 mod 256)
                bits = int(np.array([shifted], np.float32).view(np.int32)[0])
                assert bits - 0x4B400000 == qq
                assert (ri - bits * m) & 0xFF == want
