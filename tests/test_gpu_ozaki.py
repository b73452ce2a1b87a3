"""The INT8 tensor-core (tcgen05 kind::i8) Chinese-remainder emulation of the RRSVD A-products
(csrc/ozaki.cuh) against numpy's complex128 product — the reference's cblas_zgemm call site
(linalg.cpp:20-40) as used by randomized.cpp:88-99 (Y = A·Ω, Z = Aᴴ·Q) and 57-66 (Bᴴ = Aᴴ·Q)."""
import numpy as np
import pytest

from tests.conftest import cplx_randn

pytestmark = pytest.mark.gpu


def _err(got, want, a, b):
    """max-entry error over the operand scale max|A|·||B[:, j]||_1 (the integer scheme's bound)."""
    amax = np.max(np.maximum(np.abs(a.real), np.abs(a.imag)))
    col = np.sum(np.abs(b), axis=0)
    return float(np.max(np.abs(got - want) / (amax * col[None, :] + 1e-300)))


SHAPES = [(2000, 110, 2000), (300, 40, 257), (1000, 210, 700), (129, 8, 4000), (700, 128, 130)]


@pytest.mark.parametrize("m,n,k", SHAPES)
@pytest.mark.parametrize("adj", [False, True])
def test_ozaki_matches_zgemm(ctx, m, n, k, adj):
    import paper_1504_00992_b200 as P
    rng = np.random.default_rng(m + 7 * n + 13 * k + adj)
    a = cplx_randn(rng, *((k, m) if adj else (m, k)))
    b = cplx_randn(rng, k, n)
    want = (a.conj().T if adj else a) @ b
    got = P.ozaki_gemm(a, adj, b, 16, ctx=ctx)
    e = _err(got, want, a, b)
    print(f"\nozaki16 {m}x{n}x{k} adj={adj}: err {e:.2e}")
    # 16 moduli: kA + kX = 125 - 2 - log2(2k) >= 107 bits -> per-entry rounding <= 2^-53 of the scale
    assert e <= 1e-15
    dm = P.gemm(a, adj, b, ctx=ctx)
    assert np.max(np.abs(got - dm)) <= 1e-13 * np.sqrt(k) * np.max(np.abs(want))


@pytest.mark.parametrize("moduli,bar", [(14, 1e-13), (12, 1e-10)])
def test_ozaki_fewer_moduli(ctx, moduli, bar):
    import paper_1504_00992_b200 as P
    rng = np.random.default_rng(moduli)
    a = cplx_randn(rng, 1000, 1000)
    b = cplx_randn(rng, 1000, 64)
    got = P.ozaki_gemm(a, False, b, moduli, ctx=ctx)
    e = _err(got, a @ b, a, b)
    print(f"\nozaki{moduli}: err {e:.2e}")
    assert e <= bar


def test_ozaki_graded_rows_and_columns(ctx):
    """A TEBD Θ has rows spanning many decades (λ-weighted); columns of X are scaled apart."""
    import paper_1504_00992_b200 as P
    rng = np.random.default_rng(5)
    a = cplx_randn(rng, 800, 600) * np.exp(-np.arange(800) / 40.0)[:, None]
    b = cplx_randn(rng, 600, 50) * (10.0 ** rng.uniform(-30, 30, 50))[None, :]
    for adj in (False, True):
        aa = a if not adj else a.conj().T.copy()
        want = a @ b
        got = P.ozaki_gemm(aa, adj, b, 16, ctx=ctx)
        assert _err(got, want, a, b) <= 1e-15


def test_ozaki_nonfinite_and_zero(ctx):
    import paper_1504_00992_b200 as P
    rng = np.random.default_rng(9)
    a = cplx_randn(rng, 256, 256)
    b = cplx_randn(rng, 256, 20)
    z = P.ozaki_gemm(np.zeros_like(a), False, b, 16, ctx=ctx)
    assert np.all(z == 0)
    a[3, 7] = np.nan
    got = P.ozaki_gemm(a, False, b, 16, ctx=ctx)
    assert np.all(np.isnan(got))
    b2 = b.copy()
    b2[5, 4] = np.inf
    got = P.ozaki_gemm(np.nan_to_num(a), False, b2, 16, ctx=ctx)
    assert np.all(np.isnan(got[:, 4])) and np.all(np.isfinite(np.delete(got, 4, axis=1)))


def test_ozaki_device_tensors(ctx):
    import torch
    import paper_1504_00992_b200 as P
    g = torch.Generator(device="cuda").manual_seed(3)
    a = torch.randn(2000, 2000, dtype=torch.complex128, device="cuda", generator=g)
    b = torch.randn(2000, 110, dtype=torch.complex128, device="cuda", generator=g)
    got = P.ozaki_gemm(a, False, b, 16, ctx=ctx)
    want = a @ b
    assert torch.max(torch.abs(got - want)).item() <= 1e-12


def test_emulated_batch_isolates_a_nonfinite_problem(ctx, ref):
    """A batch large enough for the emulated A-products (3 x 2000^2) with a NaN in one matrix: that
    problem's σ / w are NaN (as the FP64 path gives), the others are unaffected and match the
    reference's rrsvd_fixed_rank (randomized.cpp:109-122) with the same Ω."""
    import paper_1504_00992_b200 as P
    rng = np.random.default_rng(1)
    As = [cplx_randn(rng, 2000, 2000) * (0.97 ** np.arange(2000))[None, :] for _ in range(3)]
    As[1][5, 7] = np.nan
    S, w = P.rrsvd_fixed_rank_batch(As, 100, 10, 2, [1, 2, 3], mode=P.OMEGA_REFERENCE, ctx=ctx)
    assert [bool(np.all(np.isfinite(s))) for s in S] == [True, False, True]
    assert np.isnan(w[1]) and np.isfinite(w[0]) and np.isfinite(w[2])
    for i in (0, 2):
        _, s_ref, _, w_ref = ref.fixed_rank(As[i], 100, 10, 2, i + 1, vectors=False)
        assert np.max(np.abs(np.asarray(S[i]) - s_ref)) < 1e-10 * s_ref[0]
        assert abs(w[i] - w_ref) < 1e-10


def test_prepared_operator_reused(ctx):
    """rrsvd_b200_ozaki_prepare once, _apply many times with both ops (the row-sharded RRSVD's
    pattern), _release: every product at the emulation's accuracy."""
    import paper_1504_00992_b200 as P
    rng = np.random.default_rng(11)
    a = cplx_randn(rng, 1500, 900) * (0.99 ** np.arange(900))[None, :]
    op = P.OzakiOperator(a, 15, ctx=ctx)
    try:
        for _ in range(3):
            x = cplx_randn(rng, 900, 110)
            assert _err(op.mul(False, x), a @ x, a, x) <= 1e-15
            q = cplx_randn(rng, 1500, 60)
            assert _err(op.mul(True, q), a.conj().T @ q, a.conj().T, q) <= 1e-15
    finally:
        op.close()
    assert P.ozaki_usable(2000, 2000) in (0, 15)


def test_streamed_k_chunks(ctx):
    """The row-sharded driver's streamed products (sharded.DeviceOps._streamed): an A wider than
    the int32 accumulator's K bound applied by prepared column blocks — op N accumulated over the
    blocks on the device (CRT with C += ...), op C one block of rows each."""
    import torch
    from paper_1504_00992_b200 import sharded
    ops = sharded.DeviceOps(ctx)
    ops.MAX_K = 512
    g = torch.Generator(device="cuda").manual_seed(5)
    a = torch.randn(700, 1500, dtype=torch.complex128, device="cuda", generator=g)
    x = torch.randn(1500, 40, dtype=torch.complex128, device="cuda", generator=g)
    q = torch.randn(700, 40, dtype=torch.complex128, device="cuda", generator=g)
    y = ops._streamed(a, False, x, 15)
    z = ops._streamed(a, True, q, 15)
    scale = float(torch.max(torch.abs(a)))
    assert float(torch.max(torch.abs(y - a @ x))) <= 1e-14 * scale * 1500
    assert float(torch.max(torch.abs(z - a.conj().T @ q))) <= 1e-14 * scale * 700


def test_emulation_contracts(ctx):
    """The emulation's ABI rejects what it cannot compute exactly (ContractViolation, status 1):
    moduli outside [8, 16], shapes outside [128, 32768], a mismatched panel, accumulation into host
    memory — and the context stays usable afterwards."""
    import paper_1504_00992_b200 as P
    rng = np.random.default_rng(2)
    a = cplx_randn(rng, 256, 256)
    x = cplx_randn(rng, 256, 8)
    with pytest.raises(P.ContractViolation):
        P.ozaki_gemm(a, False, x, 7, ctx=ctx)
    with pytest.raises(P.ContractViolation):
        P.ozaki_gemm(a, False, x, 17, ctx=ctx)
    with pytest.raises(P.ContractViolation):
        P.OzakiOperator(cplx_randn(rng, 64, 256), 15, ctx=ctx)
    op = P.OzakiOperator(a, 15, ctx=ctx)
    try:
        with pytest.raises(P.ContractViolation):
            op.mul(False, cplx_randn(rng, 200, 8))
        with pytest.raises(P.ContractViolation):
            op.mul(False, x, out=np.zeros((256, 8), np.complex128), accumulate=True)
        y = op.mul(False, x)
        assert _err(y, a @ x, a, x) <= 1e-15
    finally:
        op.close()
