"""First-contact GPU checks: DMMA zgemm vs the reference zgemm, device Ω vs reference Ω."""
import numpy as np
import pytest

from tests.conftest import cplx_randn

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,n,k", [(8, 8, 4), (64, 64, 64), (100, 37, 129), (512, 74, 512), (3, 200, 1000)])
@pytest.mark.parametrize("adj", [False, True])
@pytest.mark.parametrize("adj_b", [False, True])
def test_zgemm_matches_reference(ctx, ref, m, n, k, adj, adj_b):
    """rrsvd::gemm (linalg.cpp:20-35) with every op combination, adj_b included."""
    import paper_1504_00992_b200 as P
    rng = np.random.default_rng(m * 1000 + n + k)
    a = cplx_randn(rng, *((k, m) if adj else (m, k)))
    b = cplx_randn(rng, *((n, k) if adj_b else (k, n)))
    got = P.gemm(a, adj, b, adj_b, ctx=ctx)
    want = ref.gemm(a, adj, b, adj_b)
    # test_linalg.cpp:86-90 bar: 1e-13 relative to the operand scale
    assert np.max(np.abs(got - want)) <= 1e-13 * np.sqrt(k) * 4


def test_peaks(ctx):
    import paper_1504_00992_b200 as P
    dmma = P.probe_peak(0, ctx=ctx)
    dfma = P.probe_peak(1, ctx=ctx)
    print(f"\nFP64 DMMA peak {dmma:.2f} TF/s, DFMA peak {dfma:.2f} TF/s")
    assert dmma > 1.0 and dfma > 1.0
