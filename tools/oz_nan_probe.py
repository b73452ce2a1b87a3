import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1504_00992_b200 as P
from tests.conftest import cplx_randn
rng = np.random.default_rng(1)
As = [cplx_randn(rng, 2000, 2000) for _ in range(3)]
As[1][5, 7] = np.nan
try:
    S, w = P.rrsvd_fixed_rank_batch(As, 100, 10, 2, [1, 2, 3])
    print("result sigma finite:", [bool(np.all(np.isfinite(s))) for s in S], "w", w)
except Exception as e:
    print("raised", type(e).__name__, e)
