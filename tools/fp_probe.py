"""Fixed-precision growth probe: device vs reference on a rank-6 120x80 matrix (shim_test shape)."""
import itertools
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1504_00992_b200 as P
from oracle import ref

ctx = P.Context(0)
l = ref.gaussian_test_matrix(120, 6, 4); r = ref.gaussian_test_matrix(80, 6, 5)
a = l @ r.conj().T
for g, l0, q in itertools.product((0, 1, 2, 3, 4, 5), (1, 2, 3, 5, 8), (0, 1)):
    u, s, v, w, c = ref.fixed_precision(a, 1e-8, 4, l0, q, 11, growth_block=g)
    try:
        res = P.rrsvd_fixed_precision(a, 1e-8, 4, l0, q, 11, growth_block=g, ctx=ctx)
        ds = np.max(np.abs(res.sigma[:6] - s[:6])) / s[0]
        print(f"g={g} l0={l0} q={q}: ref l={len(s)} cert={c} | dev l={res.achieved_rank} cert={res.tolerance_certified} dsig={ds:.2e}"
              + ("" if (res.achieved_rank == len(s) and res.tolerance_certified == c) else "   <-- MISMATCH"))
    except Exception as e:
        print(f"g={g} l0={l0} q={q}: ref l={len(s)} cert={c} | dev EXC {e}")
