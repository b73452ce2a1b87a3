"""The chain-block partition on the device: 2 and 3 simulated ranks on one GPU (loopback comm:
the driver's NCCL exchanges replaced by in-process hand-over of device tensors) must reproduce
the unpartitioned device evolve — same χ profile, λ and observables."""
import numpy as np
import pytest

import paper_1504_00992_b200 as P
from paper_1504_00992_b200 import models as M
from paper_1504_00992_b200.parallel import (BlockSpec, ChainPartition, DeviceBlock, LoopbackHub,
                                            evolve_loopback, partition)
from paper_1504_00992_b200.tebd import DeviceMps, build_gates, evolve

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 3])
def test_device_partition_equals_single(world):
    n, chi, dt, steps = 12, 10, 0.05, 4
    terms = {b: t for b, t in enumerate(M.ising_terms(n, 1.0, 0.7))}
    plan, gates = build_gates([2] * n, terms, dt)
    kw = dict(randomized=True, target_rank=chi, oversampling=4, det_crossover=6, seed=0)

    single = DeviceMps([2] * n, chi)
    evolve(single, terms, dt, steps, P.DecimationBackend(**kw), gates=gates, plan=plan)

    hub = LoopbackHub(world)
    parts, blocks = [], []
    for r, (a, b) in enumerate(partition(n, world)):
        spec = BlockSpec(r, world, a, b, n)
        blk = DeviceBlock(spec, [2] * n, chi)
        blk.set_edges(np.ones(1) if a > 0 else None, np.ones(1) if spec.has_ghost and b + 1 < n else None)
        blocks.append(blk)
        parts.append(ChainPartition(blk, hub.comm(r), list(terms)))
    evolve_loopback(parts, gates, plan, dt, steps, [P.DecimationBackend(**kw) for _ in range(world)], 0)

    sz = M.SZ
    for blk in blocks:
        own = blk.spec.b - blk.spec.a
        for i in range(own):
            gsite = blk.spec.a + i
            assert blk.mps.dims(i) == single.dims(gsite)
            if gsite + 1 < n:
                assert np.max(np.abs(blk.mps.lam(i) - single.lam(gsite))) < 1e-12
            assert abs(blk.mps.expectation_local(i, sz) - single.expectation_local(gsite, sz)) < 1e-10
