"""Chain-block partition host logic on CPU: gloo world_size 2 processes and the
in-process loopback must reproduce the unpartitioned chain exactly (same per-bond operations,
same global seeds)."""
import os
import socket
import tempfile

import numpy as np
import pytest

from paper_1504_00992_b200 import models as M
from paper_1504_00992_b200.parallel import (BlockSpec, ChainPartition, LoopbackHub, evolve_loopback,
                                            partition)
from tests.numpy_block import NumpyBlock

N_SITES, CHI, DT, STEPS = 10, 6, 0.07, 4
KW = dict(randomized=True, target_rank=CHI, oversampling=3, det_crossover=4)


def chain():
    terms = M.ising_terms(N_SITES, 1.0, 0.8)
    plan = M.trotter_plan_3rd(DT)
    gates = {(s, b): M.bond_gate(terms[b], c * DT) for s, (p, c) in enumerate(plan)
             for b in range(N_SITES - 1) if b % 2 == p}
    up = np.zeros((1, 2, 1), complex)
    up[0, 0, 0] = 1.0
    return plan, gates, [up.copy() for _ in range(N_SITES)], [np.ones(1) for _ in range(N_SITES - 1)]


def serial_reference():
    plan, gates, g, l = chain()
    spec = BlockSpec(0, 1, 0, N_SITES, N_SITES)
    blk = NumpyBlock(spec, g, l, CHI, KW)
    part = ChainPartition(blk, LoopbackHub(1).comm(0), list(range(N_SITES - 1)))
    kept = evolve_loopback([part], gates, plan, DT, STEPS, [None], 100)
    return blk, kept


def assemble(blocks):
    gam, lam = [], []
    for blk in blocks:
        own = blk.spec.b - blk.spec.a
        gam += blk.g[:own]
        nb = own if blk.spec.has_ghost else own - 1
        lam += blk.lam[:nb]
    return gam, lam


def test_partition_shapes():
    assert partition(10, 2) == [(0, 5), (5, 10)]
    assert partition(101, 4, first_block=26)[0] == (0, 26)
    with pytest.raises(ValueError):
        partition(3, 2)


@pytest.mark.parametrize("world", [2, 3])
def test_loopback_partition_equals_serial(world):
    ref_blk, ref_kept = serial_reference()
    plan, gates, g, l = chain()
    parts, blocks = [], []
    hub = LoopbackHub(world)
    for r, (a, b) in enumerate(partition(N_SITES, world)):
        spec = BlockSpec(r, world, a, b, N_SITES)
        blk = NumpyBlock(spec, g, l, CHI, KW)
        blocks.append(blk)
        parts.append(ChainPartition(blk, hub.comm(r), list(range(N_SITES - 1))))
    kept = evolve_loopback(parts, gates, plan, DT, STEPS, [None] * world, 100)
    gam, lam = assemble(blocks)
    assert abs(kept - ref_kept) < 1e-14
    assert [x.shape for x in gam] == [x.shape for x in ref_blk.g]
    for a, b in zip(lam, ref_blk.lam):
        assert np.array_equal(a, b)
    for a, b in zip(gam, ref_blk.g):
        assert np.array_equal(a, b)


def _gloo_worker(rank, world, port_, outdir):
    import torch.distributed as dist

    from paper_1504_00992_b200.parallel import TorchComm
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port_}", rank=rank, world_size=world)
    plan, gates, g, l = chain()
    a, b = partition(N_SITES, world)[rank]
    spec = BlockSpec(rank, world, a, b, N_SITES)
    blk = NumpyBlock(spec, g, l, CHI, KW)
    part = ChainPartition(blk, TorchComm("cpu"), list(range(N_SITES - 1)))
    kept = part.evolve(gates, plan, DT, STEPS, None, 100)
    own = b - a
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), kept=kept,
             **{f"g{i}": blk.g[i] for i in range(own)},
             **{f"l{i}": blk.lam[i] for i in range(own if spec.has_ghost else own - 1)})
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks_equal_serial():
    import torch.multiprocessing as mp
    ref_blk, ref_kept = serial_reference()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port_ = s.getsockname()[1]
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_gloo_worker, args=(2, port_, d), nprocs=2, join=True)
        gam, lam, kept = [], [], 1.0
        for r in range(2):
            z = np.load(os.path.join(d, f"rank{r}.npz"))
            kept *= float(z["kept"])
            gam += [z[k] for k in sorted((k for k in z.files if k.startswith("g")), key=lambda k: int(k[1:]))]
            lam += [z[k] for k in sorted((k for k in z.files if k.startswith("l")), key=lambda k: int(k[1:]))]
    assert abs(kept - ref_kept) < 1e-14
    for a, b in zip(lam, ref_blk.lam):
        assert np.array_equal(a, b)
    for a, b in zip(gam, ref_blk.g):
        assert np.array_equal(a, b)
