"""The chain-block partition behind the C ABI (rrsvd_b200_evolve_partitioned):
ranks driven as host threads of one process with the host-staged loopback transport (ranks never
wait on each other's kernels on the device), and the NCCL transport at one rank.  A partitioned
run must reproduce the single-GPU evolve (global call-index seeds): observables and entropies
within 1e-10, the same χ profile and the seed counter where the unpartitioned evolve leaves it."""
import threading

import numpy as np
import pytest

import paper_1504_00992_b200 as P
from paper_1504_00992_b200 import models as Mdl
from paper_1504_00992_b200.parallel import (NativeComm, NativeLoopbackHub, evolve_partitioned,
                                            partition)
from paper_1504_00992_b200.tebd import DeviceMps, PreparedGates, build_gates, evolve

pytestmark = pytest.mark.gpu

KW = dict(randomized=True, target_rank=10, oversampling=6, power_iterations=2, det_crossover=0, seed=17)


def run_partitioned(n, chi, terms, dt, steps, world, make_comm):
    plan, gates = build_gates([2] * n, terms, dt)
    blocks = partition(n, world)
    out, errs = [None] * world, []

    def rank_main(r):
        try:
            a, b = blocks[r]
            ghost = r + 1 < world
            sites = list(range(a, b + (1 if ghost else 0)))
            ctx = P.Context(0)
            blk = DeviceMps([2] * len(sites), chi, ctx=ctx)
            local = {(s, gb - a): g for (s, gb), g in gates.items() if gb - a < len(sites) - 1 and gb >= a}
            pg = PreparedGates(local, ctx)
            be = P.DecimationBackend(**KW)
            comm = make_comm(ctx, r)
            d = evolve_partitioned(blk, comm, a, n, pg, plan, list(terms), steps, be)
            out[r] = (a, b, ghost, blk, be.seed, d, ctx, comm, pg)
        except Exception as e:  # noqa: BLE001
            import sys
            import traceback
            traceback.print_exc(file=sys.stderr)
            errs.append((r, e))

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    return out


def reference_run(n, chi, terms, dt, steps):
    full = DeviceMps([2] * n, chi)
    be = P.DecimationBackend(**KW)
    evolve(full, terms, dt, steps, be)
    return full, be.seed


def compare(full, parts, n):
    for a, b, ghost, blk, *_ in parts:
        for s in range(a, b):
            assert abs(blk.expectation_local(s - a, Mdl.SZ) - full.expectation_local(s, Mdl.SZ)) < 1e-10, s
        for j in range(a, b if ghost else b - 1):
            assert abs(blk.schmidt_entropy(j - a) - full.schmidt_entropy(j)) < 1e-10, j
            assert blk.dims(j - a)[2] == full.dims(j)[2]


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_loopback_matches_single_gpu(world):
    n, chi, dt, steps = 12, 12, 0.08, 6
    terms = dict(enumerate(Mdl.ising_terms(n, 1.0, 0.8)))
    hub = NativeLoopbackHub(world)
    parts = run_partitioned(n, chi, terms, dt, steps, world, lambda ctx, r: NativeComm.loopback(ctx, hub, r))
    full, seed = reference_run(n, chi, terms, dt, steps)
    assert all(p[4] == seed for p in parts)
    assert max(p[5].max_bond_dim for p in parts) == max(full.bond_dims())
    compare(full, parts, n)


def test_partitioned_nccl_one_rank():
    """The NCCL transport end to end at one rank (this box has one GPU): libnccl loads, the
    communicator initialises, and the run equals the unpartitioned evolve."""
    n, chi, dt, steps = 10, 8, 0.08, 4
    terms = dict(enumerate(Mdl.ising_terms(n, 1.0, 0.8)))
    uid = NativeComm.unique_id()
    parts = run_partitioned(n, chi, terms, dt, steps, 1, lambda ctx, r: NativeComm.nccl(ctx, 1, 0, uid))
    full, seed = reference_run(n, chi, terms, dt, steps)
    assert parts[0][4] == seed
    compare(full, parts, n)


def test_loopback_peer_failure_does_not_hang():
    """A rank whose call fails releases its peers: their receives raise instead of waiting forever
    (rank 1's block has chi_max = 0, a contract violation before any exchange)."""
    n, chi, dt, steps = 12, 12, 0.08, 2
    terms = dict(enumerate(Mdl.ising_terms(n, 1.0, 0.8)))
    plan, gates = build_gates([2] * n, terms, dt)
    blocks = partition(n, 2)
    hub = NativeLoopbackHub(2)
    errs = [None, None]

    def rank_main(r):
        a, b = blocks[r]
        sites = list(range(a, b + (1 if r == 0 else 0)))
        ctx = P.Context(0)
        blk = DeviceMps([2] * len(sites), chi if r == 0 else 0, ctx=ctx)
        local = {(s, gb - a): g for (s, gb), g in gates.items() if gb - a < len(sites) - 1 and gb >= a}
        pg = PreparedGates(local, ctx)
        comm = NativeComm.loopback(ctx, hub, r)
        try:
            evolve_partitioned(blk, comm, a, n, pg, plan, list(terms), steps, P.DecimationBackend(**KW))
        except Exception as e:  # noqa: BLE001
            errs[r] = e

    th = [threading.Thread(target=rank_main, args=(r,), daemon=True) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert not any(t.is_alive() for t in th), "a rank is still blocked on its failed peer"
    assert isinstance(errs[1], P.ContractViolation)
    assert errs[0] is not None and "peer rank failed" in str(errs[0])
