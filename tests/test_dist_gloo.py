"""Multi-process time ranks over torch.distributed (gloo on CPU).

The "nccl" executor of pfasst_run places time rank n on process n % world
and hands the fine / coarse initial values and the converged flag between
processes with point-to-point messages (NCCL on GPUs).  Here the same
exchange code runs over gloo with the oracle as the per-rank engine
(tests/oracle_engine.py), and every process must reproduce the oracle's
serial schedule bit for bit: iteration counts, V-cycles, convergence flags,
the residual trace and the final value -- including frozen ranks (cached
payloads instead of resends) and multi-block chaining.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import pintlab_oracle as O
from paper_1407_6486_b200 import heat, hierarchy, multigrid as mg, pfasst, quadrature
from tests.oracle_engine import OracleEngine


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def make_levels(n, nodes, policy):
    return [hierarchy.Level(heat.HeatOperator(heat.Grid(1, nn)), quadrature.uniform_table(k - 1),
                            mg.MgConfig(), policy, space_interp_order=4)
            for nn, k in zip(n, nodes)]


CASES = {
    # name: (grids, nodes, policy, P, blocks, tol, max_iter)
    "two_level_fixed": ((64, 32), (5, 3), mg.FixedCycles(1), 4, 1, 1e-10, 20),
    "three_level_tol_blocks": ((64, 32, 16), (5, 3, 2), mg.ToTolerance(1e-12), 5, 2, 1e-9, 12),
    "unconverged": ((32, 16), (3, 2), mg.FixedCycles(1), 3, 1, 1e-300, 3),
    # several ranks per process (wavefront issue order), staggered freezing
    "six_ranks_two_blocks": ((64, 32), (5, 3), mg.FixedCycles(1), 6, 2, 1e-9, 15),
}


def _worker(rank, world, port, name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        grids, nodes, pol, p, blocks, tol, mi = CASES[name]
        levels = make_levels(grids, nodes, pol)
        u0 = heat.initial_condition(levels[0].grid, 1)
        res = pfasst.pfasst_run(levels, torch.from_numpy(u0), 0.1 * blocks, p, blocks=blocks,
                                tol=tol, max_iter=mi, executor="nccl",
                                engine_factory=OracleEngine)
        q.put((rank, res.rank_iterations, res.rank_vcycles, res.converged,
               [(t.block, t.rank, t.iteration, t.level, t.residual, t.vcycles)
                for t in res.trace], res.u.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", sorted(CASES))
def test_distributed_schedule_matches_serial_oracle(name, world):
    grids, nodes, pol, p, blocks, tol, mi = CASES[name]
    levels = make_levels(grids, nodes, pol)
    u0 = heat.initial_condition(levels[0].grid, 1)
    ref = O.pfasst_run(OracleEngine(levels, 0.0, []).levels, u0, 0.1 * blocks, p, blocks, tol, mi)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = [q.get(timeout=240) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, iters, vcyc, conv, trace, u in out:
        assert iters == ref.rank_iterations
        assert vcyc == ref.rank_vcycles
        assert conv == ref.converged
        assert trace == [tuple(t) for t in ref.trace]
        assert np.array_equal(u, ref.u), rank
