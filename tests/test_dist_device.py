"""The multi-process executor on the DEVICE path (GPU).

``pfasst_run(executor="nccl")`` places time rank n on process n % world and
hands payloads between processes with torch.distributed point-to-point
messages.  This box has one GPU and NCCL refuses two ranks on one device, so
two processes share cuda:0 over a gloo group and the exchange stages the
device payloads through host memory (DistExchange.host_wire).  Everything
else -- DeviceEngine, the cyclic rank placement, the wavefront issue order of
several ranks per process, the send fences, frozen-predecessor caching, the
block-end broadcast and the per-solve log gathering -- is the code a
multi-GPU NCCL run executes.  The kernels of one process never wait on the
other's: every hand-off is a blocking host-side exchange.

Each run must equal the golden reference run (counts, per-solve log,
convergence, trace, u within 1e-10) and the single-process device run bit
for bit.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402

from tests.golden_io import case  # noqa: E402

RUNS = ["run_cfg1", "run_same_n_3lvl", "run_cfg3_small", "run_cfg4_small"]


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _levels(m):
    from paper_1407_6486_b200 import heat, hierarchy, multigrid as mg, quadrature
    pol = mg.FixedCycles(m["policy"][1]) if m["policy"][0] == "fixed" else \
        mg.ToTolerance(*m["policy"][1:])
    orders = m.get("orders") or [2] * len(m["ns"])
    return [hierarchy.Level(heat.HeatOperator(heat.Grid(m["d"], n), 1.0, o),
                            quadrature.uniform_table(k - 1),
                            mg.MgConfig(m["sm"], m["om"], m["pre"], m["post"]), pol,
                            space_interp_order=m.get("interp", 4))
            for n, k, o in zip(m["ns"], m["nodes"], orders)]


def _run(name, executor):
    from paper_1407_6486_b200 import pfasst
    a, m = case(name)
    log = []
    res = pfasst.pfasst_run(_levels(m), torch.from_numpy(a["u0"]).cuda(),
                            m["dt"] * m["p"] * m["blocks"], m["p"], blocks=m["blocks"],
                            tol=m["tol"], max_iter=20, executor=executor,
                            record_final_values=True, solve_log=log)
    fv = [[v.cpu().numpy() if hasattr(v, "cpu") else np.asarray(v) for v in blk]
          for blk in res.final_values]
    return (res.rank_iterations, res.rank_vcycles, res.converged,
            [(t.block, t.rank, t.iteration, t.level, t.residual, t.vcycles) for t in res.trace],
            res.u.cpu().numpy(), log, fv)


def _worker(rank, world, port, name, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, _run(name, "nccl")))
    except Exception as exc:          # surface the failure in the parent
        q.put((rank, repr(exc)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", RUNS)
def test_two_processes_on_one_gpu_equal_single_process(name):
    a, m = case(name)
    single = _run(name, "serial")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    world = 2
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = [q.get(timeout=600) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    for rank, got in out:
        assert not isinstance(got, str), got
        iters, vcyc, conv, trace, u, log, fv = got
        assert iters == single[0] == m["rank_iterations"]
        assert vcyc == single[1] == m["rank_vcycles"]
        assert conv == single[2] == m["converged"]
        assert trace == single[3]                      # residuals bit for bit
        assert np.array_equal(u, single[4]), rank
        assert log == single[5]
        assert [r for blk in log for r in blk] == m["solves"]
        for b1, b2 in zip(fv, single[6]):
            assert all(np.array_equal(x, y) for x, y in zip(b1, b2))
        scale = np.max(np.abs(a["u"]))
        assert np.max(np.abs(u - a["u"])) <= 1e-10 * scale
