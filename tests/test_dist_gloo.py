"""Multi-process (world_size 2, gloo, CPU) coverage of the sharding path: the
partition, padding, global-id RNG offsets and the all-gather reassembly of
parallel.solve_sharded give exactly the single-process result.  The per-rank
solve is the fp64 oracle here (no GPU on this box); on B200 it is hjcd_solve."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from params import params
from paper_2510_07514_b200 import hjcd, inputs, parallel

P = params(M=16, K=4, B=8, ccd_iters=16, lm_iters=16)


class FakeRobot:
    dof = 7


def oracle_solve_fn(robot, targets, cfg):
    p = dict(P)
    q, pe, oe, st = oracle.solve(inputs.panda(), p, targets.numpy(), tid_offset=int(cfg.target_index_offset))
    return (torch.from_numpy(q.astype(np.float32)), torch.from_numpy(pe.astype(np.float32)),
            torch.from_numpy(oe.astype(np.float32)), torch.from_numpy(st))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, tg, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = hjcd.hjcd_config()
    cfg.target_index_offset = 0
    out = parallel.solve_sharded(FakeRobot(), torch.from_numpy(tg), cfg, solve_fn=oracle_solve_fn)
    if rank == 0:
        ret.put([o.numpy() for o in out])
    dist.barrier()
    dist.destroy_process_group()


def test_partition():
    assert parallel.partition(10, 4, 0) == (0, 3, 3)
    assert parallel.partition(10, 4, 3) == (9, 1, 3)
    assert parallel.partition(3, 8, 5) == (3, 0, 1)
    total = sum(parallel.partition(1001, 8, r)[1] for r in range(8))
    assert total == 1001


def test_pack_roundtrip():
    q = torch.randn(5, 7)
    pe, oe = torch.rand(5), torch.rand(5)
    st = torch.tensor([0, 1, 2, 3, 0], dtype=torch.int32)
    out = parallel.unpack(parallel.pack(q, pe, oe, st), 7)
    assert all(torch.equal(a, b) for a, b in zip(out, (q, pe, oe, st)))


@pytest.mark.parametrize("T", [5, 6])
def test_sharded_equals_single_process(T):
    ch = inputs.panda()
    tg = oracle.fk(ch, inputs.halton_configs(ch, T)).astype(np.float32)
    ctx = mp.get_context("spawn")
    ret = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, tg, ret)) for r in range(2)]
    for p in procs:
        p.start()
    got = ret.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = oracle.solve(ch, dict(P), tg)
    assert np.array_equal(got[0], ref[0].astype(np.float32))
    assert np.array_equal(got[3], ref[3])


def _bench(args, env_extra):
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py")] + args, cwd=root, env=env,
                       capture_output=True, text=True, timeout=600)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    return r.returncode, (json.loads(lines[-1]) if lines else None), r.stderr


def test_bench_gpus_flag_launches_ranks():
    # bench.py --gpus 2 outside torchrun re-launches itself under
    # torch.distributed.run with 2 ranks (127.0.0.1 rendezvous); --check-launch
    # runs the multi-rank plumbing without a solve, so it is CPU-testable (gloo)
    env = {"HJCD_DIST_BACKEND": "gloo"}
    env_clean = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    os_env = os.environ.copy()
    try:
        os.environ.clear()
        os.environ.update(env_clean)
        rc, out, err = _bench(["--gpus", "2", "--check-launch"], env)
        assert rc == 0, err[-2000:]
        assert out == {"check": "launch", "n_gpus": 2, "ranks": [0, 1], "backend": "gloo"}
        # under a launcher the world size must equal --gpus
        rc, out, err = _bench(["--gpus", "2", "--check-launch"], {"WORLD_SIZE": "1"})
        assert rc == 2 and "WORLD_SIZE=1 but --gpus 2" in err
    finally:
        os.environ.clear()
        os.environ.update(os_env)
