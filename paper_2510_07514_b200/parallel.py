"""Multi-GPU sharding of HJCD-IK (one process per GPU, torch.distributed).

Targets are independent (Alg. 2 runs per target), so the only
parallel axis across GPUs is the target batch.  Rank r solves a contiguous
block of ceil(T / W) targets with config.target_index_offset = r * ceil(T / W);
the RNG counter uses the GLOBAL target id, so the gathered result is bitwise
the single-GPU result.  The one exchange step is an all-gather of packed
per-target rows [q (n), pos_err, ori_err, status] (north_star: "only an NCCL
all-gather of results").  No data-path collective exists inside the solve.
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple

import torch
import torch.distributed as dist

from . import hjcd


def partition(T: int, world: int, rank: int) -> Tuple[int, int, int]:
    """(start, count, block): rank's rows [start, start + count) of T, blocks of
    `block` = ceil(T / world) rows (the last rank may hold fewer real rows)."""
    block = (T + world - 1) // world
    start = min(T, rank * block)
    count = max(0, min(T, start + block) - start)
    return start, count, block


def pack(q, pe, oe, st) -> torch.Tensor:
    """[T, n + 3] float32 rows: q, pos_err, ori_err, status (exact small ints)."""
    return torch.cat([q, pe[:, None], oe[:, None], st.to(torch.float32)[:, None]], dim=1).contiguous()


def unpack(rows: torch.Tensor, n: int):
    return (rows[:, :n].contiguous(), rows[:, n].contiguous(), rows[:, n + 1].contiguous(),
            rows[:, n + 2].to(torch.int32).contiguous())


def _all_gather_rows(rows: torch.Tensor, group=None) -> torch.Tensor:
    world = dist.get_world_size(group)
    out = torch.empty((world * rows.shape[0], rows.shape[1]), dtype=rows.dtype, device=rows.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, rows, group=group)
    elif rows.is_cuda:   # gloo with device tensors (functional multi-rank check): via host memory
        host = [torch.empty_like(rows, device="cpu") for _ in range(world)]
        dist.all_gather(host, rows.cpu(), group=group)
        out.copy_(torch.cat(host))
    else:
        dist.all_gather(list(out.chunk(world)), rows, group=group)
    return out


def solve_distributed(robot: "hjcd.Robot", local_targets: torch.Tensor, cfg: "hjcd.hjcd_config",
                      group=None, workspace=None, solve_fn: Optional[Callable] = None):
    """Each rank solves ITS targets (equal count on every rank; cfg carries the
    rank's target_index_offset); returns the all-gathered (q, pos_err, ori_err,
    status) of all ranks, rank-major."""
    fn = solve_fn or (lambda r, t, c: hjcd.solve(r, t, c, workspace=workspace))
    q, pe, oe, st = fn(robot, local_targets, cfg)
    rows = _all_gather_rows(pack(q, pe, oe, st), group)
    return unpack(rows, robot.dof)


def solve_sharded(robot: "hjcd.Robot", targets: torch.Tensor, cfg: "hjcd.hjcd_config", group=None,
                  workspace=None, solve_fn: Optional[Callable] = None):
    """Every rank holds all T targets; rank r solves its block and the blocks are
    all-gathered: the result equals a single-device solve of all T targets."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    T = targets.shape[0]
    start, count, block = partition(T, world, rank)
    local = targets[start:start + count]
    if count < block:   # pad with invalid rows (status 3, dropped after the gather)
        pad = torch.zeros((block - count, 7), dtype=targets.dtype, device=targets.device)
        local = torch.cat([local, pad])
    local = local.contiguous()
    c = type(cfg).from_buffer_copy(cfg)
    c.target_index_offset = int(cfg.target_index_offset) + start
    if block == 0:
        raise ValueError("no targets")
    q, pe, oe, st = solve_distributed(robot, local, c, group=group, workspace=workspace, solve_fn=solve_fn)
    return q[:T], pe[:T], oe[:T], st[:T]
