"""Multi-GPU plumbing for the hybrid iteration.

One process per GPU, each with its own GpuEngine over its own request stream (seed = base + rank)
and a replica of the model. The only data-path collective is the NCCL all-reduce of the selected
parameters' gradients, once per tick in which ANY replica runs fine-tune rows (HybridModel.apply_update).
Whether a tick is such a tick is agreed on the host over a gloo group (a 4-byte CPU all-reduce), so
the device stream never stalls for a flag.
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


class Lockstep:
    def __init__(self, flag_group=None, grad_group=None):
        self.flag_group = flag_group
        self.grad_group = grad_group

    @property
    def active(self) -> bool:
        return self.flag_group is not None

    def any_ft(self, local: bool) -> bool:
        if self.flag_group is None:
            return local
        t = torch.tensor([1 if local else 0], dtype=torch.int32)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.flag_group)
        return bool(t.item())

    def barrier(self) -> None:
        if self.flag_group is not None:
            dist.barrier(group=self.flag_group)

    def max_over_ranks(self, value: float) -> float:
        if self.flag_group is None:
            return value
        t = torch.tensor([value], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.flag_group)
        return float(t.item())

    def sum_over_ranks(self, value: float) -> float:
        if self.flag_group is None:
            return value
        t = torch.tensor([value], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.flag_group)
        return float(t.item())


def init_from_env(device_backend: str = "nccl") -> tuple[int, int, Lockstep]:
    """(rank, world, lockstep) from torchrun's env; world 1 -> no process groups."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world == 1:
        return 0, 1, Lockstep()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group(backend=device_backend)
    flag = dist.new_group(backend="gloo")
    grad = dist.group.WORLD if device_backend == "nccl" else flag
    return rank, world, Lockstep(flag, grad)
