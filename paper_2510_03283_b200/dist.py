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

    def tick(self, local_ft: bool, active: bool = True) -> tuple[bool, bool]:
        """The per-tick agreement, ONE 8-byte gloo all-reduce(max): (any replica has FT rows, any replica still
        has work). Every rank calls it exactly once per tick round -- an executed tick, or an idle round of a
        rank whose trace has drained (GpuEngine.run_ticks) -- so the rounds pair up in order and a drained
        rank never leaves the others blocked."""
        if self.flag_group is None:
            return local_ft, active
        t = torch.tensor([1 if local_ft else 0, 1 if active else 0], dtype=torch.int32)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.flag_group)
        return bool(t[0].item()), bool(t[1].item())

    def any_ft(self, local: bool) -> bool:
        return self.tick(local, True)[0]

    def min_over_ranks(self, value: float) -> float:
        return -self.max_over_ranks(-value)

    def assert_equal(self, value: int, what: str) -> None:
        """Cross-replica check (e.g. the weight checksum after every k fine-tune updates): raises on every rank
        when any two ranks disagree."""
        if self.flag_group is None:
            return
        t = torch.tensor([value, -value], dtype=torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.flag_group)
        if int(t[0]) != -int(t[1]):
            raise RuntimeError(f"replicas diverged: {what} differs across ranks ({int(t[0])} vs {-int(t[1])})")

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
