"""Multi-replica lockstep on CPU with gloo (world_size 2): the FT flag agreement and the gradient
exchange keep replicas bit-identical even when only one replica has fine-tune rows in a tick."""
import os

import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.model_ref import adamw_reference
    from paper_2510_03283_b200.dist import Lockstep

    lock = Lockstep(dist.group.WORLD, dist.group.WORLD)
    torch.manual_seed(0)
    p = torch.randn(64)
    m, v = torch.zeros(64), torch.zeros(64)
    step = 0
    has_ft_by_tick = [[True, False], [False, False], [False, True], [True, True]]
    for t, flags in enumerate(has_ft_by_tick):
        local = flags[rank]
        if lock.any_ft(local) != any(flags):
            q.put(("flag mismatch", rank, t))
        if any(flags):
            g = torch.full((64,), float(rank + 1 + t)) if local else torch.zeros(64)
            dist.all_reduce(g, group=lock.grad_group)   # HybridModel.apply_update's exchange
            step += 1
            adamw_reference(p, m, v, g, 1e-3, 0.9, 0.999, 1e-8, 0.0, 1 - 0.9 ** step, 1 - 0.999 ** step)
    assert lock.max_over_ranks(float(rank)) == world - 1
    assert lock.sum_over_ranks(1.0) == world
    q.put(("p", rank, p.numpy().tobytes()))
    dist.destroy_process_group()


def test_lockstep_two_replicas_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    msgs = [q.get() for _ in range(2)]
    assert all(m[0] == "p" for m in msgs), msgs
    assert msgs[0][2] == msgs[1][2], "replicas diverged"
