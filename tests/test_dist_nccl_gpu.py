"""The N>1 data path on a real GPU (the sandbox has one B200): a world-size-1 NCCL process group drives the same
code the 8-GPU run uses -- GpuEngine in lockstep (the gloo flag group agrees on fine-tune ticks), the gradient
exchange through torch.distributed.all_reduce on the device tensors (bf16 and fp32 modes), the masked AdamW after
it. With one rank the all-reduce is the identity, so the fp32 exchange must leave every master weight and Adam
moment bit-identical to the run without a process group; the bf16 exchange rounds the gradient once
and must stay within that rounding. Runs in a spawned process so the process group does not leak into other tests."""
import os
import socket

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(mode, q):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).parent))
    sys.path.insert(0, str(Path(__file__).parents[1]))
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2510_03283_b200.dist import Lockstep
    from paper_2510_03283_b200.engine import GpuEngine
    from paper_2510_03283_b200.model import HybridModel
    from paper_2510_03283_b200.weights import init_weights
    from paper_2510_03283_b200.workloads import c1

    torch.cuda.set_device(0)
    pg = lock = None
    if mode != "none":
        dist.init_process_group("nccl", rank=0, world_size=1)
        lock = Lockstep(dist.new_group(backend="gloo"), dist.group.WORLD)
        pg = dist.group.WORLD
    wl = c1()
    model = HybridModel(wl.model, wl.train, init_weights(wl.model, seed=0), max_slots=256,
                        max_prompt_len=wl.max_prompt_len, prompt_groups=2048, process_group=pg,
                        grad_allreduce="f32" if mode == "f32" else "bf16")
    eng = GpuEngine(*wl.engine_args(), model=model, mode="P", lockstep=lock)
    eng.run_ticks(40)
    torch.cuda.synchronize()
    q.put((mode, model.adam_step, model.master.cpu().numpy().copy(), model.m.cpu().numpy().copy(),
           sum(len(v) for v in eng.decoded_tokens().values())))
    if mode != "none":
        dist.destroy_process_group()


def test_nccl_gradient_exchange_world1():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    out = {}
    for mode in ("none", "f32", "bf16"):
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(_free_port())
        p = ctx.Process(target=_run, args=(mode, q))
        p.start()
        r = q.get(timeout=600)
        p.join(timeout=120)
        assert p.exitcode == 0, f"{mode} run failed"
        out[r[0]] = r[1:]
    import numpy as np

    steps, master, m, toks = out["none"]
    assert steps > 0, "no fine-tune update in the window"
    s32, master32, m32, toks32 = out["f32"]
    assert s32 == steps and toks32 == toks
    assert np.array_equal(master32.view(np.int32), master.view(np.int32)), "fp32 exchange changed the masters"
    assert np.array_equal(m32.view(np.int32), m.view(np.int32))
    s16, master16, _, _ = out["bf16"]
    assert s16 == steps
    # one bf16 rounding of each step's gradient moves each AdamW step by a fraction of lr: bounded by 2 lr per step
    from paper_2510_03283_b200.workloads import c1

    lr = c1().train.lr
    assert np.isfinite(master16).all() and np.abs(master - master16).max() <= 2 * lr * steps
