"""Lockstep replicas through the real engine on CPU (gloo, world size 2): two GpuEngine replicas, each
with its own request stream (seed = base + rank) and a FakeModel device, run the same run_ticks protocol
bench.py runs under torchrun. Rank 1's trace is much shorter, so it drains first and must keep joining
the tick rounds idle. Checked: every rank sees the same sequence of (any FT, any active) agreements,
fine-tune updates happen on the same rounds on both ranks, the replicas' weights stay bit-identical, the
drained rank never blocks the other, and each replica's scheduler decisions equal a solo run of its own
trace (lockstep changes when updates happen, never what the reference decides)."""
import dataclasses
import json
import os

import torch.distributed as dist
import torch.multiprocessing as mp


def _solo_timeline(rank):
    from fakes import FakeModel
    from paper_2510_03283_b200.engine import GpuEngine

    wl = _workload(rank)
    fm = FakeModel(wl.model, wl.train, max_prompt_len=wl.max_prompt_len)
    eng = GpuEngine(*wl.engine_args(), model=fm, mode="P")
    eng.keep_outputs = False
    eng.run()
    return eng.timeline


def _workload(rank):
    from paper_2510_03283_b200.workloads import c1

    wl = c1(seed=rank)
    return dataclasses.replace(wl, trace_cfg=dataclasses.replace(wl.trace_cfg, duration=5.0 if rank == 0 else 1.0))


def _worker(rank, world, port, q):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).parent))
    sys.path.insert(0, str(Path(__file__).parents[1]))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from fakes import FakeModel
        from paper_2510_03283_b200.dist import Lockstep
        from paper_2510_03283_b200.engine import GpuEngine

        class LoggingLockstep(Lockstep):
            log: list = []

            def tick(self, local_ft, active=True):
                r = super().tick(local_ft, active)
                self.log.append(r)
                return r

        lock = LoggingLockstep(dist.group.WORLD, dist.group.WORLD)
        wl = _workload(rank)
        fm = FakeModel(wl.model, wl.train, max_prompt_len=wl.max_prompt_len)
        fm.pg = dist.group.WORLD
        eng = GpuEngine(*wl.engine_args(), model=fm, mode="P", lockstep=lock)
        eng.keep_outputs = False
        executed = []
        while True:  # bench.py's protocol: run_ticks(k) rounds, then agree whether anyone still has work
            executed.append(eng.run_ticks(7))
            if lock.max_over_ranks(float(executed[-1])) == 0.0:
                break
        q.put(dict(rank=rank, log=lock.log, executed=executed, idle=eng.idle_rounds, updates=fm.updates,
                   checksum=fm.weight_checksum(), timeline=json.dumps(eng.timeline, sort_keys=True, default=str)))
    except Exception as e:  # pragma: no cover - surfaced by the parent
        import traceback

        q.put(dict(rank=rank, error=traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def test_two_gpu_engine_replicas_lockstep_drain_safe():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(2):
        m = q.get(timeout=300)
        out[m["rank"]] = m
    for p in procs:
        p.join(60)
    for m in out.values():
        assert "error" not in m, m.get("error")
    a, b = out[0], out[1]
    assert a["log"] == b["log"], "ranks disagreed on a tick round"
    assert sum(a["executed"]) > sum(b["executed"]) and b["idle"] > 0, "rank 1 should drain first and idle"
    assert sum(a["executed"]) + a["idle"] == sum(b["executed"]) + b["idle"], "round counts differ"
    assert a["updates"] == b["updates"] > 0
    assert sum(1 for ft, _ in a["log"] if ft) == a["updates"]
    assert a["checksum"] == b["checksum"], "replica weights diverged"
    for r in (0, 1):  # lockstep never changes a replica's scheduler decisions
        assert out[r]["timeline"] == json.dumps(_solo_timeline(r), sort_keys=True, default=str)
