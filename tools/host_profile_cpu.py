"""Host-path profile without a GPU: the real GpuEngine loop (mode P) over a stub model whose step() does no
device work, so the reference bookkeeping + batch building + scheduling can be timed and cProfiled here.
Usage: python tools/host_profile_cpu.py [c2|c3|c4] [--profile]"""
import cProfile
import pstats
import sys
import time
from pathlib import Path
from types import SimpleNamespace

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2510_03283_b200.engine import GpuEngine  # noqa: E402
from paper_2510_03283_b200.workloads import WORKLOADS  # noqa: E402


class StubModel:
    def __init__(self, cfg, max_slots, max_prompt_len, prompt_groups):
        self.cfg = cfg
        self.max_slots = max_slots
        self.maxpp = (max_prompt_len + 15) // 16
        self.prompt_groups = prompt_groups
        self.h2d_bytes = 0

    def step(self, batch, ft_global=None):
        return SimpleNamespace(dec_tokens=None, ref_lp=None, head_norm=None, ft_loss=None)

    def apply_trim(self, slots, kept):
        pass

    def release_slots(self, slots):
        pass


def main():
    name = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "c2"
    wl = WORKLOADS[name](seed=1)
    model = StubModel(wl.model, 1024, wl.max_prompt_len, (1 << 19) // 16)
    eng = GpuEngine(*wl.engine_args(), model=model, mode="P")
    eng.keep_outputs = False
    eng.run_ticks(wl.bench_skip)
    n = 32
    best = []
    for _ in range(6):  # min over windows: this container's CPU is shared and noisy
        t0 = time.perf_counter()
        eng.run_ticks(n)
        best.append(1e3 * (time.perf_counter() - t0) / n)
    print(f"{name}: host min {min(best):.3f} median {sorted(best)[3]:.3f} ms/tick (stub model, no device work)")
    if "--phases" in sys.argv:  # wall time per phase (wrapped methods; nested phases are included in parents)
        acc = {}

        def wrap(obj, name, label=None):
            f = getattr(obj, name)

            def g(*a, **k):
                t = time.perf_counter()
                try:
                    return f(*a, **k)
                finally:
                    acc[label or name] = acc.get(label or name, 0.0) + time.perf_counter() - t
            setattr(obj, name, g)
        for nm in ("_plan", "_execute", "build_batch", "_admit", "_maybe_evict_for_head", "_batch_head_stats",
                   "_exec_decode", "_exec_prefill", "_exec_ft", "_route_back", "_retire", "_estimate"):
            wrap(eng, nm)
        wrap(eng.queue, "refresh", "queue.refresh")
        wrap(eng.queue, "push", "queue.push")
        wrap(model, "step", "model.step")
        t0 = time.perf_counter()
        eng.run_ticks(n)
        tot = time.perf_counter() - t0
        print(f"phases over {n} ticks, total {1e3 * tot / n:.3f} ms/tick (timer overhead included)")
        for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
            print(f"  {k:24s} {1e3 * v / n:8.3f} ms/tick")
    if "--profile" in sys.argv:
        pr = cProfile.Profile()
        pr.enable()
        eng.run_ticks(n)
        pr.disable()
        pstats.Stats(pr).sort_stats("tottime").print_stats(30)


if __name__ == "__main__":
    main()
