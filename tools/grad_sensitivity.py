"""Is the GPU's fine-tune gradient error inherent to bf16 activations or a kernel defect?

For every fine-tune tick of a recorded GpuEngine run, compares the selected-parameter gradients of
  gpu   the B200 path (records),
  f32   the fp32 oracle (oracle/model_ref.py, same bf16-rounded weights, same pre-update state),
  b16   the same oracle with every GEMM / attention operand and output rounded to bf16 (fp32 residual stream,
        fp32 softmax / norms statistics: the numerics of the B200 kernels, emulated by torch autograd)
per tensor: rel-L2(gpu, f32), rel-L2(b16, f32), rel-L2(gpu, b16). If gpu~b16 << gpu~f32, the error is the
bf16 activation numerics, not the kernels.

    python tools/grad_sensitivity.py [c4|c3|c2|gpt2-2l|c1]
"""
import dataclasses
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import torch  # noqa: E402

from paper_2510_03283_b200.refpath import ensure_macesim  # noqa: E402

ensure_macesim()

import oracle.model_ref as mr  # noqa: E402


class Bf16Model(mr.OracleModel):
    def _lin(self, x, name, params):
        y = (x.to(torch.bfloat16) @ params[name + ".w"].to(torch.bfloat16).t()).float()
        if self.cfg.has_bias:
            y = y + params[name + ".b"]
        return y.to(torch.bfloat16).float()

    def _norm(self, x, name, params):
        return super()._norm(x, name, params).to(torch.bfloat16).float()

    def attention(self, q, K, V, mask):
        r = lambda t: t.to(torch.bfloat16).float()  # noqa: E731
        return r(super().attention(r(q), r(K), r(V), mask))

    def final(self, x, params=None):
        params = params or self.w
        h = self._norm(x, "final_norm", params)
        return h @ params["embed"].to(torch.bfloat16).float().t()


def scenario(name):
    from paper_2510_03283_b200.config import ModelConfig
    from paper_2510_03283_b200.workloads import c1, c2

    if name == "gpt2-2l":
        cfg = ModelConfig("gpt2-2l", "gpt2", 2, 768, 12, 12, 64, 3072, 50257, max_pos=1024)
        wl = c2(seed=5, arrival_rate=60.0, duration=4.0)
        wl = dataclasses.replace(wl, model=cfg, trace_cfg=dataclasses.replace(wl.trace_cfg, retrain_rate=0.3))
        return wl, 24, False
    if name == "c1":
        return c1(), 40, False
    from test_parity_shapes_gpu import _wl

    return _wl(name), 12, True


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    from paper_2510_03283_b200.config import selected_param_names
    from paper_2510_03283_b200.engine import GpuEngine
    from paper_2510_03283_b200.model import HybridModel
    from paper_2510_03283_b200.weights import init_weights

    torch.backends.cuda.matmul.allow_tf32 = False
    wl, ticks, until_mixed = scenario(name)
    cfg = wl.model
    w = init_weights(cfg, seed=0, device="cuda")
    model = HybridModel(cfg, wl.train, w, max_slots=512, max_prompt_len=wl.max_prompt_len,
                        max_decode_steps=wl.sched.max_decode_steps, prompt_groups=8192)
    eng = GpuEngine(*wl.engine_args(), model=model, mode="P", record=True)
    for _ in range(ticks):
        if eng.run_ticks(1) == 0:
            break
        b = eng.records[-1]["batch"]
        if until_mixed and b.n_dec and b.ft_pairs:
            break
    torch.cuda.synchronize()
    sel = selected_param_names(cfg, wl.train)
    f32 = mr.OracleExecutor(cfg, w, wl.train, sel, "cuda")
    b16 = mr.OracleExecutor(cfg, w, wl.train, sel, "cuda")
    bm = Bf16Model.__new__(Bf16Model)
    bm.__dict__.update(b16.model.__dict__)
    b16.model = bm
    for rec in eng.records:
        b = rec["batch"]
        if not b.ft_pairs:
            continue
        pairs = [(p.rid, p.prompt, p.chosen, p.rejected) for p in b.ft_pairs]
        lf, mf, gf = f32.dpo_step(pairs)
        lb, mb, gb = b16.dpo_step(pairs)
        print(f"tick {rec['tick']}: pairs {len(pairs)} loss gpu {list(map(float, rec['ft_loss']))} f32 {lf} b16 {lb}")
        print(f"   margin gpu {[round(float(x), 5) for x in rec['ft_margin']]} f32 {[round(x, 5) for x in mf]} "
              f"b16 {[round(x, 5) for x in mb]}")
        for n in sel:
            g = rec["grad"][n].cuda().float()
            rel = lambda a, c: float((a - c).norm() / (c.norm() + 1e-30))  # noqa: E731
            print(f"   {n:28s} gpu~f32 {rel(g, gf[n]):.3e}  b16~f32 {rel(gb[n], gf[n]):.3e}  gpu~b16 {rel(g, gb[n]):.3e}"
                  f"  |g| {float(gf[n].norm()):.3e}")
        for ex in (f32, b16):
            ex.load_state(rec["master"], rec["adam_m"], rec["adam_v"])


if __name__ == "__main__":
    main()
