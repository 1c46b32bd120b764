"""Per-tick device time of the C2 bench window split by tick kind (with / without fine-tune rows):
replays the same recorded ticks with a CUDA event pair around each tick."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import restore, snapshot  # noqa: E402
from paper_2510_03283_b200.engine import GpuEngine  # noqa: E402
from paper_2510_03283_b200.model import HybridModel  # noqa: E402
from paper_2510_03283_b200.weights import init_weights  # noqa: E402
from paper_2510_03283_b200.workloads import WORKLOADS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
wl = WORKLOADS[name]()
cfg = wl.model
model = HybridModel(cfg, wl.train, init_weights(cfg, 0, "cuda"), max_slots=1024, max_prompt_len=wl.max_prompt_len,
                    max_decode_steps=wl.sched.max_decode_steps, prompt_groups=wl.kv_tokens // 16,
                    decode_pages=1024 * cfg.n_kv_heads * wl.decode_pages_per_head)
eng = GpuEngine(*wl.engine_args(), model=model, mode="P")
eng.keep_outputs = False
eng.run_ticks(wl.bench_skip + 5)
torch.cuda.synchronize()
snap = snapshot(model)
model.tape = []
eng.run_ticks(64)
tape, model.tape = model.tape, None
restore(model, snap)
model.replay(tape)
restore(model, snap)
torch.cuda.synchronize()
# group tape ops per tick: a "step" op starts a tick; trims / releases belong to the preceding step
ticks = []
for op in tape:
    if op[0] == "step":
        ticks.append([op])
    elif ticks:
        ticks[-1].append(op)
evs = []
dec_only = []  # (event pair, algorithmic HBM bytes) of ticks with decode rows only
KIND_PREFILL = 0
for ops in ticks:
    bt = ops[0][1]
    pure = bt.n_dec > 0 and not bt.ft_pairs and not (bt.seqs[:, 0] == KIND_PREFILL).any()
    byts = model.decode_attn_bytes(bt) * cfg.n_layers if pure else 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    model.replay(ops)
    e1.record()
    evs.append((e0, e1, bool(bt.ft_pairs), bt))
    if pure:
        dec_only.append((e0, e1, byts, bt.n_dec))
torch.cuda.synchronize()
if dec_only:
    import json as _json
    hbm = _json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    wbytes = 2 * sum(v.numel() for k, v in model.w.items() if k != "pos_emb")  # every weight streamed once
    ms = np.array([a.elapsed_time(b) for a, b, _, _ in dec_only])
    roof = np.array([(wbytes + kv) / (hbm * 1e9) * 1e3 for _, _, kv, _ in dec_only])
    print(f"decode-only ticks {len(dec_only)}: mean {ms.mean():.3f} ms, rows {np.mean([r for *_, r in dec_only]):.0f}, "
          f"HBM roofline (weights + KV once) {roof.mean():.3f} ms -> frac {float((roof / ms).mean()):.3f}")
ft = [a.elapsed_time(b) for a, b, f, _ in evs if f]
nf = [a.elapsed_time(b) for a, b, f, _ in evs if not f]
print(f"{name}: {len(evs)} ticks; FT ticks {len(ft)} mean {np.mean(ft) if ft else 0:.3f} ms; "
      f"non-FT ticks {len(nf)} mean {np.mean(nf) if nf else 0:.3f} ms; total {sum(ft) + sum(nf):.1f} ms")
b = [x[3] for x in evs]
print("rows/tick mean", np.mean([x.total_tokens for x in b]), "decode rows mean", np.mean([x.n_dec for x in b]),
      "FT rows on FT ticks", np.mean([x.T - x.ft0 for x in b if x.ft_pairs]) if ft else 0)
