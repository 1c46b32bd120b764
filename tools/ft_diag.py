"""Fine-tune parity diagnostics (run on the B200): C1 (or a 2-layer family) through GpuEngine with records,
then per FT tick: policy / pi_ref log-probs of every pair (device vs fp32 oracle vs bf16 emulation) and the
per-tensor gradient rel-L2 of both against the fp32 oracle. Usage: python tools/ft_diag.py [n_ft_ticks]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import torch  # noqa: E402

from paper_2510_03283_b200.refpath import ensure_macesim  # noqa: E402

ensure_macesim()


def rel(a, b):
    return float((a.float() - b.float()).norm() / (b.float().norm() + 1e-30))


def main():
    from oracle.model_ref import TickOracle
    from paper_2510_03283_b200.build import build
    from paper_2510_03283_b200.config import selected_param_names
    from test_engine_c1_gpu import run_c1

    build()
    n_show = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    eng, res, w = run_c1(record=True)
    cfg, tcfg = eng.mcfg, eng.model.tcfg
    sel = selected_param_names(cfg, tcfg)
    orc = TickOracle(cfg, w, tcfg, sel)
    orb = TickOracle(cfg, w, tcfg, sel, emulate_bf16=True)
    shown = 0
    for rec in eng.records:
        b = rec["batch"]
        toks = rec["dec_tokens"] if rec["dec_tokens"] is not None else []
        _, ft = orc.run_tick(b, toks, rec["kept_post"])
        _, ftb = orb.run_tick(b, toks, rec["kept_post"])
        if ft is None:
            continue
        print(f"== tick {rec['tick']}: {len(b.ft_pairs)} pairs, T={b.T} ft0={b.ft0} R={b.ft_logit_rows.shape[0]}")
        for i, p in enumerate(b.ft_pairs):
            lo, lb = orc.ex.last_lp[i], orb.ex.last_lp[i]
            print(f"  pair {p.rid}: P={len(p.prompt)} nc={len(p.chosen)} nr={len(p.rejected)}"
                  f"  lp gpu {rec['ft_lp'][i]} ref_gpu {rec['ref_lp'][i]}"
                  f"  f32 ({lo[0]:.4f},{lo[1]:.4f}) ref ({lo[2]:.4f},{lo[3]:.4f})"
                  f"  emu ({lb[0]:.4f},{lb[1]:.4f})  loss gpu {rec['ft_loss'][i]:.6f} f32 {ft[0][i]:.6f}"
                  f" emu {ftb[0][i]:.6f}  margin gpu {rec['ft_margin'][i]:.5f} f32 {ft[1][i]:.5f} emu {ftb[1][i]:.5f}")
        for n in sel:
            g, go, gb = rec["grad"][n], ft[2][n], ftb[2][n]
            cos = float(torch.nn.functional.cosine_similarity(g.reshape(1, -1).float(), go.reshape(1, -1).float()))
            print(f"  grad {n:28s} gpu {rel(g, go):.3e} emu {rel(gb, go):.3e}  |g|/|go| {float(g.norm() / go.norm()):.4f}"
                  f" cos {cos:.5f}")
        for o in (orc, orb):
            o.ex.load_state(rec["master"], rec["adam_m"], rec["adam_v"])
        shown += 1
        if shown >= n_show:
            break


if __name__ == "__main__":
    main()
