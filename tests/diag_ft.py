import sys; sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import torch
from test_engine_c1_gpu import run_c1
from oracle.model_ref import TickOracle
from paper_2510_03283_b200.config import selected_param_names
eng, res, w = run_c1(record=True)
cfg, tcfg = eng.mcfg, eng.model.tcfg
orc = TickOracle(cfg, w, tcfg, selected_param_names(cfg, tcfg))
for rec in eng.records[:40]:
    b = rec["batch"]
    toks = rec["dec_tokens"] if rec["dec_tokens"] is not None else []
    logits, ft = orc.run_tick(b, toks, rec["kept_post"])
    if b.n_dec:
        g = rec["dec_logits"]
        print("tick", rec["tick"], "n_dec", b.n_dec, "rel", ((g - logits).norm() / logits.norm()).item())
    if ft:
        print("FT tick", rec["tick"], "gpu lp", rec["ft_lp"].tolist(), "gpu ref", rec["ref_lp"].tolist())
        print("   oracle", orc.ex.last_lp)
        for n, go in ft[2].items():
            gg = rec["grad"][n]
            print("   grad", n, ((gg - go).norm() / (go.norm() + 1e-12)).item(), go.norm().item())
        orc.ex.load_state(rec["master"], rec["adam_m"], rec["adam_v"])
