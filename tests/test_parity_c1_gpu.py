"""C1 parity: every tick GpuEngine executed on the B200 (config C1, the whole 75-tick trace: prefill,
decode with pruned per-head windows, and 41 DPO fine-tune ticks) is replayed by the fp32 CPU oracle from
the same tick batch. Tolerances: tests/parity_util.py."""
import pytest

from parity_util import check_records
from test_engine_c1_gpu import run_c1

pytestmark = pytest.mark.gpu


def test_c1_every_tick_matches_oracle(ctx):
    eng, res, w = run_c1(record=True)
    st = check_records(eng, w, eng.mcfg, eng.model.tcfg, label="C1")
    assert st["tokens"] == 442
    assert st["ft_ticks"] > 0 and st["adamw_bit_exact"] == st["ft_ticks"]
