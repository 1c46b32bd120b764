"""KV allocator safety on the B200: the device free-stack top always equals the host mirror's count
(kvmanager.DecodePageMirror), and a decode pool too small for the trace raises KvCapacityError before
the tick launches -- the device status word never records a pop from an empty stack."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def _engine(decode_pages):
    from paper_2510_03283_b200.engine import GpuEngine
    from paper_2510_03283_b200.model import HybridModel
    from paper_2510_03283_b200.weights import init_weights
    from paper_2510_03283_b200.workloads import c1

    wl = c1()
    w = init_weights(wl.model, seed=0)
    model = HybridModel(wl.model, wl.train, w, max_slots=64, max_prompt_len=wl.max_prompt_len, prompt_groups=512,
                        decode_pages=decode_pages)
    return GpuEngine(*wl.engine_args(), model=model, mode="P"), model


def test_device_stack_matches_host_mirror(ctx):
    eng, model = _engine(None)
    for _ in range(6):
        eng.run_ticks(10)
        torch.cuda.synchronize()
        top, status = model.kv_status()
        assert status == 0
        assert top == model.kv_mirror.free
    base = model.dec_base.cpu().numpy()
    assert (base == model.kv_mirror.base[: base.shape[0]]).all()


def test_exhausted_decode_pool_raises_before_launch(ctx):
    from paper_2510_03283_b200.kvmanager import KvCapacityError

    eng, model = _engine(decode_pages=8 * 3)  # room for three decode rings of 8 KV heads
    with pytest.raises(KvCapacityError):
        eng.run_ticks(75)
    torch.cuda.synchronize()
    top, status = model.kv_status()
    assert status == 0, "a device pop hit the empty stack"
    assert top == model.kv_mirror.free >= 0
