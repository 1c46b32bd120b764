"""Run the REFERENCE's own test suite (/root/reference/pkg/tests, read-only, never copied) with the drop-in: every
engine the reference's tests build -- through their helpers (helpers.run_sim -> Engine(...)) or the package's
run_simulation (engine.py:788-800, the CLI's path) -- is a GpuEngine (mode P) over the CPU stand-in device
(tests/fakes.FakeModel: no kernels, the page manager and every device call recorded). The reference's assertions
(closed-form TTFT/TBT, conservation, determinism, policy behaviour, acceptance replays, CLI runs) are then checked
against the drop-in's bookkeeping.

Test infrastructure only (runs in the build container, where /root/reference exists). matplotlib is absent from
this image; the reference's report module needs only `matplotlib.use` / `rcParams` / `pyplot` at import, so a
minimal stub is put on the path for the CLI / acceptance tests (as SURVEY §8(c) describes).
    python tools/reference_suite_dropin.py [pytest args...]
"""
import os
import sys
import tempfile
import types
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
REF_TESTS = Path("/root/reference/pkg/tests")


def _matplotlib_stub(where: Path) -> None:
    pkg = where / "matplotlib"
    pkg.mkdir(parents=True, exist_ok=True)
    (pkg / "__init__.py").write_text("rcParams = {}\ndef use(*a, **k):\n    pass\n")
    # a figure records the labels of what is drawn on it and writes them into a minimal SVG on savefig
    (pkg / "pyplot.py").write_text(
        "_labels = []\n"
        "class _Ax:\n"
        "    def savefig(self, path, *a, **k):\n"
        "        body = ''.join('<text>%s</text>' % t for t in _labels)\n"
        "        open(path, 'w').write('<svg xmlns=\"http://www.w3.org/2000/svg\">' + body + '</svg>')\n"
        "        _labels.clear()\n"
        "    def __getattr__(self, name):\n"
        "        def f(*a, **k):\n"
        "            if k.get('label') is not None:\n"
        "                _labels.append(str(k['label']))\n"
        "            return _Ax()\n"
        "        return f\n"
        "    def __iter__(self):\n"
        "        return iter([_Ax(), _Ax()])\n"
        "def subplots(*a, **k):\n"
        "    n = k.get('nrows', a[0] if a else 1)\n"
        "    return _Ax(), ([_Ax() for _ in range(n)] if n > 1 else _Ax())\n"
        "def savefig(path, *a, **k):\n"
        "    _Ax().savefig(path)\n"
        "def __getattr__(name):\n"
        "    return _Ax().__getattr__(name)\n")


class DropInPlugin:
    """Installed before collection: macesim.engine.Engine -> a GpuEngine factory with the reference's signature."""

    def pytest_configure(self, config):
        sys.path.insert(0, str(ROOT))
        sys.path.insert(0, str(ROOT / "tests"))
        from paper_2510_03283_b200.refpath import ensure_macesim

        ensure_macesim()
        import macesim.engine as me
        from fakes import FakeModel
        from paper_2510_03283_b200.config import ModelConfig, TrainConfig
        from paper_2510_03283_b200.engine import GpuEngine

        class DropInEngine(GpuEngine):
            def __init__(self, trace, profile, sched_cfg, priority_params, cache_cfg, env, engine_cfg,
                         metrics_horizon=None):
                H = cache_cfg.num_heads
                cfg = ModelConfig("tiny-dropin", "llama", 2, 64 * H, H, H, 32, 256, 50000, max_pos=16384)
                model = FakeModel(cfg, TrainConfig(), max_slots=1 << 16, max_prompt_len=16384,
                                  prompt_groups=1 << 20)
                super().__init__(trace, profile, sched_cfg, priority_params, cache_cfg, env, engine_cfg,
                                 metrics_horizon, model=model, mode="P")
                self.keep_outputs = False

        me.Engine = DropInEngine
        self.engine_cls = DropInEngine


def main() -> int:
    import pytest

    if not REF_TESTS.exists():
        print("reference tests not present (only in the build container)")
        return 0
    tmp = Path(tempfile.mkdtemp(prefix="mace_ref_suite_"))
    _matplotlib_stub(tmp / "stub")
    sys.path.insert(0, str(tmp / "stub"))
    sys.path.insert(0, str(REF_TESTS))
    os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
    sys.dont_write_bytecode = True
    args = [str(REF_TESTS), "-q", "-p", "no:cacheprovider", "--rootdir", str(tmp)]
    args += sys.argv[1:]
    return pytest.main(args, plugins=[DropInPlugin()])


if __name__ == "__main__":
    sys.exit(main())
