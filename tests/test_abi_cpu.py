"""The C-ABI library loads without a GPU and exports every symbol include/mace_b200.h declares."""
import ctypes
import re
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "mace_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*|long long)\s+(mace_\w+)\s*\(", text, re.M)))


def test_header_symbols_exported_and_bound():
    from paper_2510_03283_b200._lib import SIGNATURES, lib
    from paper_2510_03283_b200.build import build

    build()
    L = lib()
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(L, s), f"{s} declared in include/mace_b200.h but not exported"
        assert s in SIGNATURES, f"{s} has no ctypes binding"
    assert L.mace_version() >= 1


def test_no_gpu_means_loud_failure():
    import torch

    from paper_2510_03283_b200._lib import Ctx, MaceError

    if torch.cuda.is_available():
        return
    try:
        Ctx(0)
    except MaceError as e:
        assert "sm_100" in str(e)
    else:
        raise AssertionError("ctx creation must fail without a B200")


def test_product_never_imports_oracle():
    for p in (ROOT / "paper_2510_03283_b200").glob("*.py"):
        assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", p.read_text(), re.M), p


def test_ctypes_struct_layouts_match_the_header(tmp_path):
    """Every ctypes mirror of a header struct has the C compiler's size and field offsets (gcc here)."""
    import subprocess

    from paper_2510_03283_b200 import _lib

    structs = [_lib.MaceGemmArgs, _lib.MaceKvLayout, _lib.MaceAttnArgs, _lib.MaceLayerWeights, _lib.MaceLayerGrads,
               _lib.MaceModelDesc, _lib.MaceSavedActs, _lib.MaceTickBuffers, _lib.MaceTickDesc, _lib.MaceLoraLayer]
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "mace_b200.h"', "int main(void) {"]
    expect = []
    for st in structs:
        n = st.__name__
        lines.append(f'  printf("%zu\\n", sizeof({n}));')
        expect.append(ctypes.sizeof(st))
        for f, _ in st._fields_:
            lines.append(f'  printf("%zu\\n", offsetof({n}, {f}));')
            expect.append(getattr(st, f).offset)
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    assert got == expect
