"""The C-ABI library loads and exports every symbol include/intfsim_b200.h
declares; the ctypes mirrors match the C struct layouts.  No compute (CPU)."""
import os
import re
import subprocess

import pytest

from paper_2512_18725_b200 import _abi, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "intfsim_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|int64_t) (intf_\w+)\(", text, flags=re.M)))


def test_library_is_built_for_sm100a():
    lib = build.build()
    out = subprocess.run(["cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_every_declared_symbol_is_exported():
    lib = _abi.load()
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) == set(_abi.SIGNATURES), set(syms) ^ set(_abi.SIGNATURES)
    assert lib.intf_abi_version() == 1


def test_struct_layouts_match_header(tmp_path):
    src = tmp_path / "sz.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "intfsim_b200.h"\n'
        "int main(){printf(\"%zu %zu %zu %zu %zu %zu %zu %zu\\n\", sizeof(intf_table), sizeof(intf_scenario),"
        " sizeof(intf_model), sizeof(intf_batch), sizeof(intf_replay_buffers), sizeof(intf_predictor),"
        " offsetof(intf_replay_buffers, seg_stride), offsetof(intf_scenario, seed));return 0;}\n"
    )
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    import ctypes

    want = [ctypes.sizeof(_abi.Table), ctypes.sizeof(_abi.Scenario), ctypes.sizeof(_abi.Model),
            ctypes.sizeof(_abi.Batch), ctypes.sizeof(_abi.ReplayBuffers), ctypes.sizeof(_abi.Predictor),
            _abi.ReplayBuffers.seg_stride.offset, _abi.Scenario.seed.offset]
    assert got == want


def test_bad_input_is_reported_not_crashing():
    lib = _abi.load()
    rc = lib.intf_replay(None, None, None, None)
    assert rc == 1 and "null" in _abi.last_error()


def test_hot_path_fails_loudly_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2512_18725_b200 as p

    with pytest.raises(RuntimeError, match="CUDA"):
        p.percentile([1.0, 2.0], 50)
