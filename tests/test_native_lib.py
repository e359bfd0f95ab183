"""The C-ABI library loads without a GPU and exports every symbol
include/podcg.h declares; struct layouts agree between C and ctypes."""

import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "podcg.h")


def _declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rk_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = _declared()
    for required in ("rk_spmv", "rk_spmm", "rk_pcg_steps", "rk_pcg_entry", "rk_gram", "rk_gemm_nn", "rk_gemv_t",
                     "rk_gemv_n", "rk_csr_diagonal", "rk_csr_asymmetry", "rk_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_1512_05820_b200 import _native

    lib = _native.load_library()
    for name in _declared():
        assert hasattr(lib, name), name
    assert set(_declared()) == set(_native.EXPORTED_SYMBOLS)


def test_struct_layouts_match_c(tmp_path):
    from paper_1512_05820_b200 import _native

    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "podcg.h"\n'
                   'int main(){printf("%zu %zu %zu %zu %zu %d\\n", sizeof(rk_pcg_plan), sizeof(rk_pcg_state),'
                   ' sizeof(rk_csr), offsetof(rk_pcg_plan, mode), offsetof(rk_pcg_plan, st), RK_PCG_TICKETS);'
                   'return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    got = [ctypes.sizeof(_native.RkPcgPlan), ctypes.sizeof(_native.RkPcgState), ctypes.sizeof(_native.RkCsr),
           _native.RkPcgPlan.mode.offset, _native.RkPcgPlan.st.offset, _native.PCG_TICKETS]
    assert list(map(int, out)) == got


def test_library_is_built_for_sm100a_only():
    so = os.path.join(ROOT, "paper_1512_05820_b200", "_lib", "libpodcg.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    assert "DMMA" in sass          # fp64 tensor-core path for the Gram / reconstruction
    assert "LDGSTS" in sass        # cp.async staging


def test_device_entry_points_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_1512_05820_b200 as pk
    from paper_1512_05820_b200._native import NativeUnavailable

    with pytest.raises(NativeUnavailable):
        pk.SparseSpdMatrix.identity(3)
