"""The C-ABI library builds, loads and exports exactly what include/lsk.h declares.

No compute calls here (no GPU in the build container): only symbol presence,
signature bookkeeping and the pure-host helpers.
"""

import os
import re
import subprocess


from conftest import ROOT
from paper_2605_00837_b200 import _lib

HEADER = os.path.join(ROOT, "include", "lsk.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lsk_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (lsk_\w+)$", out, flags=re.M))
    for name in declared():
        assert name in exported, name
        assert hasattr(lib, name)


def test_ctypes_signatures_cover_header():
    assert sorted(_lib.SIGNATURES) == declared()


def test_no_torch_types_in_abi():
    src = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    for bad in ("torch", "at::", "Tensor", "c10"):
        assert bad not in src


def test_pure_host_helpers():
    lib = _lib.load()
    assert lib.lsk_version() >= 1
    assert lib.lsk_solve_dense_max_cols() == 8192
    assert lib.lsk_trace_capacity(200, 10) == 21
    assert lib.lsk_trace_capacity(25, 10) == 4
    assert lib.lsk_update_beta_workspace_bytes(1, 1) > 0
    assert lib.lsk_build_cost_workspace_bytes() > 0


def test_sm100a_cubin_present():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_packed_solver_sass():
    """The dense kernels run the packed f32x2 path (FADD2/FFMA2) and MUFU ex2;
    bitwise freedom from FMA contraction is proven on the GPU
    (tests/test_gpu_parity.py::test_argument_build_bitwise)."""
    out = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    body, keep = [], False
    for ln in out.splitlines():
        if "Function :" in ln:
            keep = "k_solve_dense" in ln
        elif keep:
            body.append(ln)
    text = "\n".join(body)
    for op in ("FADD2", "FFMA2", "MUFU.EX2", "UBLKCP"):
        assert re.search(r"\b" + re.escape(op) + r"\b", text), op
