"""The C-ABI library loads and exports every symbol include/pcgpu.h declares
(no compute calls: runs without a GPU)."""
import ctypes
import os
import re

import pytest

from paper_1912_03744_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "pcgpu.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pcgpu_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_header_symbols():
    lib = N.load()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(N.EXPORTS) == syms


def test_abi_version_and_struct_sizes():
    lib = N.load()
    assert lib.pcgpu_abi_version() == N.PCGPU_ABI_VERSION
    # ctypes mirrors of the C structs: natural alignment on x86-64
    assert ctypes.sizeof(N.Table) == 24
    assert ctypes.sizeof(N.Outcome) == 16
    assert ctypes.sizeof(N.StepResultC) == 48


def test_create_rejects_invalid_config_without_gpu():
    # validation happens before any CUDA call (solver.cpp:33-42 semantics)
    from paper_1912_03744_b200 import configs
    from paper_1912_03744_b200.desc import build_desc
    from paper_1912_03744_b200.source import NullSource
    case = configs.step_cell(True)
    case.solver.max_iter = 0
    d, keep = build_desc(case.grid(), case.materials, NullSource(), case.timing, case.solver)
    h = ctypes.c_void_p()
    assert N.load().pcgpu_create(ctypes.byref(d), ctypes.byref(h)) == N.ERR_CONFIG
    assert b"max_iter" in N.load().pcgpu_last_error(None)


def test_oracle_libraries_load():
    from oracle import oracle as O
    if O.port_available():
        O._load_port()
    if O.ref_available():
        O._load_ref()
