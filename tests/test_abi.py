"""C-ABI contract checks that need no GPU: the library loads, exports every
symbol include/nw.h declares, and fails loudly (NW_E_CUDA) without a device."""
from __future__ import annotations

import ctypes
import os
import re
import subprocess

import pytest

import paper_2412_21103_b200 as nwb
from paper_2412_21103_b200 import nw as nwmod

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "nw.h")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(nw_[a-z_]+)\s*\(", txt)))


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for name in ("nw_align_pair", "nw_align_batch", "nw_score_only", "nw_traceback"):
        assert name in syms


def test_library_exports_every_declared_symbol():
    lib = nwb.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", nwmod.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r"\bT (nw_\w+)", out))
    assert set(declared_symbols()) <= exported
    assert set(nwmod.EXPORTED) == set(declared_symbols())


def test_library_is_sm100a_native():
    out = subprocess.run(["cuobjdump", "--list-elf", nwmod.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", nwmod.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "VIMNMX" in sass  # DPX max (north_star: DPX intrinsics)


def test_strerror_and_no_device_behaviour():
    lib = nwb.lib()
    assert lib.nw_strerror(0) == b"ok"
    assert lib.nw_strerror(2) == b"residue not in alphabet"
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("device present")
    except Exception:
        pass
    h = ctypes.c_void_p()
    assert lib.nw_ctx_create(0, None, ctypes.byref(h)) == nwmod.NW_E_CUDA
    with pytest.raises(nwb.NWError):
        nwb.Context(0)


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2412_21103_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f), errors="replace").read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "nw_oracle" not in txt, f


def test_batch_ops_offsets_host_helper():
    import numpy as np
    offs = np.array([0, 3, 5, 9], dtype=np.int64)
    oo = nwb.nw_batch_ops_offsets(offs, None)
    # pairs (0,1) (0,2) (1,2): (3+2) (3+4) (2+4)
    assert oo.tolist() == [0, 5, 12, 18]
    oo = nwb.nw_batch_ops_offsets(offs, np.array([[2, 0]], dtype=np.int32))
    assert oo.tolist() == [0, 7]
