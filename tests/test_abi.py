"""The C ABI (include/ivk.h) without a GPU: libivk.so loads, exports every
declared entry point, the ctypes descriptor layouts match the C structs,
and argument validation fails loudly before any device work."""

import ctypes as C
import os
import re
import subprocess

import pytest

from harness import ROOT
from paper_2202_07381_b200 import _lib

HEADER = os.path.join(ROOT, "include", "ivk.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]*?\b(ivk_\w+)\s*\(", text, re.M)))


def test_library_builds_and_loads():
    from paper_2202_07381_b200 import _build
    if _build.needs_build():
        _build.build()
    lib = _lib.load()
    assert lib.ivk_version() >= 1


def test_every_declared_symbol_is_exported_and_bound():
    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 14
    for n in names:
        assert hasattr(lib, n), n
        assert n in _lib.EXPORTED, f"{n} has no ctypes prototype"


STRUCTS = {
    "ivk_operator_desc": _lib.OperatorDesc,
    "ivk_k1_tiles": _lib.K1Tiles,
    "ivk_patch_desc": _lib.PatchDesc,
    "ivk_kron_desc": _lib.KronDesc,
    "ivk_transfer_desc": _lib.TransferDesc,
    "ivk_coarse_desc": _lib.CoarseDesc,
    "ivk_quad_table": _lib.QuadTable,
    "ivk_convection_desc": _lib.ConvectionDesc,
    "ivk_general_desc": _lib.GeneralDesc,
    "ivk_mhd_desc": _lib.MHDDesc,
    "ivk_general_transfer_desc": _lib.GeneralTransferDesc,
    "ivk_modal_desc": _lib.ModalDesc,
    "ivk_peer_view": _lib.PeerView,
}


def test_struct_layouts_match_header(tmp_path):
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', 'int main(void){']
    for cname, py in STRUCTS.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-o", str(exe), str(src)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    got = {}
    for ln in out:
        if ln.strip():
            s, f, v = ln.split()
            got[(s, f)] = int(v)
    for cname, py in STRUCTS.items():
        assert got[(cname, "size")] == C.sizeof(py), cname
        for fname, _ in py._fields_:
            assert got[(cname, fname)] == getattr(py, fname).offset, (cname, fname)


def test_validation_errors_without_device():
    lib = _lib.load()
    rc = lib.ivk_stage_apply(None, None, None, None, None)
    assert rc == -1
    assert b"NULL" in lib.ivk_last_error()
    d = _lib.OperatorDesc()
    d.stages = 5
    d.n_nodes = d.n_p = 1
    assert lib.ivk_stage_apply(C.byref(d), None, None, None, None) == -1
    assert b"stages" in lib.ivk_last_error()
    with pytest.raises(_lib.IvkError):
        _lib.check(lib.ivk_patch_apply(None, None, None, None), "patch_apply")
    assert lib.ivk_coarse_solve(None, None, None, None) == -1
    assert lib.ivk_restrict(None, None, None, None) == -1


def test_no_cpu_fallback():
    import numpy as np
    import torch
    if torch.cuda.is_available():
        pytest.skip("CPU-only check")
    from harness import setup
    from paper_2202_07381_b200.stages import StageSystem
    disc, tab, conv, case = setup("crossed")
    S = StageSystem(disc.blocks[0], tab, 0.1, disc.cdofs[0])
    with pytest.raises(_lib.IvkError):
        S.matvec(np.zeros(S.dim))
