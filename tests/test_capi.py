"""The C-ABI library loads without a GPU and exports every declared symbol;
the ctypes mirrors of the descriptor structs match the C layout."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_2102_09811_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "heatbem_b200.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char \*)\s*(hb_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_what_python_binds():
    assert sorted(_native.EXPORTED) == declared()


def test_library_exports_every_declared_symbol():
    L = _native.load()
    for name in declared():
        assert hasattr(L, name), name
    assert L.hb_version() == 1000
    assert L.hb_last_error() is not None


def test_struct_layout_matches_c(tmp_path):
    prog = tmp_path / "sz.c"
    prog.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "heatbem_b200.h"\n'
                    'int main(void){printf("%zu %zu %zu %zu\\n", sizeof(hb_mesh_desc), sizeof(hb_assembly_desc),'
                    ' offsetof(hb_mesh_desc, star_max), offsetof(hb_assembly_desc, workspace_bytes));return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(prog), "-o", str(exe)])
    a, b, c, d = map(int, subprocess.check_output([str(exe)]).split())
    assert a == ctypes.sizeof(_native.MeshDesc) and b == ctypes.sizeof(_native.AssemblyDesc)
    assert c == _native.MeshDesc.star_max.offset and d == _native.AssemblyDesc.workspace_bytes.offset


def test_invalid_arguments_return_error_codes_without_gpu():
    """Argument validation happens before any CUDA call: null descriptors,
    unsupported combinations and bad sizes come back as codes + messages."""
    L = _native.load()
    assert L.hb_assemble(None, None, None) == -1
    m, a = _native.MeshDesc(), _native.AssemblyDesc()
    a.op, a.test_p1, a.trial_p1, a.symmetric = 1, 1, 1, 1
    assert L.hb_assemble(ctypes.byref(m), ctypes.byref(a), None) == -4
    assert b"unsupported" in L.hb_last_error()
    a.op, a.test_p1, a.trial_p1, a.symmetric = 0, 0, 0, 1
    a.E_t, a.d_begin, a.d_end = 4, 0, 8
    assert L.hb_assemble(ctypes.byref(m), ctypes.byref(a), None) == -1
    assert L.hb_toeplitz_apply(0, 1, 1, None, 0, 0, 1, None, None, None) == -1
