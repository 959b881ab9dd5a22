"""CPU checks of the product boundary: the C-ABI library builds, loads, and exports every symbol
that include/es.h declares (no compute calls without a GPU)."""
import ctypes
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def es():
    from tools.build import build_lib
    build_lib()
    import paper_2312_07874_b200 as es
    return es


def test_library_exports_every_declared_symbol(es):
    names = es.declared_symbols()
    assert len(names) >= 18
    lib = ctypes.CDLL(es.LIB_PATH)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", es.LIB_PATH], capture_output=True, text=True).stdout
    for n in names:
        assert f" T {n}" in out, n


def test_library_is_sm100a(es):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", es.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_oracle_not_linked_into_product(es):
    out = subprocess.run(["ldd", es.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle" not in out
    src = os.path.join(ROOT, "paper_2312_07874_b200")
    for dirpath, _, files in os.walk(src):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h", ".inc")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "oracle.h" not in txt and "liboracle" not in txt, f


def test_setup_rejects_bad_arguments_without_gpu(es):
    # argument validation happens before any CUDA call
    h = ctypes.c_void_p()
    rc = es.es_setup(ctypes.byref(h), None, 2, es.es_map_fn(0), None, None)
    assert rc == es.ES_ERR_ARG


def test_setup_rejects_unknown_interface_flux_without_gpu(es):
    # es_options.interface_flux outside {0, 1, 2, 3} is a configuration error, found before any CUDA call
    import numpy as np
    import es_inputs as I
    mesh = I.split_cartesian(2, 3, 1.0)
    ev = np.ascontiguousarray(mesh["elem_vertices"], np.int64)
    evx = np.ascontiguousarray(mesh["elem_vertex_coords"], np.float64)
    per = np.ascontiguousarray(mesh["period"], np.float64)
    m = es.es_mesh(2, len(ev), ev.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                   evx.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), per.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    for bad in (4, -1):
        o = es.es_options(1.4, bad, 0, 1, None, None, 0, 0, 0, 0)
        h = ctypes.c_void_p()
        rc = es.es_setup(ctypes.byref(h), ctypes.byref(m), 2, es.es_map_fn(0), None, ctypes.byref(o))
        assert rc == es.ES_ERR_CONFIG
        assert b"interface_flux" in es.es_last_error(h)
        es.es_destroy(h)


def test_struct_layouts_match_header(es, tmp_path):
    # the ctypes mirrors of es_mesh / es_options have the field offsets and sizes the C compiler gives
    # the declarations in include/es.h (an appended or reordered field breaks every caller silently)
    structs = {"es_mesh": es.es_mesh, "es_options": es.es_options}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "es.h"', "int main(void) {"]
    for name, py in structs.items():
        lines.append(f'  printf("{name} size %zu\\n", sizeof({name}));')
        for f, _ in py._fields_:
            lines.append(f'  printf("{name} {f} %zu\\n", offsetof({name}, {f}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c99", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = {}
    for ln in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines():
        s, f, v = ln.split()
        got[(s, f)] = int(v)
    for name, py in structs.items():
        assert got[(name, "size")] == ctypes.sizeof(py), name
        for f, _ in py._fields_:
            assert got[(name, f)] == getattr(py, f).offset, (name, f)
