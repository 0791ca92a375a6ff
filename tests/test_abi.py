"""CPU-side checks of the boundary: the C-ABI library builds, loads without a
GPU, and exports every entry point include/tds.h declares.  No compute calls."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_1410_2698_b200 as tds
from paper_1410_2698_b200 import build as tbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    tbuild.build()
    return tds.load_library()


def header_functions():
    src = open(os.path.join(ROOT, "include", "tds.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tds_[a-z_]+)\s*\(", src)))


def test_header_declares_the_abi():
    fns = header_functions()
    assert set(fns) == set(tds.ABI_SYMBOLS), fns
    for name in ("tds_build_index", "tds_search", "tds_fetch_results"):   # north star names
        assert name in fns


def test_library_exports_every_symbol(lib):
    for name in header_functions():
        assert hasattr(lib, name), name
    assert lib.tds_version().decode().startswith("tds-b200")


def test_exports_are_extern_c():
    out = os.popen(f"nm -D --defined-only {tbuild.LIB}").read()
    for name in header_functions():
        assert re.search(rf"\bT {name}$", out, flags=re.M), name


def test_arch_is_sm_100a():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {tbuild.LIB}").read()
    assert "sm_100a" in out


def test_null_arguments_fail_cleanly(lib):
    # argument checks run before any device work
    out = ctypes.c_void_p()
    assert lib.tds_build_index(None, 0, None, None, ctypes.byref(out)) == 1
    assert b"NULL" in lib.tds_last_error() or b"n == 0" in lib.tds_last_error()
    assert lib.tds_search(None, 1, None, 0, 1.0, 0.0, 1.0, 0, None, ctypes.byref(out), None) == 1
    st = tds._Stats()
    assert lib.tds_result_stats(None, ctypes.byref(st)) == 1
    assert lib.tds_result_count(None) == 0


def test_no_oracle_import_in_product():
    pkg = os.path.join(ROOT, "paper_1410_2698_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "tds_oracle" not in txt, f


def test_struct_layouts_match_the_header(tmp_path):
    """The binding's ctypes mirrors of tds_stats / tds_search_req /
    tds_index_params have the header's sizes and field offsets (gcc)."""
    import ctypes
    src = tmp_path / "layout.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "tds.h"\n'
        'int main(void){printf("%zu %zu %zu %zu %zu %zu %zu\\n", sizeof(tds_stats), offsetof(tds_stats, ms_schedule),'
        ' offsetof(tds_stats, kind), offsetof(tds_stats, pair_tests_alt), sizeof(tds_search_req),'
        ' offsetof(tds_search_req, stream), sizeof(tds_index_params)); return 0;}\n')
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)])
    got = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    S, R, P = tds._Stats, tds._SearchReq, tds._Params
    want = [ctypes.sizeof(S), S.ms_schedule.offset, S.kind.offset, S.pair_tests_alt.offset, ctypes.sizeof(R),
            R.stream.offset, ctypes.sizeof(P)]
    assert got == want
