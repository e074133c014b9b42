"""CPU-side checks of the C ABI (no GPU): the library builds, loads, exports
every entry point include/tcudb.h declares, and the ctypes mirrors of the ABI
structs match the C layout (sizeof / offsetof from a gcc-compiled probe)."""
import ctypes
import os
import re
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tcudb.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tcudb_[a-z_0-9]+)\s*\(", src)) - {"tcudb_alloc_fn", "tcudb_free_fn"})


def test_library_builds_and_exports_all_symbols():
    from paper_2112_07552_b200 import build
    lib_path = build.build()
    lib = ctypes.CDLL(lib_path)
    names = declared_functions()
    assert len(names) >= 9
    for n in names:
        assert hasattr(lib, n), f"{n} declared in tcudb.h but not exported"
    from paper_2112_07552_b200._lib import EXPORTS
    assert sorted(EXPORTS) == names


def test_sass_has_tcgen05_and_tma():
    """The GEMM object carries UTC*MMA (tcgen05.mma), UTMALDG (TMA) and LDTM (tcgen05.ld)."""
    from paper_2112_07552_b200 import build
    build.build()
    obj = os.path.join(ROOT, "paper_2112_07552_b200", "build", "gemm_tc.o")
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    assert "UTCIMMA" in sass and "UTCHMMA" in sass
    assert "UTMALDG" in sass and "LDTM" in sass
    assert "HMMA" not in re.sub(r"UTCHMMA", "", sass)  # no legacy mma.sync path


PROBE = r"""
#include <stdio.h>
#include <stddef.h>
#include "tcudb.h"
int main(void) {
  printf("col %zu %zu\n", sizeof(tcudb_col), offsetof(tcudb_col, type));
  printf("table %zu %zu %zu %zu\n", sizeof(tcudb_table), offsetof(tcudb_table, key), offsetof(tcudb_table, group),
         offsetof(tcudb_table, value));
  printf("query %zu\n", sizeof(tcudb_query));
  printf("result %zu %zu %zu\n", sizeof(tcudb_result), offsetof(tcudb_result, g_type), offsetof(tcudb_result, on_host));
  printf("stats %zu %zu %zu %zu %zu\n", sizeof(tcudb_stats), offsetof(tcudb_stats, G), offsetof(tcudb_stats, density_union),
         offsetof(tcudb_stats, ms_stats), offsetof(tcudb_stats, ms_total));
  return 0;
}
"""


def test_ctypes_layout_matches_header():
    from paper_2112_07552_b200 import _lib as L
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "probe.c")
        exe = os.path.join(d, "probe")
        open(c, "w").write(PROBE)
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe])
        out = dict((l.split()[0], list(map(int, l.split()[1:]))) for l in
                   subprocess.run([exe], capture_output=True, text=True).stdout.splitlines())
    assert out["col"] == [ctypes.sizeof(L.Col), L.Col.type.offset]
    assert out["table"] == [ctypes.sizeof(L.TableS), L.TableS.key.offset, L.TableS.group.offset, L.TableS.value.offset]
    assert out["query"] == [ctypes.sizeof(L.Query)]
    assert out["result"] == [ctypes.sizeof(L.Result), L.Result.g_type.offset, L.Result.on_host.offset]
    assert out["stats"] == [ctypes.sizeof(L.Stats), L.Stats.G.offset, L.Stats.density_union.offset,
                            L.Stats.ms_stats.offset, L.Stats.ms_total.offset]


def test_engine_fails_loudly_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2112_07552_b200 import Engine
    with pytest.raises(Exception):
        Engine(0)
