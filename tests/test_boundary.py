"""CPU suite: the C-ABI library builds for sm_100a, loads, and exports every
symbol include/slimsell_b200.h declares; the product path has no CPU fallback
and never reaches into oracle/. No compute calls here (no GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2010_09913_b200")


@pytest.fixture(scope="module")
def libpath():
    from paper_2010_09913_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        _lib.build()
    return _lib.LIB_PATH


def test_library_exports_header_symbols(libpath):
    from paper_2010_09913_b200 import _lib
    names = _lib.header_symbols()
    assert len(names) >= 20
    lib = ctypes.CDLL(libpath)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert lib.ssb_abi_version() == 2


def test_library_is_sm100a_only(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, arches


def test_no_cpu_fallback_in_product():
    """The product package must not import or execute the oracle."""
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h", ".hpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "liboracle" not in text and "libslimsell_ref" not in text, f


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    from paper_2010_09913_b200 import _lib
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "absent.so"))
    with pytest.raises(ImportError):
        _lib.lib()


def test_new_entry_points_reject_bad_arguments_without_a_device(libpath):
    """Round-2 entry points validate their arguments before touching a
    device: status codes and the thread-local message, as the rest of the ABI."""
    import numpy as np

    from paper_2010_09913_b200 import _lib as L
    lib = L.lib()
    EINVAL = L.SSB_EINVAL
    out = ctypes.c_void_p()
    ids = (ctypes.c_int * 9)(*([0] * 9))
    assert lib.ssb_ctx_create(0, ids, ctypes.byref(out)) == EINVAL
    assert lib.ssb_ctx_create(9, ids, ctypes.byref(out)) == EINVAL
    assert b"ranks" in lib.ssb_last_error()
    bounds = np.zeros(8, np.int64)
    cl = np.ones(4, np.int32)
    assert lib.ssb_partition_segments(cl.ctypes.data_as(L.i32p), 4, 32, 0, 1,
                                      bounds.ctypes.data_as(L.i64p)) == EINVAL
    assert lib.ssb_partition_segments(cl.ctypes.data_as(L.i32p), 4, 32, 1, 1, None) == EINVAL
    v = ctypes.c_int64()
    assert lib.ssb_validate_bfs_exact(None, None, 0, None, None, 0, ctypes.byref(v), None, 0) == EINVAL
    assert lib.ssb_sharded_bfs(None, 0, None, None, None, None, None, 0, None, None) == EINVAL
    assert lib.ssb_spmv_segment(None, 0, None, None, 0, 0, 0) == EINVAL
    assert lib.ssb_bfs_shard_front(None, 1, ctypes.byref(v)) == EINVAL
