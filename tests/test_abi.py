"""C-ABI boundary checks that need no GPU (-m "not gpu"): the library builds/loads, exports every
symbol include/linr.h declares, and host-side validation behaves as documented."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "linr.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|size_t|void|const char\s*\*)\s*\*?\s*(linr_\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def L():
    import paper_2407_13218_b200.build as b
    b.build()
    from paper_2407_13218_b200 import linr
    return linr.library()


def test_exports_every_declared_symbol(L):
    names = declared_functions()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    from paper_2407_13218_b200 import linr
    assert set(names) == set(linr.ABI_FUNCTIONS)


def test_version_and_error_string(L):
    assert L.linr_version() == 2
    assert isinstance(L.linr_last_error(), bytes)


def test_storage_bytes_host_only(L):
    from paper_2407_13218_b200.linr import _Desc
    d = _Desc(1000, 0, 128, 2, 1, 0, None, None, None)
    emb = L.linr_storage_bytes(ctypes.byref(d), 0)
    attr = L.linr_storage_bytes(ctypes.byref(d), 1)
    live = L.linr_storage_bytes(ctypes.byref(d), 2)
    assert emb == 1024 * 128 * 2          # capacity padded to a multiple of 256 rows
    assert attr == 1024 * 8
    assert live == 256 + 1024 // 8
    bad = _Desc(1000, 0, 100, 2, 1, 0, None, None, None)   # dim not a multiple of 16
    assert L.linr_storage_bytes(ctypes.byref(bad), 0) == 0
    bad = _Desc(10, 0xFFFFFFFF - 5, 64, 0, 1, 0, None, None, None)   # ids beyond 2^32-1
    assert L.linr_storage_bytes(ctypes.byref(bad), 0) == 0


def test_validation_without_gpu(L):
    out = ctypes.c_void_p()
    assert L.linr_index_create(None, ctypes.byref(out)) == -1
    assert L.linr_search(None, None, 1, 1, None, None, 10, None, 0, None, None, None, None) == -1
    assert b"null" in L.linr_last_error()
    assert L.linr_merge_keys(None, None, 1, 1, 1, None, 0, None, None, None, None) == -1
    assert L.linr_search_workspace_bytes(None, 1, 1, 10) == 0


def test_oracle_and_product_share_no_code():
    """The oracle and the CUDA library are independent (task rule: no shared code or headers)."""
    osrc = open(os.path.join(ROOT, "oracle", "linr_oracle.cpp")).read()
    includes = re.findall(r"#include\s*[<\"]([^>\"]+)", osrc)
    assert all("linr" not in i and "csrc" not in i for i in includes), includes
    for f in os.listdir(os.path.join(ROOT, "paper_2407_13218_b200", "csrc")):
        inc = re.findall(r"#include\s*[<\"]([^>\"]+)", open(os.path.join(ROOT, "paper_2407_13218_b200", "csrc", f)).read())
        assert all("oracle" not in i for i in inc), (f, inc)
    for f in ("__init__.py", "linr.py", "sharded.py"):
        txt = open(os.path.join(ROOT, "paper_2407_13218_b200", f)).read()
        assert "import oracle" not in txt and "from oracle" not in txt
