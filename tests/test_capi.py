"""C-ABI boundary checks that run without a GPU: the library loads, exports
every symbol include/iwpp_b200.h declares, and sizes workspaces."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "iwpp_b200.h")


@pytest.fixture(scope="module")
def lib():
    from paper_1209_3314_b200 import _lib, build
    build.build()
    return _lib.load_library()


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(iwpp_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    from paper_1209_3314_b200 import _lib
    assert sorted(_lib.EXPORTS) == _declared()


def test_library_exports_every_declared_symbol(lib):
    for name in _declared():
        assert hasattr(lib, name), name
        assert ctypes.cast(getattr(lib, name), ctypes.c_void_p).value


def test_version_and_workspace_sizes(lib):
    assert b"sm_100a" in lib.iwpp_version()
    r = lib.iwpp_recon_workspace_bytes(4096, 4096, 0, 8)
    assert 4096 < r < 64 << 20
    e = lib.iwpp_edt_workspace_bytes(4096, 4096, 8)
    assert e >= 5 * 4 * 4096 * 4096
    h = lib.iwpp_recon_host_workspace_bytes(4096, 4096, 2, 8)
    assert h >= 2 * 4 * 4096 * 4096


def test_sm100a_cubin_present():
    """The shared object carries sm_100a SASS (no PTX-JIT fallback)."""
    import shutil
    import subprocess
    from paper_1209_3314_b200 import build
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "--list-elf", build.LIB], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
