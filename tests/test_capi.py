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


def test_ctypes_structs_match_the_header(tmp_path):
    """The ctypes mirrors in _lib.py have the C layout of the header's structs
    (size and every field offset, as gcc lays them out)."""
    import shutil
    import subprocess
    from paper_1209_3314_b200 import _lib
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    pairs = [("iwpp_recon_opts", _lib.ReconOpts), ("iwpp_stats", _lib.Stats),
             ("iwpp_edt_mg_slab", _lib.MgSlab)]
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "iwpp_b200.h"', "int main(void) {"]
    for cname, py in pairs:
        lines.append(f'  printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'  printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)],
                   check=True)
    got = dict(l.rsplit(" ", 1) for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                        check=True).stdout.splitlines())
    for cname, py in pairs:
        assert int(got[f"{cname} size"]) == ctypes.sizeof(py), cname
        for fname, _ in py._fields_:
            assert int(got[f"{cname} {fname}"]) == getattr(py, fname).offset, (cname, fname)
