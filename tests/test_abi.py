"""C-ABI boundary checks that need no GPU: libvplgi.so loads, exports every
symbol include/vplgi.h declares, and the host-only calls behave."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _declared():
    txt = (ROOT / "include/vplgi.h").read_text()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(vpl_[a-z_0-9]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    import paper_2203_11484_b200 as V
    from paper_2203_11484_b200 import build as B
    B.build()
    return V.load_library()


def test_header_declares_the_six_calls():
    d = _declared()
    for name in ["vpl_scene_upload", "vpl_build_bvh", "vpl_classify_near_far", "vpl_generate_vpls",
                 "vpl_render_gbuffer", "vpl_gather_indirect"]:
        assert name in d


def test_library_exports_every_declared_symbol(lib):
    import paper_2203_11484_b200 as V
    out = subprocess.run(["nm", "-D", "--defined-only", str(V.LIB_PATH)], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (vpl_\w+)", out))
    missing = [s for s in _declared() if s not in exported]
    assert not missing, missing
    assert sorted(V.EXPORTS) == _declared()
    for s in _declared():
        getattr(lib, s)


def test_library_is_sm100a_code(lib):
    import paper_2203_11484_b200 as V
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(V.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    assert "sm_100a" in out


def test_host_only_calls(lib):
    assert lib.vpl_abi_version() == 4
    assert lib.vpl_status_string(0) == b"ok"
    assert lib.vpl_status_string(-2) == b"buffer too small"
    n = C.c_size_t()
    assert lib.vpl_scene_bytes(1000, 4, C.byref(n)) == 0 and n.value > 1000 * 36
    assert lib.vpl_scene_bytes(0, 4, C.byref(n)) == -1            # EINVAL
    assert lib.vpl_scene_bytes(10, 0, C.byref(n)) == -1
    assert lib.vpl_scene_bytes(10, 65, C.byref(n)) == -1
    assert b"n_tris" in lib.vpl_last_error()
    assert lib.vpl_scene_upload(None, None, 10, None, 1, None, None, 0, None, None) == -1


def test_binding_has_no_cpu_fallback(tmp_path):
    import paper_2203_11484_b200 as V
    saved = V._lib
    V._lib = None
    try:
        with pytest.raises(ImportError):
            V.load_library(tmp_path / "missing.so")
    finally:
        V._lib = saved
