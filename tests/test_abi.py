"""C-ABI boundary checks that need no GPU: libvca.so builds for sm_100a,
loads, exports every symbol include/vca.h and include/vca_io.h declare, and validates arguments
before touching CUDA."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_2304_12384_b200 import vca

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = "".join(open(os.path.join(ROOT, "include", h)).read() for h in ("vca.h", "vca_io.h"))
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(vca_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert declared_functions() == sorted(vca.EXPORTS)


def test_library_exports_every_declared_symbol():
    L = vca.lib()
    out = subprocess.run(["nm", "-D", "--defined-only", vca._build.LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (vca_[a-z0-9_]+)\b", out))
    for name in declared_functions():
        assert hasattr(L, name)
        assert name in exported, name


def test_built_for_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", vca._build.LIB], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_status_strings_and_version():
    assert vca.version().startswith("vca-b200")
    assert vca.status_string(0) == "ok"
    assert "alignment" in vca.status_string(-6) or "misaligned" in vca.status_string(-6)
    assert vca.status_string(-999) == "unknown status"


def _create(*args):
    L = vca.lib()
    h = ctypes.c_void_p()
    rc = L.vca_create(*args, ctypes.byref(h))
    if rc == 0:
        L.vca_destroy(h)
    return rc, h


@pytest.mark.parametrize("args,code", [
    ((3840, 2160, 12, 0, 32, 1), -3),   # bit depth
    ((3840, 2160, 9, 0, 32, 1), -3),
    ((3840, 2160, 8, 1, 32, 1), -4),    # 4:2:2 unsupported (R-9)
    ((3840, 2160, 8, 2, 32, 0), -4),
    ((3841, 2160, 8, 0, 32, 0), -5),    # odd width
    ((0, 2160, 8, 0, 32, 0), -5),
    ((3840, 2160, 8, 0, 12, 0), -2),    # block size
    ((3840, 2160, 8, 0, 64, 0), -2),
    ((3840, 2160, 8, 0, 8, 1), -2),     # low-pass needs chroma block >= 8 (R-9)
    ((3840, 2160, 8, 0, 4, 1), -2),
    ((640, 360, 8, 0, 0, 1), -2),       # auto w = 8 at 360p -> low-pass rejected
    ((3840, 2160, 8, 0, 32, 2), -1),
])
def test_create_validation_no_gpu(args, code):
    rc, h = _create(*args)
    assert rc == code
    assert not h.value


def test_null_arguments():
    L = vca.lib()
    assert L.vca_create(64, 64, 8, 0, 0, 0, None) == -1
    assert L.vca_get_info(None, None) == -1
    assert L.vca_scratch_bytes(None, 4) == 0
    assert L.vca_reset(None, 0) == -1
    assert L.vca_profile_enable(None, 1) == -1
    L.vca_destroy(None)  # no-op
