"""C-ABI contract checks that need no GPU: the library builds for sm_100a,
loads, exports every symbol include/cuasm_ffn.h declares, and its argument
validation / no-device behaviour returns status codes instead of crashing."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2501_08071_b200 as ffn
from paper_2501_08071_b200 import build as ffn_build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cuasm_ffn.h")


@pytest.fixture(scope="module")
def lib():
    ffn_build.build()
    return ffn.load_library()


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cuasm_[a-z_]+)\s*\(", src)))


def test_header_declares_the_north_star_entry_points():
    names = header_functions()
    for required in ("cuasm_ffn_init", "cuasm_ffn_forward", "cuasm_ffn_destroy"):
        assert required in names


def test_library_exports_every_declared_symbol(lib):
    names = header_functions()
    assert sorted(ffn.EXPORTED_SYMBOLS) == names
    out = subprocess.run(["nm", "-D", "--defined-only", ffn.lib_path()], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (cuasm_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    for n in names:
        assert hasattr(lib, n)


def test_abi_version(lib):
    assert lib.cuasm_ffn_abi_version() == 1


def test_library_is_sm100a_cubin():
    out = subprocess.run(["cuobjdump", "--list-elf", ffn.lib_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_sass_uses_tcgen05_and_tma():
    sass = subprocess.run(["cuobjdump", "-sass", ffn.lib_path()], capture_output=True, text=True).stdout
    for op in ("UTCHMMA", "UTMALDG", "LDTM", "UTCBAR"):
        assert op in sass, op
    assert re.search(r"\bHMMA\b", sass) is None  # no legacy mma.sync path


def test_null_handle_and_no_device(lib):
    vp = ctypes.c_void_p
    # NULL handle -> INVALID_ARG, never a crash
    assert lib.cuasm_ffn_forward(None, None, None, None, None, None, 1, 8, 8, 1e-6, None) == ffn.ERR_INVALID_ARG
    assert lib.cuasm_ffn_destroy(None) == ffn.OK
    assert lib.cuasm_ffn_set_option(None, 0, 0) == ffn.ERR_INVALID_ARG
    # init on a CPU-only host: UNSUPPORTED with a message, *h stays NULL
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible; covered by the gpu tests")
    h = vp(1234)
    st = lib.cuasm_ffn_init(ctypes.byref(h), 0, 0)
    assert st in (ffn.ERR_UNSUPPORTED, ffn.ERR_CUDA)
    assert h.value is None
    assert lib.cuasm_ffn_last_error(None)
    # bad dtype is rejected before touching the device
    assert lib.cuasm_ffn_init(ctypes.byref(h), 0, 7) == ffn.ERR_INVALID_ARG


def test_python_binding_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    with pytest.raises(Exception):
        ffn.FusedFFN("cuda:0", torch.bfloat16)
