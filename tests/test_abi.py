"""C ABI: libkpo.so loads without a GPU and exports exactly what include/kpo.h declares."""
import ctypes
import os
import subprocess

import pytest

from paper_2601_17654_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_lib.LIB_PATH):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2601_17654_b200", "csrc"), "-j8"], check=True)
    return _lib.load()


def test_every_header_symbol_is_exported_and_typed(lib):
    declared = _lib.header_symbols()
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(_lib.SIGNATURES) == declared  # the Python binding covers the header exactly


def test_nm_shows_c_linkage():
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    for name in _lib.header_symbols():
        assert name in exported, name


def test_status_convention_without_gpu(lib):
    # argument validation happens before any CUDA call: invalid input -> KPO_ERR_INVALID + message
    st = lib.kpo_gemm(None, None, None, None, 0, 0, 0, 0, 0, 0, 0, 0, 0, None, None)
    assert st == _lib.KPO_ERR_INVALID
    assert b"null" in lib.kpo_last_error()
    n = ctypes.c_int64(0)
    assert lib.kpo_rmsnorm_bwd_partial_rows(4096, 3072, ctypes.byref(n)) == 0 and n.value > 0
    assert lib.kpo_version() >= 1
    with pytest.raises(_lib.KpoError):
        _lib.call("kpo_rope", None, 0, None, 0, 1, 1, 128, ctypes.c_float(1e4), 0, 0, None)


def test_sm100a_cubin_present():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_tcgen05_and_tma_in_sass():
    """The GEMM is a Blackwell-native kernel: UTC*MMA (tcgen05.mma), UTMALDG (TMA), LDTM (tcgen05.ld)."""
    out = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in out or "UTCMMA" in out
    assert "UTMALDG" in out
    assert "LDTM" in out


def test_fused_swiglu_entry_points_validate_without_gpu(lib):
    """kpo_gemm_swiglu / kpo_gemm_swiglu_bwd / the blocked SwiGLU kernels reject bad shapes before any CUDA
    call (the error behaviour the layer relies on when it decides whether to fuse)."""
    fake = ctypes.c_void_p(1 << 20)  # non-null, 16B-aligned; never dereferenced on the error paths
    with pytest.raises(_lib.KpoError, match="multiple of 256"):  # N = 2*ffn must hold 128-row gate/up blocks
        _lib.call("kpo_gemm_swiglu", fake, fake, fake, fake, 512, 384, 256, 256, 256, 384, 192, 0, fake, None)
    with pytest.raises(_lib.KpoError, match="M must be >= 256"):
        _lib.call("kpo_gemm_swiglu", fake, fake, fake, fake, 128, 512, 256, 256, 256, 512, 256, 0, fake, None)
    with pytest.raises(_lib.KpoError, match="multiple of 256"):  # ffn itself: two blocks per tile
        _lib.call("kpo_gemm_swiglu_bwd", fake, fake, fake, fake, 512, 384, 256, 256, 384, 768, 768, 0, fake, None)
    with pytest.raises(_lib.KpoError, match="block"):
        _lib.call("kpo_swiglu_bwd_blocked", fake, fake, fake, 16, 1024, 100, None)
