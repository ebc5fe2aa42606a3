"""Host-side checks of the C-ABI library that need no GPU (CPU suite)."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2103_06998_b200 as adi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "adi_maxwell.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(adi_[A-Za-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def built():
    return adi.build()


def test_library_exports_every_declared_symbol(built):
    syms = declared_symbols()
    assert len(syms) >= 20
    L = ctypes.CDLL(built)
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    assert sorted(syms) == sorted(adi.EXPORTS)


def test_library_is_sm100a(built):
    out = subprocess.run(["cuobjdump", "--list-elf", built], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_device(built):
    """On a box without a GPU the binding must fail loudly, never compute."""
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(adi.AdiError):
        adi.Patch(4, 2, 0.1)


def test_bad_args_rejected_before_device(built):
    L = adi.lib()
    h = ctypes.c_void_p()
    for n, p, tau in [(0, 2, 0.1), (4, 0, 0.1), (4, 6, 0.1), (4, 2, -1.0), (4, 2, float("nan"))]:
        cfg = adi.AdiConfig(n, p, tau, 0, 0, 0, 1, None)
        assert L.adi_create(ctypes.byref(cfg), ctypes.byref(h)) == adi.ADI_ERR_ARG
        assert h.value is None
        assert L.adi_last_error()
