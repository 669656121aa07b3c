"""CPU checks of the C-ABI boundary: libhf.so builds, loads without a GPU and
exports every entry point include/hf.h declares; the binding exposes them and
fails loudly (no CPU fallback) when the library is missing."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "hf.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hf_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2208_01907_b200 import build
    lib_path = build.build()
    lib = ctypes.CDLL(lib_path)
    names = _declared()
    assert len(names) >= 18
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    from paper_2208_01907_b200 import hf
    assert set(names) <= set(hf.EXPORTED)


def test_error_path_without_context():
    from paper_2208_01907_b200 import hf
    lib = hf.load()
    # NULL context -> HF_ERR_INVALID_ARG, never a crash
    assert lib.hf_scale(None, 4, None, 4, None) == hf.HF_ERR_INVALID_ARG
    assert lib.hf_factor_lowprec(None, 4, None, 4, None, None, None, None, None) == hf.HF_ERR_INVALID_ARG
    assert lib.hf_last_error(None) is not None


def test_binding_fails_loudly_without_library(monkeypatch, tmp_path):
    from paper_2208_01907_b200 import hf
    monkeypatch.setattr(hf, "_lib", None)
    monkeypatch.setattr(hf, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(ImportError):
        hf.load()


def test_sm100a_code_in_library():
    import subprocess
    from paper_2208_01907_b200 import build
    lib_path = build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib_path], capture_output=True, text=True).stdout
    assert "DMMA" in sass and "FFMA" in sass      # FP64 tensor path and FP32 FFMA path present
