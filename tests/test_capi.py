"""CPU-side checks of the drop-in boundary: libautosp.so builds for sm_100a, loads,
exports exactly what include/autosp.h declares, and reports errors through the
status-code convention (no compute calls: there is no GPU here)."""

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def lib():
    from paper_2604_27089_b200 import _build, _lib
    _build.build()
    return _lib.load()


def _declared():
    text = (ROOT / "include" / "autosp.h").read_text()
    return sorted(set(re.findall(r"AUTOSP_API\s+[\w\s\*]+?\b(autosp_\w+)\s*\(", text)))


def test_header_declares_entry_points():
    names = _declared()
    for n in ("autosp_a2a", "autosp_a2a_wait", "autosp_attn_fwd", "autosp_attn_bwd",
              "autosp_symm_alloc", "autosp_symm_open"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    from paper_2604_27089_b200 import _lib
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (autosp_\w+)", out))
    assert set(_declared()) <= exported
    assert set(_declared()) == set(_lib.EXPORTS)  # the ctypes binding covers the header


def test_abi_version_and_sm100a_cubin(lib):
    from paper_2604_27089_b200 import _lib
    assert lib.autosp_abi_version() == 3
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_sass_uses_tcgen05_and_tma(lib):
    from paper_2604_27089_b200 import _lib
    sass = subprocess.run(["cuobjdump", "-sass", str(_lib.LIB_PATH)], capture_output=True,
                          text=True).stdout
    assert "UTCHMMA" in sass or "UTCMMA" in sass  # tcgen05.mma
    assert "UTMALDG" in sass  # TMA tensor loads
    assert "LDTM" in sass and "STTM" in sass  # TMEM <-> registers


def test_validation_errors_map_to_status_codes(lib):
    from paper_2604_27089_b200 import _lib
    from paper_2604_27089_b200.errors import ValidationError
    # bad direction -> AUTOSP_ERR_VALIDATION before any CUDA call
    rc = lib.autosp_a2a(7, None, 1, 1, 8, 8, 2, 2, 0, None, None, 1, None)
    assert rc == 2
    assert b"direction" in lib.autosp_last_error()
    with pytest.raises(ValidationError):
        _lib.check(rc, "a2a")
    # indivisible sequence (reference sp_pass.py:145-146)
    t = _lib.A2ATensor(1, 0, 0, 0, 0, 0, 0, 0, 4, 0)
    ptrs = (ctypes.c_void_p * 2)(16, 16)
    rc = lib.autosp_a2a(0, ctypes.byref(t), 1, 1, 9, 8, 2, 2, 0, ptrs, ptrs, 1, None)
    assert rc == 2 and b"divisible" in lib.autosp_last_error()
    # heads not divisible by world (sp_pass.py:147-148)
    t = _lib.A2ATensor(16, 0, 0, 0, 0, 0, 0, 0, 3, 0)
    rc = lib.autosp_a2a(0, ctypes.byref(t), 1, 1, 8, 8, 2, 2, 0, ptrs, ptrs, 1, None)
    assert rc == 2 and b"heads" in lib.autosp_last_error()
    # unsupported head dim in attention
    z = _lib.AttnTensor(16, 64, 64, 8)
    rc = lib.autosp_attn_fwd(z, z, z, z, 16, 1, 1, 1, 8, 48, 1.0, 1, None)
    assert rc == 3


def test_ops_fail_loudly_without_library(monkeypatch, tmp_path):
    from paper_2604_27089_b200 import _lib
    from paper_2604_27089_b200.errors import ExtensionMissingError
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", tmp_path / "missing.so")
    with pytest.raises(ExtensionMissingError):
        _lib.load()


def test_check_word_covers_every_tensor_of_a_call(lib):
    """the symmetric-offset check word folds in EVERY destination descriptor of
    a call (offset, strides, heads), not only tensor 0's offset."""
    from paper_2604_27089_b200 import _lib

    def word(offs, heads=(8, 8, 8)):
        arr = (_lib.A2ATensor * 3)(*[_lib.A2ATensor(16, 0, 0, 0, o, 1, 2, 3, h, 0)
                                     for o, h in zip(offs, heads)])
        return lib.autosp_a2a_check(0, arr, 3)

    base = word((0, 4096, 8192))
    assert base == word((0, 4096, 8192))
    assert base != word((0, 4096, 9216))   # a later tensor's offset diverged
    assert base != word((0, 5120, 8192))
    assert base != word((0, 4096, 8192), heads=(8, 8, 16))
    spec = _lib.PushSpec(2, 0, 1024, 1, 2, 3, None, None, 1)
    assert lib.autosp_push_check(ctypes.byref(spec), 4) != lib.autosp_push_check(
        ctypes.byref(_lib.PushSpec(2, 0, 2048, 1, 2, 3, None, None, 1)), 4)
