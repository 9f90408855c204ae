"""The C-ABI libraries load and export exactly what include/*.h declares
(no compute calls here: this runs without a GPU)."""

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

from paper_2408_11853_b200 import native

ROOT = Path(__file__).resolve().parent.parent
LIBS = {"mfgpu.h": "libmfgpu.so", "mfgpu_test.h": "libmfgpu.so", "mfhost.h": "libmfhost.so"}


def declared(header):
    text = (ROOT / "include" / header).read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b((?:mfg|mfgt|mfh)_[a-z0-9_]+)\s*\(", text)))


@pytest.mark.parametrize("header", sorted(LIBS))
def test_library_exports_every_declared_symbol(header):
    names = declared(header)
    assert names, header
    lib_path = ROOT / "paper_2408_11853_b200" / "lib" / LIBS[header]
    lib = ctypes.CDLL(str(lib_path))
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    nm = subprocess.run(["nm", "-D", "--defined-only", str(lib_path)], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}$", nm, re.M), n


def test_gpu_library_is_sm100a():
    lib = ROOT / "paper_2408_11853_b200" / "lib" / "libmfgpu.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(lib)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", str(lib)], capture_output=True, text=True).stdout
    for mnemonic in ("UTCHMMA", "UTMALDG", "LDTM"):  # tcgen05.mma, TMA, tcgen05.ld
        assert mnemonic in sass, mnemonic


def test_create_fails_cleanly_with_code_and_message(tmp_path):
    lib = native.gpu()
    cfg = native.MfgConfig(str(tmp_path / "missing.mfrg").encode(), 0, 0, 0, 0, 0)
    h = ctypes.c_void_p()
    rc = lib.mfg_create(ctypes.byref(cfg), ctypes.byref(h))
    assert rc != 0 and not h.value
    code, msg = native.last_error(None)
    assert code == rc and msg


def test_host_library_null_safety():
    lib = native.host()
    assert lib.mfh_vocab_size(None) == 0
    assert lib.mfh_plan(None, 0, 0, 1, 1, None) == 2  # mini_batch < 1 rejected


def test_mfeval_driver_links_and_reports_usage():
    """examples/mfeval.cpp links against both C-ABI libraries (no GPU call here)."""
    exe = ROOT / "paper_2408_11853_b200" / "lib" / "mfeval"
    assert exe.exists(), "build() produces lib/mfeval"
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 2 and "usage:" in r.stderr
    nm = subprocess.run(["nm", "-D", "--undefined-only", str(exe)], capture_output=True, text=True).stdout
    for sym in ("mfh_encode_tsv", "mfh_plan", "mfh_pack_roles", "mfg_create", "mfg_score_batch"):
        assert sym in nm, sym
