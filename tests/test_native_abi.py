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


def _container_with_index(tmp_path, patch):
    """A valid tiny container whose JSON tensor index is rewritten by `patch`."""
    import json
    import struct

    from oracle import fixtures as fx
    from oracle import mfrg
    man = fx.tiny_manifest("comet-qe")
    w = fx.fixture_weights(man, 3)
    path = tmp_path / "c.mfrg"
    mfrg.write(str(path), mfrg.manifest_dict(**man), [(n, "f32", w[n]) for n, _ in fx.tensor_shapes(man)])
    raw = path.read_bytes()
    hlen = struct.unpack("<I", raw[8:12])[0]
    header = json.loads(raw[12:12 + hlen])
    payload = raw[(12 + hlen + 63) // 64 * 64:]
    patch(header["tensors"])
    hb = json.dumps(header, sort_keys=True, separators=(",", ":")).encode()
    pad = (-(12 + len(hb))) % 64
    bad = tmp_path / "bad.mfrg"
    bad.write_bytes(b"MFRG0001" + struct.pack("<I", len(hb)) + hb + b"\0" * pad + payload)
    return str(path), str(bad)


@pytest.mark.parametrize("what,patch,needle", [
    ("negative offset", lambda t: t[1].update(offset=-t[1]["nbytes"] // 64 * 64), "offset"),
    ("past end", lambda t: t[-1].update(offset=t[-1]["offset"] + 1 << 20), "past end"),
    ("overlap", lambda t: t[1].update(offset=t[0]["offset"]), "overlap"),
    ("duplicate", lambda t: t[1].update(name=t[0]["name"]), "duplicate"),
    ("huge offset", lambda t: t[0].update(offset=2 ** 62), "past end"),
])
def test_native_container_check_rejects_bad_index(tmp_path, what, patch, needle):
    """mfg_check_container (host only, the checks mfg_create runs before the GPU)."""
    lib = native.gpu()
    good, bad = _container_with_index(tmp_path, patch)
    assert lib.mfg_check_container(good.encode()) == 0
    rc = lib.mfg_check_container(bad.encode())
    code, msg = native.last_error(None)
    assert rc == 3 and code == 3 and needle in msg, (what, msg)
