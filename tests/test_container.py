"""`.mfrg` container codec (product reader + streaming writer) against the
reference's format (byte-identical files, same validation errors)."""

import numpy as np
import pytest

import paper_2408_11853_b200 as mf
from oracle import fixtures as fx
from oracle import mfrg
from paper_2408_11853_b200.errors import (
    BadMagicError,
    ChecksumMismatchError,
    ContainerError,
    DuplicateTensorError,
    TensorSizeError,
    TruncatedFileError,
    UnknownTensorError,
)


def _tensors(man, w, dtype="f32"):
    np_dt = np.float16 if dtype == "f16" else np.float32
    return [(n, dtype, w[n].shape, w[n].astype(np_dt)) for n, _ in fx.tensor_shapes(man)]


def test_writer_is_byte_identical_to_independent_writer(tmp_path, golden):
    man = fx.tiny_manifest("comet-qe")
    w = fx.fixture_weights(man, 1234)
    a = mf.write_container(mf.ModelManifest(**man), _tensors(man, w), tmp_path / "a.mfrg")
    b = mfrg.write(tmp_path / "b.mfrg", mfrg.manifest_dict(**man), [(n, "f32", w[n]) for n, _ in fx.tensor_shapes(man)])
    assert a == b == golden["tiny"]["comet-qe/post"]["checksum"]
    assert (tmp_path / "a.mfrg").read_bytes() == (tmp_path / "b.mfrg").read_bytes()


@pytest.mark.parametrize("backing", [mf.Backing.MMAP, mf.Backing.EAGER])
def test_round_trip_and_views(tmp_path, backing):
    rng = np.random.default_rng(7)
    for i in range(20):
        names = [f"t{j}" for j in range(int(rng.integers(1, 6)))]
        arrays = {}
        tensors = []
        for n in names:
            shape = tuple(int(s) for s in rng.integers(1, 6, size=int(rng.integers(1, 3))))
            dt = str(rng.choice(["f32", "f16"]))
            a = rng.standard_normal(shape).astype(np.float32 if dt == "f32" else np.float16)
            arrays[n] = a
            tensors.append((n, dt, shape, a.tobytes()))
        path = tmp_path / f"c{i}.mfrg"
        mf.write_container(mf.ModelManifest(**fx.tiny_manifest("comet-qe")), tensors, path)
        with mf.open_container(path, backing) as c:
            for n in names:
                v = c.get_tensor(n)
                assert v.tobytes() == arrays[n].tobytes() and not v.flags.writeable
        _, raw = mfrg.read(path)
        assert all(raw[n].tobytes() == arrays[n].tobytes() for n in names)
        # flip one payload byte -> checksum mismatch on validated open
        data = bytearray(path.read_bytes())
        start = 12 + int.from_bytes(data[8:12], "little")
        start += (-start) % 64
        victim = int(rng.integers(start, len(data)))
        data[victim] ^= 0xFF
        path.write_bytes(bytes(data))
        with pytest.raises(ChecksumMismatchError):
            mf.open_container(path, backing)
        mf.open_container(path, backing, validate=False).close()


def test_format_errors(tmp_path):
    p = tmp_path / "bad.mfrg"
    p.write_bytes(b"NOTMAGIC" + b"\x00" * 10)
    with pytest.raises(BadMagicError):
        mf.open_container(p)
    p.write_bytes(b"MFRG0001" + (1000).to_bytes(4, "little") + b"{}")
    with pytest.raises(TruncatedFileError):
        mf.read_manifest(p)
    man = mf.ModelManifest(**fx.tiny_manifest("comet-qe"))
    with pytest.raises(DuplicateTensorError):
        mf.write_container(man, [("a", "f32", (1,), b"\0" * 4), ("a", "f32", (1,), b"\0" * 4)], p)
    with pytest.raises(TensorSizeError):
        mf.write_container(man, [("a", "f32", (2,), b"\0" * 4)], p)
    mf.write_container(man, [("a", "f32", (1,), b"\0" * 4)], p)
    with mf.open_container(p) as c:
        with pytest.raises(UnknownTensorError, match="'zz'"):
            c.get_tensor("zz")
    with pytest.raises(ContainerError, match="divisible"):
        mf.ModelManifest(**fx.tiny_manifest("comet", d_model=10, n_heads=3))
    with pytest.raises(ContainerError, match="unknown norm_style"):
        mf.ModelManifest(**fx.tiny_manifest("comet", norm_style="mid"))


def test_manifest_round_trip(tmp_path):
    man = mf.ModelManifest(**fx.tiny_manifest("bleurt", head_hidden=[8, 4], norm_style="pre"))
    w = fx.fixture_weights(fx.tiny_manifest("bleurt", head_hidden=[8, 4]), 3)
    mf.write_container(man, [(n, "f32", a.shape, a) for n, a in w.items()], tmp_path / "m.mfrg")
    got = mf.read_manifest(tmp_path / "m.mfrg")
    assert got.like is mf.Kind.BLEURT and got.head_hidden == [8, 4]
    assert got.norm_style is mf.NormStyle.PRE and len(got.checksum) == 64
