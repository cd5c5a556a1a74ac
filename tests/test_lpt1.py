"""LPT1 containers: bit-exact round trips and the distinct
errors the spec lists (TRIVIAL examples of SPEC.md:540-542)."""
import numpy as np
import pytest

from paper_1506_00014_b200 import lpt1


def test_roundtrip_is_byte_identical(tmp_path):
    rng = np.random.default_rng(0)
    img = rng.standard_normal((32, 32)).astype(np.float32)
    c = lpt1.Container("image", img, lpt1.image_grid(32), {"phantom": "random", "seed": 0})
    path = tmp_path / "a.lpt"
    lpt1.write_container(path, c)
    raw = path.read_bytes()
    back = lpt1.read_container(path)
    assert back.kind == "image" and back.dtype == "f32" and back.grid == c.grid and back.meta == c.meta
    assert back.data.tobytes() == img.tobytes()
    assert lpt1.encode(back) == raw
    assert len(raw) == 8 + int.from_bytes(raw[4:8], "little") + 4 * 32 * 32


def test_complex_spectrum_and_sinogram_grids():
    z = (np.arange(12) + 1j * np.arange(12)[::-1]).reshape(3, 4).astype(np.complex64)
    c = lpt1.decode(lpt1.encode(lpt1.Container("spectrum", z)))
    assert c.dtype == "c32" and np.array_equal(c.data, z)
    g = lpt1.sinogram_grid(96, 64)
    s = lpt1.decode(lpt1.encode(lpt1.Container("sinogram", np.ones((96, 64), np.float32), g)))
    assert s.grid["axis0"]["count"] == 96 and abs(s.grid["axis0"]["spacing"] - np.pi / 96) < 1e-15


def test_distinct_errors():
    good = lpt1.encode(lpt1.Container("image", np.zeros((64, 64), np.float32), lpt1.image_grid(64)))
    with pytest.raises(lpt1.BadMagicError):
        lpt1.decode(b"LPT2" + good[4:])
    with pytest.raises(lpt1.TruncatedError):
        lpt1.decode(good[:-3])  # a truncated file, not a crash
    with pytest.raises(lpt1.TruncatedError):
        lpt1.decode(good[:6])
    with pytest.raises(lpt1.ShapeError):
        lpt1.decode(good[:-4 * 64])  # header says 64 x 64, payload holds 63 rows
    with pytest.raises(lpt1.ShapeError):
        lpt1.decode(good + b"\0\0\0\0")
    hdr = b'{"kind":"volume","rows":1,"cols":1,"dtype":"f32"}'
    with pytest.raises(lpt1.SchemaError):
        lpt1.decode(b"LPT1" + len(hdr).to_bytes(4, "little") + hdr + b"\0" * 4)
    hdr = b'{"kind":"image","rows":"1","cols":1,"dtype":"f32"}'
    with pytest.raises(lpt1.SchemaError):
        lpt1.decode(b"LPT1" + len(hdr).to_bytes(4, "little") + hdr + b"\0" * 4)
    with pytest.raises(lpt1.SchemaError):
        lpt1.decode(b"LPT1" + (3).to_bytes(4, "little") + b"\xff\xfe{")
    assert all(issubclass(e, ValueError) for e in (lpt1.BadMagicError, lpt1.TruncatedError, lpt1.ShapeError,
                                                   lpt1.SchemaError))
