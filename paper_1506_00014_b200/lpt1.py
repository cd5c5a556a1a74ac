"""LPT1 containers: the file format that images, sinograms and kernel spectra
cross on either side of the operators (the reference's
`proj/src/io.cpp` is an empty namespace).

Layout: magic b"LPT1" | header_len (uint32, little endian) | UTF-8 JSON header
{"kind": "image" | "sinogram" | "spectrum", "rows", "cols", "dtype": "f32" |
"c32", "grid": GridSpec fields, "meta": {...}} | row-major little-endian
IEEE-754 float32 payload (complex as interleaved re, im), exactly
rows * cols * 4 * (1 | 2) bytes. read(write(x)) is byte-identical.

Errors are distinct (each a ValueError, like the reference's
std::invalid_argument family): BadMagicError, TruncatedError (file shorter
than its header or payload), ShapeError (payload length disagrees with
rows x cols), SchemaError (header JSON missing/invalid fields).
"""
from __future__ import annotations

import json
import math
import struct
from dataclasses import dataclass, field

import numpy as np

MAGIC = b"LPT1"
KINDS = ("image", "sinogram", "spectrum")
DTYPES = {"f32": (np.dtype("<f4"), 1), "c32": (np.dtype("<c8"), 2)}
GRID_KINDS = ("cartesian", "polar", "logpolar_fine", "logpolar_sector")  # types.hpp GridKind


class BadMagicError(ValueError):
    pass


class TruncatedError(ValueError):
    pass


class ShapeError(ValueError):
    pass


class SchemaError(ValueError):
    pass


def axis(count: int, origin: float, spacing: float) -> dict:
    """AxisSpec (types.hpp): sample i at origin + i * spacing."""
    return {"count": int(count), "origin": float(origin), "spacing": float(spacing)}


def image_grid(N: int) -> dict:
    """Cartesian raster on [-1/2, 1/2)^2, rows = x2 (geometry.cpp:19-25)."""
    return {"kind": "cartesian", "axis0": axis(N, -0.5, 1.0 / N), "axis1": axis(N, -0.5, 1.0 / N)}


def sinogram_grid(n_theta: int, N: int) -> dict:
    """Polar grid: theta_i = i pi / n_theta, s_j = -1/2 + j / N (geometry.cpp:27-33)."""
    return {"kind": "polar", "axis0": axis(n_theta, 0.0, math.pi / n_theta), "axis1": axis(N, -0.5, 1.0 / N)}


@dataclass
class Container:
    kind: str
    data: np.ndarray  # rows x cols, float32 or complex64
    grid: dict = field(default_factory=dict)
    meta: dict = field(default_factory=dict)

    @property
    def dtype(self) -> str:
        return "c32" if np.iscomplexobj(self.data) else "f32"


def _header(c: Container) -> bytes:
    if c.kind not in KINDS:
        raise SchemaError(f"kind must be one of {KINDS}, got {c.kind!r}")
    a = np.asarray(c.data)
    if a.ndim != 2:
        raise ShapeError(f"payload must be 2-D rows x cols, got shape {a.shape}")
    h = {"kind": c.kind, "rows": int(a.shape[0]), "cols": int(a.shape[1]), "dtype": c.dtype,
         "grid": c.grid, "meta": c.meta}
    return json.dumps(h, sort_keys=True, separators=(",", ":")).encode("utf-8")


def encode(c: Container) -> bytes:
    hdr = _header(c)
    dt, _ = DTYPES[c.dtype]
    payload = np.ascontiguousarray(c.data, dtype=dt).tobytes()
    return MAGIC + struct.pack("<I", len(hdr)) + hdr + payload


def decode(buf: bytes) -> Container:
    if len(buf) < 8:
        raise TruncatedError(f"{len(buf)} bytes: shorter than magic + header length")
    if buf[:4] != MAGIC:
        raise BadMagicError(f"bad magic {buf[:4]!r} (expected {MAGIC!r})")
    (hlen,) = struct.unpack("<I", buf[4:8])
    if len(buf) < 8 + hlen:
        raise TruncatedError(f"header of {hlen} bytes runs past the end of the file")
    try:
        h = json.loads(buf[8:8 + hlen].decode("utf-8"))
    except (UnicodeDecodeError, json.JSONDecodeError) as e:
        raise SchemaError(f"header is not UTF-8 JSON: {e}") from None
    if not isinstance(h, dict):
        raise SchemaError("header must be a JSON object")
    for key, typ in (("kind", str), ("rows", int), ("cols", int), ("dtype", str)):
        if not isinstance(h.get(key), typ) or isinstance(h.get(key), bool):
            raise SchemaError(f"header field {key!r} missing or not {typ.__name__}")
    if h["kind"] not in KINDS:
        raise SchemaError(f"unknown kind {h['kind']!r}")
    if h["dtype"] not in DTYPES:
        raise SchemaError(f"unknown dtype {h['dtype']!r}")
    if h["rows"] < 0 or h["cols"] < 0:
        raise SchemaError("negative shape")
    grid, meta = h.get("grid", {}), h.get("meta", {})
    if not isinstance(grid, dict) or not isinstance(meta, dict):
        raise SchemaError("grid and meta must be JSON objects")
    if grid and grid.get("kind") not in GRID_KINDS:
        raise SchemaError(f"unknown grid kind {grid.get('kind')!r}")
    dt, words = DTYPES[h["dtype"]]
    want = h["rows"] * h["cols"] * 4 * words
    got = len(buf) - 8 - hlen
    if got < want and got % (h["cols"] * 4 * words or 1) == 0 and got > 0:
        raise ShapeError(f"header says {h['rows']}x{h['cols']} but the payload holds {got // (h['cols'] * 4 * words)} rows")
    if got < want:
        raise TruncatedError(f"payload {got} bytes, header needs {want}")
    if got > want:
        raise ShapeError(f"payload {got} bytes, header needs exactly {want}")
    data = np.frombuffer(buf, dtype=dt, count=h["rows"] * h["cols"], offset=8 + hlen).reshape(h["rows"], h["cols"])
    return Container(h["kind"], data.copy(), grid, meta)


def write_container(path, c: Container) -> None:
    with open(path, "wb") as f:
        f.write(encode(c))


def read_container(path) -> Container:
    with open(path, "rb") as f:
        return decode(f.read())
