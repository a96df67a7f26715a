"""MNMA container: on-disk format for TN cores (absent from the reference code).

Layout (little-endian throughout), as the SPEC's `cli` module specifies:
  magic  b"MNMA"            4 bytes (0x4D 0x4E 0x4D 0x41)
  u32    version = 1
  u32    entry count
  index, per entry:
    u16  name length, UTF-8 name
    u8   dtype {0: f32, 1: f64}
    u8   ndim
    u64  dims[ndim]
    u64  payload offset (from file start; 64-byte aligned, strictly increasing)
  u64    metadata length, UTF-8 JSON metadata document (may be empty)
  payload: raw C-order scalar blocks at their offsets (zero padding between blocks)

Errors mirror the reference's (errors.py:52-61): bad magic / version / index ->
FormatError; payload shorter than declared -> TruncationError; repeated name ->
DuplicateEntryError. Writes are atomic (temp file + rename).
``save_layers`` / ``load_layers`` store ``CompressedLayer`` objects (family, mode shape and
row_mode_count go into the metadata document; cores/factors/matrix are the entries).
"""

from __future__ import annotations

import json
import math
import os
import struct
import tempfile

import numpy as np

from .errors import MinimaError

MAGIC = b"MNMA"
VERSION = 1
ALIGN = 64
_DT = {0: np.dtype("<f4"), 1: np.dtype("<f8")}
_DT_CODE = {np.dtype("float32"): 0, np.dtype("float64"): 1}


class FormatError(MinimaError):
    """Container file has a bad magic number, version, or index (errors.py:52)."""


class TruncationError(MinimaError):
    """Container payload is shorter than its index declares (errors.py:56)."""


class DuplicateEntryError(MinimaError):
    """Container index declares the same entry name twice (errors.py:60)."""


def _align(n: int) -> int:
    return (n + ALIGN - 1) // ALIGN * ALIGN


def write_container(path: str, entries: dict, metadata: dict | None = None) -> None:
    """Write named f32/f64 arrays (insertion order) and an optional JSON metadata document."""
    names = list(entries.keys())
    if len(set(names)) != len(names):
        raise DuplicateEntryError("duplicate entry names")
    arrays = []
    for n in names:
        a = np.asarray(entries[n])
        if a.dtype not in _DT_CODE:
            raise FormatError(f"entry {n!r}: dtype {a.dtype} not in {{float32, float64}}")
        # np.array keeps 0-d entries 0-d (ascontiguousarray would promote them to 1-d)
        arrays.append(np.array(a, dtype=a.dtype.newbyteorder("<"), order="C", copy=True))
    meta = json.dumps(metadata, sort_keys=True).encode() if metadata is not None else b""
    index_size = 12 + sum(2 + len(n.encode()) + 2 + 8 * a.ndim + 8 for n, a in zip(names, arrays)) + 8 + len(meta)
    offsets, off = [], _align(index_size)
    for a in arrays:
        offsets.append(off)
        off = _align(off + a.nbytes)
    head = bytearray(MAGIC + struct.pack("<II", VERSION, len(names)))
    for n, a, o in zip(names, arrays, offsets):
        nb = n.encode()
        head += struct.pack("<H", len(nb)) + nb + struct.pack("<BB", _DT_CODE[a.dtype], a.ndim)
        head += struct.pack(f"<{a.ndim}Q", *a.shape) + struct.pack("<Q", o)
    head += struct.pack("<Q", len(meta)) + meta
    assert len(head) == index_size
    d = os.path.dirname(os.path.abspath(path)) or "."
    fd, tmp = tempfile.mkstemp(prefix=".mnma-", dir=d)
    try:
        with os.fdopen(fd, "wb") as f:
            f.write(head)
            pos = len(head)
            for a, o in zip(arrays, offsets):
                f.write(b"\0" * (o - pos))
                f.write(a.tobytes(order="C"))
                pos = o + a.nbytes
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def read_container(path: str) -> tuple[dict, dict | None]:
    """Read a container; returns ({name: ndarray}, metadata or None). Bit-exact inverse of write."""
    with open(path, "rb") as f:
        buf = f.read()
    if len(buf) < 12 or buf[:4] != MAGIC:
        raise FormatError("bad magic")
    version, count = struct.unpack_from("<II", buf, 4)
    if version != VERSION:
        raise FormatError(f"unsupported version {version}")
    pos = 12
    index = []
    try:
        for _ in range(count):
            (ln,) = struct.unpack_from("<H", buf, pos)
            pos += 2
            name = buf[pos:pos + ln].decode()
            pos += ln
            code, ndim = struct.unpack_from("<BB", buf, pos)
            pos += 2
            dims = struct.unpack_from(f"<{ndim}Q", buf, pos)
            pos += 8 * ndim
            (off,) = struct.unpack_from("<Q", buf, pos)
            pos += 8
            if code not in _DT:
                raise FormatError(f"entry {name!r}: unknown dtype code {code}")
            index.append((name, _DT[code], tuple(int(d) for d in dims), int(off)))
        (mlen,) = struct.unpack_from("<Q", buf, pos)
        pos += 8
    except struct.error as e:
        raise FormatError(f"truncated index: {e}") from None
    if pos + mlen > len(buf):
        raise TruncationError("metadata extends past end of file")
    meta = json.loads(buf[pos:pos + mlen].decode()) if mlen else None
    names = [n for n, *_ in index]
    if len(set(names)) != len(names):
        raise DuplicateEntryError("duplicate entry names in index")
    out, prev_end = {}, pos + mlen
    for name, dt, dims, off in index:
        if off % ALIGN or off < prev_end:
            raise FormatError(f"entry {name!r}: offset {off} not 64-byte aligned / not increasing")
        nbytes = dt.itemsize * math.prod(dims)
        if off + nbytes > len(buf):
            raise TruncationError(f"entry {name!r}: payload truncated")
        out[name] = np.frombuffer(buf, dtype=dt, count=math.prod(dims), offset=off).reshape(dims).copy()
        prev_end = off + nbytes
    return out, meta


def save_layers(path: str, layers: dict) -> None:
    """Store {name: CompressedLayer} (cores/factors/matrix as entries, structure in metadata)."""
    entries, meta = {}, {"schema": "tnl-layers/1", "layers": {}}
    for lname, L in layers.items():
        meta["layers"][lname] = {"family": L.family, "mode_shape": list(L.mode_shape),
                                 "row_mode_count": L.row_mode_count}
        if L.family == "tucker":
            entries[f"{lname}.core"] = np.asarray(L.core)
            for k, u in enumerate(L.factors):
                entries[f"{lname}.factor.{k}"] = np.asarray(u)
        elif L.family in ("tt", "tr"):
            for k, c in enumerate(L.cores):
                entries[f"{lname}.core.{k}"] = np.asarray(c)
        else:
            entries[f"{lname}.matrix"] = np.asarray(L.matrix)
    write_container(path, entries, meta)


def load_layers(path: str) -> dict:
    """Inverse of save_layers: {name: CompressedLayer} (validated on construction)."""
    from .layer import CompressedLayer

    entries, meta = read_container(path)
    if not meta or "layers" not in meta:
        raise FormatError("container has no layer metadata")
    out = {}
    for lname, info in meta["layers"].items():
        fam, ms, rm = info["family"], tuple(info["mode_shape"]), int(info["row_mode_count"])
        d = len(ms)
        try:
            if fam == "tucker":
                out[lname] = CompressedLayer(fam, ms, rm, core=entries[f"{lname}.core"],
                                             factors=[entries[f"{lname}.factor.{k}"] for k in range(d)])
            elif fam in ("tt", "tr"):
                out[lname] = CompressedLayer(fam, ms, rm, cores=[entries[f"{lname}.core.{k}"] for k in range(d)])
            else:
                out[lname] = CompressedLayer(fam, ms, rm, matrix=entries[f"{lname}.matrix"])
        except KeyError as e:
            raise FormatError(f"layer {lname!r}: missing entry {e}") from None
    return out
