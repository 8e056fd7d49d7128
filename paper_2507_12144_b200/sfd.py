"""SFD1 / SWB1 containers (sfd.hpp:1-245): bit-exact float64 interchange for fields and
named weight tensors, shared with the reference library.

Both formats are: 4-byte magic, uint32 little-endian header length, UTF-8 JSON header
(nlohmann::json::dump -> compact, keys sorted), raw float64 little-endian payload.
Fields are read straight into device memory as the fp32 the kernels consume (the file
keeps fp64); writing upcasts exactly.  Read failures raise ``IoError`` with the
reference's codes (sfd.hpp:25-30).
"""
from __future__ import annotations

import json
import struct
from dataclasses import dataclass, field as dc_field
from enum import IntEnum
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np


class IoErrorCode(IntEnum):
    bad_magic = 0
    header_mismatch = 1
    payload_length_mismatch = 2
    unknown_grid_kind = 3


class IoError(RuntimeError):
    def __init__(self, code: IoErrorCode, what: str):
        super().__init__(what)
        self.code = code


def _dump(header: dict) -> bytes:
    # nlohmann::json::dump(): no whitespace, object keys in std::map (sorted) order
    return json.dumps(header, separators=(",", ":"), sort_keys=True, ensure_ascii=False).encode()


def _frame(magic: bytes, header: dict) -> bytes:
    h = _dump(header)
    return magic + struct.pack("<I", len(h)) + h


def _parse_frame(buf: bytes, magic: bytes) -> Tuple[dict, int]:
    if len(buf) < 8 or buf[:4] != magic:
        raise IoError(IoErrorCode.bad_magic, "bad magic")
    (hlen,) = struct.unpack("<I", buf[4:8])
    if len(buf) < 8 + hlen:
        raise IoError(IoErrorCode.header_mismatch, "header length exceeds file size")
    try:
        header = json.loads(buf[8:8 + hlen].decode("utf-8"))
    except (ValueError, UnicodeDecodeError):
        raise IoError(IoErrorCode.header_mismatch, "header is not valid JSON") from None
    return header, 8 + hlen


def _read(path) -> bytes:
    try:
        with open(path, "rb") as f:
            return f.read()
    except OSError:
        raise IoError(IoErrorCode.header_mismatch, f"cannot open {path}") from None


# ------------------------------------------------------------------ fields
_KIND_NAMES = {0: "equiangular", 1: "gaussian"}


def write_sfd(path, field, channel_names: Optional[Sequence[str]] = None) -> None:
    """sfd.hpp:107-131.  ``field`` is a SphericalField (device or host data)."""
    data = field.data
    if hasattr(data, "detach"):
        data = data.detach().to("cpu").double().numpy()
    data = np.ascontiguousarray(np.asarray(data, dtype="<f8"))
    g = field.grid
    C = int(data.size // (g.nlat * g.nlon))
    names = list(channel_names) if channel_names else [f"ch{c}" for c in range(C)]
    if len(names) != C:
        raise IoError(IoErrorCode.header_mismatch, "channel name count mismatch")
    header = {"grid_kind": _KIND_NAMES[g.kind], "nlat": g.nlat, "nlon": g.nlon, "channels": C,
              "channel_names": names, "dtype": "f64le", "layout": "c,h,w"}
    with open(path, "wb") as f:
        f.write(_frame(b"SFD1", header))
        f.write(data.tobytes())


@dataclass
class SfdContents:
    field: object
    channel_names: List[str]


def read_sfd(path, device=None) -> SfdContents:
    """sfd.hpp:133-174.  With ``device`` the field lands on the GPU as fp32."""
    from . import sphere as S
    buf = _read(path)
    header, off = _parse_frame(buf, b"SFD1")
    try:
        kind = header["grid_kind"]
        nlat, nlon, C = int(header["nlat"]), int(header["nlon"]), int(header["channels"])
        names = list(header["channel_names"])
        dtype, layout = header["dtype"], header["layout"]
        if not all(isinstance(v, str) for v in (kind, dtype, layout)):
            raise TypeError
    except (KeyError, TypeError, ValueError):
        raise IoError(IoErrorCode.header_mismatch, "header field missing or ill-typed") from None
    if dtype != "f64le" or layout != "c,h,w":
        raise IoError(IoErrorCode.header_mismatch, "unsupported dtype or layout")
    if len(names) != C:
        raise IoError(IoErrorCode.header_mismatch, "channel name count mismatch")
    if kind == "equiangular":
        grid = S.build_equiangular(nlat, nlon)
    elif kind == "gaussian":
        grid = S.build_gaussian(nlat, nlon)
    else:
        raise IoError(IoErrorCode.unknown_grid_kind, f"unknown grid_kind '{kind}'")
    if len(buf) - off != C * nlat * nlon * 8:
        raise IoError(IoErrorCode.payload_length_mismatch, "payload length mismatch")
    data = np.frombuffer(buf, dtype="<f8", offset=off).reshape(C, nlat, nlon)
    if device is not None:
        import torch
        data = torch.from_numpy(data.astype(np.float32)).to(device)
    else:
        data = data.copy()
    return SfdContents(S.SphericalField(grid, data), names)


# ----------------------------------------------------------------- weights
@dataclass
class NamedTensor:
    name: str
    shape: List[int]
    data: np.ndarray = dc_field(repr=False)


def write_weights(path, tensors: Sequence[NamedTensor], meta: Optional[dict] = None) -> None:
    """sfd.hpp:183-206."""
    lst, offset, payload = [], 0, []
    for t in tensors:
        d = np.ascontiguousarray(np.asarray(t.data, dtype="<f8")).reshape(-1)
        n = int(np.prod(t.shape)) if len(t.shape) else 1
        if n != d.size:
            raise IoError(IoErrorCode.header_mismatch, f"tensor shape does not match data: {t.name}")
        lst.append({"name": t.name, "shape": [int(s) for s in t.shape], "offset": offset})
        offset += n
        payload.append(d.tobytes())
    header = {"dtype": "f64le", "tensors": lst, "meta": meta if meta is not None else {}}
    with open(path, "wb") as f:
        f.write(_frame(b"SWB1", header))
        for p in payload:
            f.write(p)


@dataclass
class WeightsContents:
    tensors: List[NamedTensor]
    meta: Dict


def read_weights(path) -> WeightsContents:
    """sfd.hpp:213-243."""
    buf = _read(path)
    header, off = _parse_frame(buf, b"SWB1")
    try:
        meta = header.get("meta", {})
        tensors, total = [], 0
        for item in header["tensors"]:
            name, shape, toff = item["name"], [int(s) for s in item["shape"]], int(item["offset"])
            n = int(np.prod(shape)) if shape else 1
            if toff != total:
                raise IoError(IoErrorCode.header_mismatch, "non-contiguous tensor offsets")
            tensors.append(NamedTensor(name, shape, None))
            total += n
    except (KeyError, TypeError, ValueError):
        raise IoError(IoErrorCode.header_mismatch, "weights header field missing") from None
    if len(buf) - off != total * 8:
        raise IoError(IoErrorCode.payload_length_mismatch, "payload length mismatch")
    pos = off
    for t in tensors:
        n = int(np.prod(t.shape)) if t.shape else 1
        t.data = np.frombuffer(buf, dtype="<f8", offset=pos, count=n).reshape(t.shape).copy()
        pos += 8 * n
    return WeightsContents(tensors, meta)
