"""Layer persistence: the ``L3DI`` stream of SPEC.md:204-221.

Layout (little endian), exactly the field list of SPEC.md:221:

    "L3DI" | u16 version=1 | u8 kind (0 numeric, 1 database) | u8 element kind | u32 width | u32 height |
    f64 lower | f64 upper | u16 npoints | npoints x (f32 position, 4 x f32 rgba) |
    u16 table-name length + UTF-8 bytes (empty for numeric layers) |
    raw data plane (row-major) | mask as packed bits (row-major, MSB first, zero padded) | u32 CRC32

The CRC32 (zlib polynomial) covers every byte before the trailer.  Element-kind codes follow
SPEC.md:164's list order: int8 0, int16 1, int32 2, float16 3, float32 4, uint32 5 (database keys),
uint8 6.  The spec's field list carries no layer NAME; it travels beside the stream
(``load_layer(..., name=)``).  The codec itself (``encode_layer`` / ``decode_layer``) is pure host code
on numpy arrays; ``save_layer`` / ``load_layer`` move planes to and from the device and pack /
unpack the mask bits ON the device so only n/8 mask bytes cross PCIe.
"""
import struct
import zlib

import numpy as np

from . import _native
from .display import Palette
from .errors import BadMagic, ChecksumMismatch, TruncatedStream, UnsupportedVersion

MAGIC = b"L3DI"
VERSION = 1
ELEMENT_KINDS = ("int8", "int16", "int32", "float16", "float32", "uint32", "uint8")


def encode_layer(kind, width, height, limits, palette, table, data_bytes, mask_bits):
    """Assemble the stream from host pieces.  ``data_bytes``: raw little-endian plane bytes;
    ``mask_bits``: packed mask bytes ((w*h+7)//8)."""
    if kind not in ELEMENT_KINDS:
        raise ValueError("unknown element kind %r" % (kind,))
    name = (table or "").encode("utf-8")
    head = [MAGIC, struct.pack("<HBBII", VERSION, 1 if kind == "uint32" and table else 0, ELEMENT_KINDS.index(kind),
                               width, height),
            struct.pack("<dd", float(limits[0]), float(limits[1])), struct.pack("<H", len(palette.positions))]
    for p, c in zip(palette.positions, palette.colours):
        head.append(struct.pack("<5f", p, *c))
    head.append(struct.pack("<H", len(name)) + name)
    body = b"".join(head) + bytes(data_bytes) + bytes(mask_bits)
    return body + struct.pack("<I", zlib.crc32(body) & 0xFFFFFFFF)


def decode_layer(stream):
    """Inverse of ``encode_layer`` -> dict(kind, width, height, limits, palette, table, data, mask_bits)."""
    buf = bytes(stream)
    if len(buf) < 4 or buf[:4] != MAGIC:
        if len(buf) < 4 and MAGIC.startswith(buf):
            raise TruncatedStream("stream ends inside the magic")
        raise BadMagic("not an L3DI stream")
    pos = 4

    def take(n):
        nonlocal pos
        if pos + n > len(buf):
            raise TruncatedStream("stream truncated at byte %d" % len(buf))
        out = buf[pos:pos + n]
        pos += n
        return out

    version, layer_kind, ekind, width, height = struct.unpack("<HBBII", take(12))
    if version != VERSION:
        raise UnsupportedVersion("L3DI version %d" % version)
    if ekind >= len(ELEMENT_KINDS):
        raise UnsupportedVersion("unknown element kind code %d" % ekind)
    lower, upper = struct.unpack("<dd", take(16))
    (npoints,) = struct.unpack("<H", take(2))
    pts = np.frombuffer(take(20 * npoints), dtype="<f4").reshape(npoints, 5).astype(np.float64)
    (nlen,) = struct.unpack("<H", take(2))
    table = take(nlen).decode("utf-8")
    kind = ELEMENT_KINDS[ekind]
    n = width * height
    data = np.frombuffer(take(n * np.dtype(kind).itemsize), dtype=np.dtype(kind).newbyteorder("<")).reshape(height, width)
    mask_bits = np.frombuffer(take((n + 7) // 8), dtype=np.uint8)
    (crc,) = struct.unpack("<I", take(4))
    if crc != (zlib.crc32(buf[:pos - 4]) & 0xFFFFFFFF):
        raise ChecksumMismatch("CRC32 mismatch")
    return dict(kind=kind, database=bool(layer_kind), width=width, height=height, limits=(lower, upper),
                palette=Palette(pts[:, 0], pts[:, 1:]), table=table or None, data=data, mask_bits=mask_bits)


def _plane_to_host(t):
    torch = _native._torch()
    if t.dtype == torch.uint32:
        return t.view(torch.int32).cpu().numpy().view(np.uint32)
    return t.cpu().numpy()


def save_layer(layer):
    """SPEC.md:204-213 -> bytes.  The mask is bit-packed on the device before the copy."""
    bits = _native.pack_mask(layer.mask).cpu().numpy()
    data = np.ascontiguousarray(_plane_to_host(layer.data))
    return encode_layer(layer.kind, layer.width, layer.height, layer.limits, layer.palette, layer.table,
                        data.astype(data.dtype.newbyteorder("<"), copy=False).tobytes(), bits.tobytes())


def load_layer(stream, name="layer", pool=None):
    """bytes -> InformationLayer on the device (bit-identical planes)."""
    from .layer_core import create_layer
    torch = _native.require_cuda()
    d = decode_layer(stream)
    layer = create_layer(name, d["kind"], d["width"], d["height"], palette=d["palette"], limits=d["limits"],
                         pool=pool, table=d["table"])
    host = np.ascontiguousarray(d["data"])
    if d["kind"] == "uint32":
        layer.data.view(torch.int32).copy_(torch.from_numpy(host.view(np.int32).copy()))
    else:
        layer.data.copy_(torch.from_numpy(host.copy()))
    bits = torch.from_numpy(d["mask_bits"].copy()).to(layer.mask.device)
    _native.unpack_mask(bits, d["width"] * d["height"], layer.mask)
    return layer
