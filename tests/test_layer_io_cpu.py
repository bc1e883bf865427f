"""CPU tests of the L3DI codec, the palette type and map_value_to_color
(SPEC.md:171-194), and the oracle's display / pack definitions."""
import struct
import zlib
from types import SimpleNamespace

import numpy as np
import pytest

import paper_2501_14807_b200 as ml
from oracle import kn
from paper_2501_14807_b200 import layer_io


def _random_stream(rng, kind):
    w, h = int(rng.integers(1, 40)), int(rng.integers(1, 40))
    data = (rng.normal(size=(h, w)) * 100).astype(kind)
    mask = rng.random((h, w)) < 0.5
    npts = int(rng.integers(2, 6))
    pos = np.concatenate([[0.0], np.sort(rng.uniform(0.05, 0.95, npts - 2)), [1.0]])
    pal = ml.Palette(pos.astype(np.float32), rng.random((npts, 4)).astype(np.float32))
    table = "findings" if kind == "uint32" else None
    s = layer_io.encode_layer(kind, w, h, (-3.5, 12.25), pal, table, data.tobytes(), np.packbits(mask).tobytes())
    return s, data, mask, pal, table


@pytest.mark.parametrize("kind", layer_io.ELEMENT_KINDS)
def test_codec_round_trip_bit_identical(kind):
    rng = np.random.default_rng(hash(kind) % 1000)
    for _ in range(8):
        s, data, mask, pal, table = _random_stream(rng, kind)
        d = layer_io.decode_layer(s)
        assert d["kind"] == kind and (d["height"], d["width"]) == data.shape
        assert np.array_equal(d["data"].view(np.uint8), data.view(np.uint8))
        assert np.array_equal(np.unpackbits(d["mask_bits"])[:mask.size].reshape(mask.shape).astype(bool), mask)
        assert d["limits"] == (-3.5, 12.25) and d["table"] == table
        assert np.array_equal(d["palette"].positions, pal.positions) and np.array_equal(d["palette"].colours, pal.colours)
        assert layer_io.encode_layer(kind, d["width"], d["height"], d["limits"], d["palette"], d["table"],
                                     d["data"].tobytes(), d["mask_bits"].tobytes()) == s


def test_codec_layout_is_the_spec_field_list():
    pal = ml.Palette.grayscale()
    s = layer_io.encode_layer("int16", 3, 2, (0.0, 1.0), pal, None, np.arange(6, dtype="<i2").tobytes(), b"\xa8")
    assert s[:4] == b"L3DI"
    assert struct.unpack("<HBBII", s[4:16]) == (1, 0, layer_io.ELEMENT_KINDS.index("int16"), 3, 2)
    assert struct.unpack("<dd", s[16:32]) == (0.0, 1.0)
    assert struct.unpack("<H", s[32:34]) == (2,)
    assert struct.unpack("<5f", s[34:54]) == (0.0, 0.0, 0.0, 0.0, 1.0)
    assert struct.unpack("<H", s[74:76]) == (0,)                      # empty table name
    assert s[76:88] == np.arange(6, dtype="<i2").tobytes() and s[88:89] == b"\xa8"
    assert struct.unpack("<I", s[89:93])[0] == zlib.crc32(s[:89]) & 0xFFFFFFFF and len(s) == 93


def test_codec_errors():
    rng = np.random.default_rng(5)
    s, *_ = _random_stream(rng, "float32")
    with pytest.raises(ml.BadMagic):
        layer_io.decode_layer(b"X3DI" + s[4:])
    with pytest.raises(ml.TruncatedStream):
        layer_io.decode_layer(s[:len(s) // 2])
    with pytest.raises(ml.TruncatedStream):
        layer_io.decode_layer(s[:-1])
    with pytest.raises(ml.UnsupportedVersion):
        layer_io.decode_layer(s[:4] + struct.pack("<H", 2) + s[6:])
    bad = bytearray(s)
    bad[-10] ^= 0x40
    with pytest.raises(ml.ChecksumMismatch):
        layer_io.decode_layer(bytes(bad))


def test_palette_validation_and_json():
    with pytest.raises(ml.BadPalette):
        ml.Palette([0.0], [[0, 0, 0, 1]])
    with pytest.raises(ml.BadPalette):
        ml.Palette([0.0, 0.5, 0.5, 1.0], np.zeros((4, 4)))
    with pytest.raises(ml.BadPalette):
        ml.Palette([0.1, 1.0], np.zeros((2, 4)))
    with pytest.raises(ml.BadPalette):
        ml.Palette([0.0, 1.0], [[0, 0, 0, 1], [2, 0, 0, 1]])
    p = ml.Palette.from_json([{"position": 0, "rgba": [0, 0, 0, 1]}, {"position": 1, "rgba": [1, 1, 1, 1]}])
    assert p.positions.tolist() == [0.0, 1.0]


def test_map_value_to_color_known_answers():
    layer = SimpleNamespace(limits=(0.0, 10.0), palette=ml.Palette.grayscale())
    assert ml.map_value_to_color(layer, 0) == (0.0, 0.0, 0.0, 1.0)
    assert ml.map_value_to_color(layer, 5) == (0.5, 0.5, 0.5, 1.0)
    assert ml.map_value_to_color(layer, 25) == (1.0, 1.0, 1.0, 1.0)
    assert ml.map_value_to_color(layer, -4) == (0.0, 0.0, 0.0, 1.0)
    three = SimpleNamespace(limits=(0.0, 1.0), palette=ml.Palette([0, 0.25, 1], [[1, 0, 0, 1], [0, 1, 0, 1], [0, 0, 1, 0]]))
    assert ml.map_value_to_color(three, 0.25) == (0.0, 1.0, 0.0, 1.0)  # exact at control points
    a, b = ml.map_value_to_color(three, 0.3), ml.map_value_to_color(three, 0.6)
    assert a[1] > b[1] and a[2] < b[2]                                  # monotone per channel between points


def test_oracle_display_matches_map_value_to_color():
    rng = np.random.default_rng(7)
    pal = ml.Palette([0, 0.2, 0.7, 1], rng.random((4, 4)))
    layer = SimpleNamespace(limits=(-2.0, 6.0), palette=pal)
    data = rng.uniform(-4, 8, size=(16, 16)).astype(np.float32)
    mask = (rng.random((16, 16)) < 0.7).astype(np.uint8)
    out = kn.resolve_display(data, mask, -2.0, 6.0, pal.positions, pal.colours)
    assert (out[mask == 0] == 0).all()
    for y, x in zip(*np.nonzero(mask)):
        want = [int(np.floor(c * 255 + 0.5)) for c in ml.map_value_to_color(layer, float(data[y, x]))]
        assert out[y, x].tolist() == want
    assert np.array_equal(kn.pack_mask(mask), np.packbits(mask))
