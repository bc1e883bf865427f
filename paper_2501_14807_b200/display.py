"""Palette-based colourisation of layers.

``Palette`` / ``map_value_to_color`` are host-side (a handful of control points);
``resolve_display`` is a per-texel stream and runs in ``libmeshlayers_b200.so``.
"""
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import BadPalette


@dataclass
class Palette:
    """ordered control points (position in [0,1], RGBA in [0,1]); at least two,
    positions strictly increasing, first = 0, last = 1, colours finite."""
    positions: np.ndarray
    colours: np.ndarray

    def __post_init__(self):
        self.positions = np.ascontiguousarray(self.positions, dtype=np.float64).reshape(-1)
        self.colours = np.ascontiguousarray(self.colours, dtype=np.float64).reshape(-1, 4)
        p, c = self.positions, self.colours
        if len(p) < 2 or len(p) != len(c) or len(p) > 64:
            raise BadPalette("palette needs 2..64 control points with one RGBA colour each")
        if p[0] != 0.0 or p[-1] != 1.0 or not np.all(np.diff(p) > 0):
            raise BadPalette("positions must increase strictly from 0 to 1")
        if not np.all(np.isfinite(c)) or c.min() < 0.0 or c.max() > 1.0:
            raise BadPalette("colours must be finite and within [0, 1]")

    @classmethod
    def grayscale(cls):
        return cls([0.0, 1.0], [[0, 0, 0, 1], [1, 1, 1, 1]])

    @classmethod
    def from_json(cls, points):
        """JSON array of {position, rgba}."""
        return cls([p["position"] for p in points], [p["rgba"] for p in points])


def map_value_to_color(layer, value):
    """u = clamp((value-lower)/(upper-lower), 0, 1); piecewise-linear palette."""
    lo, hi = layer.limits
    pal = layer.palette
    u = (float(value) - lo) / (hi - lo)
    u = 0.0 if not u > 0.0 else min(u, 1.0)
    k = 0
    while k + 2 < len(pal.positions) and u > pal.positions[k + 1]:
        k += 1
    t = (u - pal.positions[k]) / (pal.positions[k + 1] - pal.positions[k])
    return tuple(float(v) for v in pal.colours[k] + t * (pal.colours[k + 1] - pal.colours[k]))


def resolve_display(layer, out=None):
    """RGBA8 plane (rows, width, 4) on the device; mask false -> transparent."""
    lo, hi = layer.limits
    return _native.resolve_display(layer.data, layer.mask, lo, hi, layer.palette.positions, layer.palette.colours,
                                   out=out)
