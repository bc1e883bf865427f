"""Independent brute-force checkers -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Pure Python, small cases only, in the spirit of SPEC.md:62, 70, 283 ("brute-force per-pixel
oracle").  They do NOT restate the reference's floating-point expressions: coverage is decided in
EXACT rational arithmetic (``fractions.Fraction``) from the geometric definition -- the texel
centre (x+0.5, y+0.5) lies inside the triangle, with the top-left rule of SPEC.md:114-117 /
KN:44-47 on the edges -- so they are a second opinion on the C restatement (``kn_port.c``) wherever
floating-point rounding cannot flip an edge sign, which is the case for inputs on a coarse binary
grid (all products exact in float64).  ``tests/test_oracle_pinned.py`` uses such inputs.
"""
from fractions import Fraction

import numpy as np


def _ccw(tri):
    (x0, y0), (x1, y1), (x2, y2) = tri
    a2 = (x1 - x0) * (y2 - y0) - (y1 - y0) * (x2 - x0)
    if a2 == 0:
        return None
    return tri if a2 > 0 else [tri[0], tri[2], tri[1]]                   # KN:32-41


def _accepts_tie(ax, ay, bx, by):
    dx, dy = bx - ax, by - ay
    return dy < 0 or (dy == 0 and dx < 0)                                 # KN:44-47


def covers(tri, x, y):
    """Exact: does the CCW-normalised triangle cover the centre of texel (x, y)?"""
    t = _ccw([(Fraction(float(px)), Fraction(float(py))) for px, py in tri])
    if t is None:
        return False
    cx, cy = Fraction(2 * x + 1, 2), Fraction(2 * y + 1, 2)
    for a, b in ((t[1], t[2]), (t[2], t[0]), (t[0], t[1])):              # edge i is opposite vertex i (KN:72-74)
        e = (b[0] - a[0]) * (cy - a[1]) - (b[1] - a[1]) * (cx - a[0])
        if e < 0 or (e == 0 and not _accepts_tie(a[0], a[1], b[0], b[1])):
            return False
    return True


def coverage(tri_xy, width, height):
    """(height, width) uint8 plane: 1 where some triangle covers the texel centre."""
    out = np.zeros((height, width), np.uint8)
    for tri in np.asarray(tri_xy, dtype=np.float64):
        for y in range(height):
            for x in range(width):
                if not out[y, x] and covers(tri, x, y):
                    out[y, x] = 1
    return out


def owner(tri_xy, width, height):
    """(height, width) int32 plane: largest index of a covering triangle, -1 if none."""
    out = np.full((height, width), -1, np.int32)
    for t, tri in enumerate(np.asarray(tri_xy, dtype=np.float64)):
        for y in range(height):
            for x in range(width):
                if covers(tri, x, y):
                    out[y, x] = t
    return out


def outline(cov, thickness):
    """uncovered texels within Chebyshev distance ``thickness`` of a covered one."""
    h, w = cov.shape
    out = np.zeros((h, w), np.uint8)
    for y in range(h):
        for x in range(w):
            if cov[y, x]:
                continue
            y0, y1, x0, x1 = max(0, y - thickness), min(h, y + thickness + 1), max(0, x - thickness), min(w, x + thickness + 1)
            out[y, x] = 1 if cov[y0:y1, x0:x1].any() else 0
    return out
