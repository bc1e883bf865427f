"""CPU checks of the FROZEN definitions of the north-star operations (oracle/kn_port.c ext_*):
independent numpy restatements on small cases plus the SPEC known answers that anchor them.
These ops have no reference code ("parity unpinned"); this file documents what they mean."""
import numpy as np
import pytest

from oracle import kn
from paper_2501_14807_b200 import synth


def _brute_surface(tri_xy, P, N, w, h):
    """Per-texel loop over triangles in submission order, float64 numpy, same formulas."""
    tri_id = -np.ones((h, w), np.int32)
    pos = np.full((3, h, w), np.nan, np.float32)
    area = np.zeros((h, w), np.float32)
    frags = 0
    for t in range(len(tri_xy)):
        xy = tri_xy[t].astype(np.float64)
        a2 = (xy[1, 0] - xy[0, 0]) * (xy[2, 1] - xy[0, 1]) - (xy[1, 1] - xy[0, 1]) * (xy[2, 0] - xy[0, 0])
        if a2 == 0.0:
            continue
        order = [0, 2, 1] if a2 < 0 else [0, 1, 2]
        v, p = xy[order], P[t][order].astype(np.float64)
        (x0, y0), (x1, y1), (x2, y2) = v
        ties = lambda ax, ay, bx, by: (by - ay) < 0 or ((by - ay) == 0 and (bx - ax) < 0)
        t0, t1, t2 = ties(x1, y1, x2, y2), ties(x2, y2, x0, y0), ties(x0, y0, x1, y1)
        for y in range(h):
            for x in range(w):
                cx, cy = x + 0.5, y + 0.5
                e0 = (x2 - x1) * (cy - y1) - (y2 - y1) * (cx - x1)
                e1 = (x0 - x2) * (cy - y2) - (y0 - y2) * (cx - x2)
                e2 = (x1 - x0) * (cy - y0) - (y1 - y0) * (cx - x0)
                if not ((e0 > 0 or (e0 == 0 and t0)) and (e1 > 0 or (e1 == 0 and t1)) and (e2 > 0 or (e2 == 0 and t2))):
                    continue
                frags += 1
                es = (e0 + e1) + e2
                l0, l1, l2 = e0 / es, e1 / es, e2 / es
                tri_id[y, x] = t
                pos[:, y, x] = ((l0 * p[0] + l1 * p[1]) + l2 * p[2]).astype(np.float32)
                cr = np.cross(p[1] - p[0], p[2] - p[0])
                a3 = np.sqrt((cr[0] * cr[0] + cr[1] * cr[1]) + cr[2] * cr[2]) * 0.5
                area[y, x] = np.float32(a3 / (abs(a2) * 0.5))
    return tri_id, pos, area, frags


def test_surface_map_definition_matches_bruteforce():
    rng = np.random.default_rng(2)
    w, h = 24, 20
    tri_xy = synth.random_soup(rng, 25, float(w))
    P = rng.normal(size=(25, 3, 3))
    N = rng.normal(size=(25, 3, 3))
    got = kn.surface_map(tri_xy, P, N, w, h)
    tri_id, pos, area, frags = _brute_surface(tri_xy, P, N, w, h)
    assert np.array_equal(got["tri_id"], tri_id)
    assert np.array_equal(got["pos"].view(np.uint32), pos.view(np.uint32))
    assert np.array_equal(got["area"].view(np.uint32), area.view(np.uint32))
    assert got["covered"] == int((tri_id >= 0).sum()) and got["overlap"] == frags - got["covered"]
    # normals are unit length where covered, zero elsewhere
    ln = np.sqrt((got["nrm"].astype(np.float64) ** 2).sum(axis=0))
    assert np.allclose(ln[tri_id >= 0], 1.0, atol=1e-6) and (ln[tri_id < 0] == 0).all()
    # row slabs are sub-ranges of the full map
    part = kn.surface_map(tri_xy, P, N, w, h, rows=(7, 15))
    assert np.array_equal(part["tri_id"], tri_id[7:15]) and np.array_equal(part["area"], got["area"][7:15])


def test_area_anchors():
    """flat 1 m^2 square fully covering a 2048^2 atlas -> 1e4/2048^2 cm^2 per texel."""
    sq_xy = lambda n: np.array([[[0, 0], [n, 0], [n, n]], [[0, 0], [n, n], [0, n]]], float)
    P = np.array([[[0, 0, 0], [1, 0, 0], [1, 1, 0]], [[0, 0, 0], [1, 1, 0], [0, 1, 0]]], float)
    assert kn.mesh_surface_area(P) == 1.0 and kn.mesh_surface_area(P[:1]) == 0.5
    n = 256
    s = kn.surface_map(sq_xy(n), P, P * 0 + [0, 0, 1.0], n, n)
    assert s["covered"] == n * n and s["overlap"] == 0
    a, c = kn.layer_area(s["area"], np.ones((n, n), np.uint8))
    assert c == n * n and abs(a - 1.0) < 1e-9
    assert abs(a / c * 1e4 - 1e4 / n ** 2) < 1e-9
    assert abs(1e4 / 2048 ** 2 - 0.00238418579) < 1e-9                       # SPEC.md:539 figure


def test_select_sphere_definition():
    rng = np.random.default_rng(3)
    pos = rng.normal(size=(3, 9, 13)).astype(np.float32)
    pos[:, rng.random((9, 13)) < 0.2] = np.nan
    c, r = (0.2, -0.1, 0.3), 1.1
    d = pos.astype(np.float64)
    d2 = ((d[0] - c[0]) ** 2 + (d[1] - c[1]) ** 2) + (d[2] - c[2]) ** 2
    hit = d2 <= r * r
    data = np.full((9, 13), 4, np.int16); mask = np.zeros((9, 13), bool); ed = np.zeros((9, 13), np.uint8)
    ed[0, :] = 1
    n = kn.select_sphere(pos, c, r, data, mask, ed, -9)
    assert n == int((hit & (np.arange(9)[:, None] > 0)).sum())               # row 0 was already edited
    assert np.array_equal(mask, hit) and np.array_equal(data == -9, hit)
    assert np.array_equal(ed != 0, hit | (np.arange(9)[:, None] == 0))


def test_select_threshold_definition():
    attr = np.array([[0.0, 0.5, 1.0, np.nan, 2.0]], np.float32)
    valid = np.array([[1, 1, 1, 1, 0]], np.uint8)
    data = np.zeros((1, 5), np.uint8); mask = np.zeros((1, 5), bool); ed = np.zeros((1, 5), np.uint8)
    assert kn.select_threshold(attr, valid, 0.5, 2.0, data, mask, ed, 3) == 2      # closed interval, NaN never hits
    assert data.tolist() == [[0, 3, 3, 0, 0]]
    assert kn.select_threshold(attr, None, 0.5, 2.0, data, mask, ed, 3) == 1       # without valid the last texel hits


@pytest.mark.parametrize("op,mask_fn", [("union", lambda a, b: a | b), ("intersection", lambda a, b: a & b),
                                        ("difference", lambda a, b: a & ~b), ("masking", lambda a, b: a & b)])
def test_layer_op_truth_table(op, mask_fn):
    ma = np.array([0, 0, 1, 1, 7, 0], np.uint8)          # any non-zero byte is true
    mb = np.array([0, 1, 0, 1, 1, 9], np.uint8)
    da = np.array([10, 11, 12, 13, 14, 15], np.uint16)
    db = np.array([20, 21, 22, 23, 24, 25], np.uint16)
    dc = np.zeros(6, np.uint16); mc = np.zeros(6, np.uint8)
    kn.layer_op(op, da, ma, db, mb, dc, mc)
    a, b = ma != 0, mb != 0
    m = mask_fn(a, b)
    assert np.array_equal(mc, m.astype(np.uint8))
    want = np.where(a, da, np.where(b, db, 0)) if op == "union" else np.where(m, da, 0)
    assert np.array_equal(dc, want)


def test_outline_and_padding_known_answers():
    cov = np.zeros((64, 64), np.uint8)
    cov[20:30, 30:40] = 1
    out = kn.outline(cov, 1)
    assert out.sum() == 44 and not (out & cov).any()
    assert kn.outline(np.ones((8, 8), np.uint8), 1).sum() == 0
    assert kn.outline(cov, 2).sum() == 14 * 14 - 100
    edited = np.zeros((64, 64), np.uint8)
    edited[25, 35] = 1                                                           # >= 2 texels from any outline texel
    data = np.zeros((64, 64), np.uint8); mask = np.zeros((64, 64), bool)
    assert kn.padding(out, edited, 1, data, mask, 5) == 0
    edited[:] = 0
    edited[20, 30] = 1                                                           # island corner
    assert kn.padding(out, edited, 1, data, mask, 5) == 5                        # 3 + 3 - 1 corner neighbours
    assert kn.padding(out, edited, 0, data, mask, 5) == 0
    assert mask.sum() == 5 and (data[mask] == 5).all() and not (mask & (cov != 0)).any()
