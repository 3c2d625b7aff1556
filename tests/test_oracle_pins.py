"""Pins for the CPU oracle (oracle/oracle.c) against things other than itself:
published known-answer vectors, a library routine (the CUDA toolkit's host
Philox), closed forms, invariants, textbook special cases and brute force on
tiny scenes.  CPU only (-m "not gpu").  DESIGN.md §3 lists, per oracle step,
which test here pins it.
"""
from __future__ import annotations

import math
import subprocess
from pathlib import Path

import numpy as np
import pytest

import oracle
import scenegen

HERE = Path(__file__).resolve().parent
INV_PI32 = np.float32(1.0 / math.pi)


@pytest.fixture(autouse=True, params=["default", "o0"])
def oracle_variant(request):
    """Every pin runs against both oracle builds: the default one (readings
    R25/R26) and the frozen O0 one (SPEC S:134-150 MT, no fma)."""
    oracle.set_default_variant(request.param)
    yield request.param
    oracle.set_default_variant("default")


# ---------------------------------------------------------------- helpers
def F_c(X, Y):
    """Point-to-parallel-rectangle form factor for a point under the corner of
    an X x Y (normalised by height) rectangle (standard closed form; Howell's
    catalogue C-11 restated)."""
    a = X / math.sqrt(1 + X * X) * math.atan(Y / math.sqrt(1 + X * X))
    b = Y / math.sqrt(1 + Y * Y) * math.atan(X / math.sqrt(1 + Y * Y))
    return (a + b) / (2 * math.pi)


def tiny_scene(verts, albedo=None, lights=None, cam=None, W=8, H=8, **kw):
    verts = np.asarray(verts, np.float64).reshape(-1, 3, 3)
    if albedo is None:
        albedo = np.full((verts.shape[0], 3), 0.5)
    if lights is None:
        lights = scenegen.make_light([0.0, 1.999, 0.0])
    if cam is None:
        cam = scenegen.make_camera([0.0, 1.0, -3.0], [0.0, 0.0, 0.0], 60.0, W, H)
    return scenegen.custom_scene(verts, albedo, lights, cam, W, H, **kw)


def floor_quad(half=2.0, y=0.0):
    return scenegen.quad_tris([-half, y, -half], [0, 0, 2 * half], [2 * half, 0, 0])   # normal +y


# ---------------------------------------------------------------- Philox (O0)
def test_philox_known_answer_vectors():
    rows = [l.split() for l in (HERE / "golden/philox4x32_10_kat.txt").read_text().splitlines()
            if l.strip() and not l.startswith("#")]
    assert len(rows) == 3
    for r in rows:
        v = [int(x, 16) for x in r]
        assert oracle.philox(v[0:4], v[4:6]).tolist() == v[6:10]


def test_philox_matches_cuda_toolkit_host_routine(tmp_path):
    exe = tmp_path / "pcu"
    subprocess.check_call(["g++", "-O1", "-I/usr/local/cuda/include", "-x", "c++",
                           str(HERE / "philox_curand_host.cpp"), "-o", str(exe)])
    rng = np.random.default_rng(7)
    ins = rng.integers(0, 2**32, (200, 6), dtype=np.uint64)
    ins[:4, 0] = [0, 1, 2, 3]
    txt = "\n".join(" ".join(f"{int(x):08x}" for x in r) for r in ins)
    out = subprocess.run([str(exe)], input=txt, capture_output=True, text=True, check=True).stdout
    ref = [[int(x, 16) for x in l.split()] for l in out.strip().splitlines()]
    for r, e in zip(ins, ref):
        assert oracle.philox(r[:4], r[4:6]).tolist() == e


def test_draw_lane_and_counter_layout():
    seed = 0x123456789ABCDEF
    key = [seed & 0xFFFFFFFF, seed >> 32]
    for stream, item, j in [(0, 0, 0), (1, 77, 5), (0, 3, 11), (2, 2**31, 6)]:
        blk = oracle.philox([j >> 2, item, stream, 0], key)
        assert oracle.draw(seed, stream, item, j) == int(blk[j & 3])


# ---------------------------------------------------------------- O1 triangle prep
def test_unit_right_triangle_area_normal_centroid():
    s = tiny_scene([[0, 0, 0], [1, 0, 0], [0, 1, 0]])
    o = oracle.OracleScene(s)
    td = o.tri_data()
    assert td["area"][0] == np.float32(0.5)
    assert td["normal"][0].tolist() == [0.0, 0.0, 1.0]
    assert np.allclose(td["centroid"][0], [1 / 3, 1 / 3, 0], atol=1e-7)
    assert int(td["aq"][0]) == 2**39                        # 0.5 * 2^40
    assert o.bad == -1


def test_degenerate_triangle_is_named():
    V = [[[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0, 0, 0], [1, 1, 1], [2, 2, 2]],
         [[0, 0, 0], [0, 0, 1], [1, 0, 0]]]
    o = oracle.OracleScene(tiny_scene(V))
    assert o.bad == 1


def test_total_area_permutation_invariant_and_matches_float64():
    s = scenegen.make_scene(2)
    td = oracle.OracleScene(s).tri_data()
    perm = np.random.default_rng(0).permutation(s.n_tris)
    s2 = scenegen.custom_scene(s.verts[perm], s.albedo[perm], s.lights, s.cam, s.width, s.height)
    td2 = oracle.OracleScene(s2).tri_data()
    assert int(td["aq"].sum()) == int(td2["aq"].sum())
    v = s.verts.astype(np.float64)
    a64 = 0.5 * np.linalg.norm(np.cross(v[:, 1] - v[:, 0], v[:, 2] - v[:, 0]), axis=1)
    assert np.allclose(td["area"], a64, rtol=2e-6)
    n64 = np.cross(v[:, 1] - v[:, 0], v[:, 2] - v[:, 0]) / (2 * a64[:, None])
    assert np.allclose(td["normal"], n64, atol=2e-6)
    assert np.allclose(td["centroid"], v.mean(1), atol=1e-6)


# ---------------------------------------------------------------- O9 MT / visibility
def test_closest_hit_closed_form_plane():
    s = tiny_scene(floor_quad(2.0, y=0.0))
    o = oracle.OracleScene(s)
    idx, t = o.closest_hit([0.3, 1.5, 0.2], [0.0, -1.0, 0.0])
    assert idx in (0, 1) and t == np.float32(1.5)
    d = np.array([0.6, -0.8, 0.0], np.float32)
    idx, t = o.closest_hit([0.0, 2.0, 0.0], d)
    assert abs(float(t) - 2.5) < 1e-6
    assert o.closest_hit([0, 1, 0], [1, 0, 0])[0] == -1     # parallel -> none
    assert o.closest_hit([0, 1, 0], [0, -1, 0], 0.0, 0.5)[0] == -1   # short t_max
    assert o.closest_hit([0, 1, 0], [0, 1, 0])[0] == -1     # pointing away


def test_closest_hit_tie_breaks_on_lowest_index():
    q = floor_quad(1.0)
    V = np.concatenate([q, q])                              # duplicated plane: equal t
    o = oracle.OracleScene(tiny_scene(V))
    idx, t = o.closest_hit([0.2, 1.0, 0.4], [0, -1, 0])
    assert idx in (0, 1) and t == np.float32(1.0)


def test_visibility_wall_empty_and_symmetry():
    wall = scenegen.quad_tris([-1, -1, 0.0], [2, 0, 0], [0, 2, 0])
    o = oracle.OracleScene(tiny_scene(wall))
    assert o.occluded([0, 0, -1], [0, 0, 1])
    assert o.occluded([0, 0, 1], [0, 0, -1])                # two-sided
    assert not o.occluded([0, 0, -1], [0, 0, -3])
    assert not o.occluded([2, 0, -1], [2, 0, 1])            # passes beside the wall
    s = scenegen.make_scene(1)
    o = oracle.OracleScene(s)
    rng = np.random.default_rng(3)
    a = rng.uniform(0.05, 1.95, (500, 3)).astype(np.float32)
    b = rng.uniform(0.05, 1.95, (500, 3)).astype(np.float32)
    assert (o.occluded_batch(a, b) == o.occluded_batch(b, a)).mean() > 0.995


def test_visibility_matches_float64_geometry_of_boxes():
    """Brute force vs hand geometry (float64 segment/box slab test) on random
    segments in the C1 room, away from box surfaces."""
    s = scenegen.make_scene(1)
    o = oracle.OracleScene(s)
    V = s.verts.astype(np.float64)
    boxes = [V[10 + 12 * k:22 + 12 * k].reshape(-1, 3) for k in range(2)]
    lo = [b.min(0) for b in boxes]
    hi = [b.max(0) for b in boxes]
    rng = np.random.default_rng(11)
    n_checked = 0
    for _ in range(3000):
        a = rng.uniform(0.05, 1.95, 3)
        b = rng.uniform(0.05, 1.95, 3)
        inside = any(np.all(p > l - 0.02) and np.all(p < h + 0.02) for p in (a, b) for l, h in zip(lo, hi))
        if inside:
            continue
        hit, margin = False, np.inf
        for l, h in zip(lo, hi):
            d = b - a
            with np.errstate(divide="ignore", invalid="ignore"):
                t0, t1 = (l - a) / d, (h - a) / d
            tn, tf = np.nanmax(np.minimum(t0, t1)), np.nanmin(np.maximum(t0, t1))
            margin = min(margin, abs(tf - tn) * np.linalg.norm(d))
            if tn < tf and tf > 0 and tn < 1:
                hit = True
        if margin < 1e-3:
            continue
        n_checked += 1
        assert o.occluded(a.astype(np.float32), b.astype(np.float32)) == hit
    assert n_checked > 1500


# ---------------------------------------------------------------- O2 classification
def test_classify_hand_cases_and_partition():
    cam = scenegen.make_camera([0, 0, 0], [0, 0, 5], 60.0, 8, 8)
    V = [[[-0.1, -0.1, 1.0], [0.1, -0.1, 1.0], [0.0, 0.1, 1.0]],          # on axis at T/2 -> near
         [[-0.1, -0.1, -1.0], [0.1, -0.1, -1.0], [0.0, 0.1, -1.0]],       # behind -> far
         [[-0.1, -0.1, 3.0], [0.1, -0.1, 3.0], [0.0, 0.1, 3.0]],          # beyond T -> far
         [[2.9, -0.1, 1.0], [3.1, -0.1, 1.0], [3.0, 0.1, 1.0]]]           # outside FOV -> far
    s = tiny_scene(V, cam=cam, T=2.0)
    lab, nn = oracle.OracleScene(s).classify()
    assert lab.tolist() == [1, 0, 0, 0] and nn == 1


def test_classify_equals_float64_definition_away_from_boundary():
    s = scenegen.make_scene(3)
    o = oracle.OracleScene(s)
    lab, nn = o.classify()
    c = s.verts.astype(np.float64).mean(1)
    cam = s.cam.astype(np.float64)
    d = c - cam[0:3]
    z, x, y = d @ cam[3:6], d @ cam[9:12], d @ cam[6:9]
    m = np.minimum.reduce([z, z * cam[12] - abs(x), z * cam[13] - abs(y), s.T**2 - (d * d).sum(1)])
    ok = np.abs(m) > 1e-4
    assert ok.mean() > 0.99
    assert np.array_equal(lab[ok].astype(bool), (m > 0)[ok])
    assert nn == int(lab.sum()) and 0 < nn < s.n_tris


# ---------------------------------------------------------------- O4-O6 Morton, table, strata
def _interleave_magic(x):
    x = np.uint64(x) & np.uint64(0x3FF)
    x = (x | (x << np.uint64(16))) & np.uint64(0x030000FF)
    x = (x | (x << np.uint64(8))) & np.uint64(0x0300F00F)
    x = (x | (x << np.uint64(4))) & np.uint64(0x030C30C3)
    x = (x | (x << np.uint64(2))) & np.uint64(0x09249249)
    return x


def test_morton_examples_and_magic_bits():
    assert oracle.morton3(0, 0, 0) == 0
    assert oracle.morton3(3, 0, 0) == 9
    assert oracle.morton3(0, 1, 0) == 2 and oracle.morton3(0, 0, 1) == 4
    assert oracle.morton3(1023, 1023, 1023) == 2**30 - 1
    rng = np.random.default_rng(5)
    for q in rng.integers(0, 1024, (300, 3)):
        ref = int(_interleave_magic(q[0]) | (_interleave_magic(q[1]) << np.uint64(1)) |
                  (_interleave_magic(q[2]) << np.uint64(2)))
        assert oracle.morton3(*map(int, q)) == ref


def test_area_table_and_lookup_examples():
    # three triangles with areas 1, 2, 3 (x 2^-10 m^2 so the fixed point is exact)
    sc = 2.0**-5
    V = [[[0, 0, 0], [sc * 2, 0, 0], [0, sc, 0]],
         [[0, 0, 1], [sc * 4, 0, 1], [0, sc, 1]],
         [[0, 0, 2], [sc * 6, 0, 2], [0, sc, 2]]]
    o = oracle.OracleScene(tiny_scene(V))
    lit = np.ones(3, np.uint8)
    order, P, codes = o.near_table(lit)
    unit = 2**30
    assert sorted(order.tolist()) == [0, 1, 2]              # permutation
    areas = np.array([1, 2, 3])[order]
    assert P.tolist() == (np.cumsum(areas) * unit).tolist()
    assert np.all(np.diff(codes.astype(np.int64)) >= 0)
    Pt = np.array([1000, 3000, 6000], np.uint64)             # S:222-224 (x1000)
    assert oracle.lookup_g(Pt, 500) == 0
    assert oracle.lookup_g(Pt, 2500) == 1
    assert oracle.lookup_g(Pt, 5999) == 2
    assert oracle.lookup_g(Pt, 0) == 0 and oracle.lookup_g(Pt, 1000) == 1


def test_strata_lie_in_their_stratum_and_counts_bounded():
    seed, K = 77, 1000
    rng = np.random.default_rng(2)
    aq = rng.integers(1, 2**40, 300).astype(np.uint64)
    P = np.cumsum(aq).astype(np.uint64)
    F = int(P[-1])
    counts = np.zeros(300, np.int64)
    for k in range(K):
        sk = oracle.stratum(seed, k, K, F)
        assert k * F // K <= sk and sk * K < (k + 1) * F     # exact integer stratum bounds
        j = oracle.lookup_g(P, sk)
        assert (j == 0 or int(P[j - 1]) <= sk) and sk < int(P[j])   # f(m) <= s < f(m+1)
        counts[j] += 1
    assert counts.sum() == K
    expect = K * aq.astype(np.float64) / F
    assert np.all(counts >= np.floor(expect) - 1) and np.all(counts <= np.ceil(expect) + 1)


def test_morton_order_is_spatially_local():
    s = scenegen.make_scene(3)
    o = oracle.OracleScene(s)
    lit = np.ones(s.n_tris, np.uint8)
    order, P, codes = o.near_table(lit)
    c = s.verts.astype(np.float64).mean(1)
    d_morton = np.linalg.norm(np.diff(c[order], axis=0), axis=1).mean()
    d_input = np.linalg.norm(np.diff(c, axis=0), axis=1).mean()
    perm = np.random.default_rng(1).permutation(s.n_tris)
    d_random = np.linalg.norm(np.diff(c[perm], axis=0), axis=1).mean()
    assert d_morton <= d_input and d_morton < 0.1 * d_random  # S:286 (locality)
    assert np.array_equal(np.sort(order), np.arange(s.n_tris))


# ---------------------------------------------------------------- O7 point in triangle
def test_point_in_triangle_vertex_and_mean():
    V = [[[0, 0, 0], [1, 0, 0], [0, 1, 0]]]
    o = oracle.OracleScene(tiny_scene(V))
    assert o.point_in_tri(0, 0.0, 0.7).tolist() == [0.0, 0.0, 0.0]     # u1=0 -> v0
    # u1 -> 1 puts the point on the edge v1-v2 opposite v0: u2 = 0 -> v2, u2 -> 1 -> v1
    assert np.allclose(o.point_in_tri(0, 1.0 - 2**-24, 0.0), [0, 1, 0], atol=1e-6)
    assert np.allclose(o.point_in_tri(0, 1.0 - 2**-24, 1.0 - 2**-24), [1, 0, 0], atol=1e-6)
    rng = np.random.default_rng(9)
    u = rng.random((20000, 2)).astype(np.float32)
    pts = np.array([o.point_in_tri(0, a, b) for a, b in u])
    assert np.all(pts[:, 0] >= 0) and np.all(pts[:, 1] >= 0) and np.all(pts.sum(1) <= 1 + 1e-6)
    assert np.allclose(pts.mean(0), [1 / 3, 1 / 3, 0], atol=1e-2)


# ---------------------------------------------------------------- O8 Eq. 2, area-light form
def test_eq2_irradiance_matches_rectangle_form_factor():
    """A tiny lit patch under the centre of the 0.5 x 0.5 light at height H:
    E = Phi*pi/(rho*D) averaged over the strata must equal
    pi * L * 4 * F_c(0.25/H, 0.25/H) (0.61286 W/m^2 at H = 1.999, L = 10)."""
    h = 1e-3
    V = [[[-h, 0, -h], [-h, 0, h], [h, 0, -h]]]                         # faces +y
    cam = scenegen.make_camera([0.0, 1.0, -1.0], [0, 0, 0], 60.0, 8, 8)
    s = tiny_scene(V, albedo=[[0.5, 0.25, 0.75]], cam=cam, T=5.0, M=20000, K_near=20000, seed=5)
    o = oracle.OracleScene(s)
    lab, nn = o.classify()
    assert nn == 1
    v, info = o.generate_vpls(lab)
    assert info["K"] == 20000 and info["M_far"] == 0 and info["flags"] == 2    # EMPTY_FAR -> K = M
    area = float(o.tri_data()["area"][0])
    D = area / 20000
    E = v["flux"].astype(np.float64) * math.pi / (np.array([0.5, 0.25, 0.75]) * D)
    closed = math.pi * 10.0 * 4 * F_c(0.25 / 1.999, 0.25 / 1.999)
    assert abs(closed - 0.61286) < 1e-4
    for c in range(3):
        m, se = E[:, c].mean(), E[:, c].std() / math.sqrt(len(E))
        assert abs(m - closed) < 4 * se + 1e-4 * closed, (m, closed, se)


def test_eq2_fully_occluded_light_gives_zero_flux():
    h = 1e-2
    V = [[[-h, 0, -h], [-h, 0, h], [h, 0, -h]],
         *scenegen.quad_tris([-1, 1.0, -1], [2, 0, 0], [0, 0, 2])]      # blocker plane at y = 1
    cam = scenegen.make_camera([0.0, 0.5, -0.5], [0, 0, 0], 60.0, 8, 8)
    s = tiny_scene(V, cam=cam, T=5.0, M=64, K_near=64, seed=1)
    o = oracle.OracleScene(s)
    lab, _ = o.classify()
    lit = o.lit(lab)
    assert lit.sum() == 0                                     # centroid test already shadowed
    # force the near table through the generator with the light filter bypassed
    # by placing the blocker above the light instead: flux must then be > 0
    V2 = [V[0], *scenegen.quad_tris([-1, 2.5, -1], [2, 0, 0], [0, 0, 2])]
    o2 = oracle.OracleScene(tiny_scene(V2, cam=cam, T=5.0, M=64, K_near=64, seed=1))
    lab2, _ = o2.classify()
    v2, info2 = o2.generate_vpls(lab2)
    assert info2["K"] == 64 and np.all(v2["flux"] > 0)


def test_lit_uses_the_light_centre_point():
    """R6 ("visible to the light source"): the lit test is the
    centroid -> light-centre segment.  Hand geometry: a 4 cm blocker on that
    segment (1 m up) leaves every light-corner segment free, so a corner-point
    test would call the patch lit; a blocker on one corner segment only must
    leave it lit."""
    h = 1e-2
    recv = [[-h, 0, -h], [-h, 0, h], [h, 0, -h]]            # normal +y, centroid (-h/3, 0, -h/3)
    cam = scenegen.make_camera([0.0, 0.5, -0.5], [0, 0, 0], 60.0, 8, 8)

    def lit_of(blocker_centre):
        b = np.asarray(blocker_centre, np.float64) + [0.005, 0.0, -0.003]   # segment off the quad's diagonal
        V = [recv, *scenegen.quad_tris(b + [-0.02, 0, -0.02], [0.04, 0, 0], [0, 0, 0.04])]
        o = oracle.OracleScene(tiny_scene(V, cam=cam, T=5.0, M=64, K_near=64, seed=1))
        lab, _ = o.classify()
        assert lab[0] == 1
        return int(o.lit(lab)[0]), o

    c = np.array([-h / 3, 0.0, -h / 3])
    Lc = np.array([0.0, 1.999, 0.0])
    corners = [Lc + [sx * 0.25, 0, sz * 0.25] for sx in (-1, 1) for sz in (-1, 1)]
    # blocker on the centre segment: no corner segment meets it (float64 geometry), yet unlit
    at = c + (Lc - c) * (1.0 / 1.999)
    lit, o = lit_of(at)
    for q in corners:
        assert o.occluded(c.astype(np.float32), q.astype(np.float32)) is False
    assert o.occluded(c.astype(np.float32), Lc.astype(np.float32)) is True
    assert lit == 0
    # blocker on the (+x, +z) corner segment only: the centre segment is free, so lit
    q = corners[3]
    lit, o = lit_of(c + (q - c) * (1.0 / 1.999))
    assert o.occluded(c.astype(np.float32), q.astype(np.float32)) is True
    assert o.occluded(c.astype(np.float32), Lc.astype(np.float32)) is False
    assert lit == 1


def test_near_vpls_represent_equal_area_and_sit_on_lit_triangles():
    s = scenegen.make_scene(3)
    o = oracle.OracleScene(s)
    lab, _ = o.classify()
    lit = o.lit(lab)
    v, info = o.generate_vpls(lab)
    K = info["K"]
    near = v[:K]
    assert np.all(near["tag"] == 0) and np.all(lit[near["tri"]] == 1)
    assert np.all(v[K:]["tag"] == 1) and np.all(lab[v[K:]["tri"]] == 0)  # far deposits on far patches
    order, P, _ = o.near_table(lit)
    aq = o.tri_data()["aq"].astype(np.float64)
    cnt = np.bincount(near["tri"], minlength=s.n_tris)[order]
    expect = K * aq[order] / float(P[-1])
    assert cnt.sum() == K
    assert np.all(cnt >= np.floor(expect) - 1) and np.all(cnt <= np.ceil(expect) + 1)
    v2, info2 = o.generate_vpls(lab)                         # determinism
    assert info2 == info and v2.tobytes() == v.tobytes()


# ---------------------------------------------------------------- O10 walk energy invariants
def _closed_box(rho=0.5, n=4):
    V = scenegen.room_tris([0, 0, 0], [2, 2, 2], n=n)
    cam = scenegen.make_camera([1.0, 1.0, 0.1], [1, 1, 2], 60.0, 8, 8)
    return tiny_scene(V, albedo=np.full((V.shape[0], 3), rho), lights=scenegen.make_light([1.0, 1.999, 1.0]),
                      cam=cam, T=0.01, M=0, K_near=0, max_depth=4, rr=0, seed=21), V


def test_walk_energy_depth1_and_albedo_powers():
    s, V = _closed_box(rho=0.5)
    o = oracle.OracleScene(s)
    labels = np.zeros(s.n_tris, np.uint8)                    # everything FAR: plain IR
    nw = 4000
    v, info = o.generate_vpls(labels, n_walks_fixed=nw, rr=0, max_depth=4)
    assert info["n_walks"] == nw
    phi_tot = math.pi * 0.25 * 10.0                           # pi * A * L
    inc = v["flux"].astype(np.float64) * math.pi / 0.5        # incident power per deposit
    for d in range(1, 5):
        tot = inc[v["depth"] == d].sum(0)
        n_d = int((v["depth"] == d).sum())
        assert n_d >= nw * 0.999                              # closed box: every walk continues
        assert np.allclose(tot, (0.5 ** (d - 1)) * phi_tot * n_d / nw, rtol=1e-5), (d, tot)


def test_walk_first_hit_fractions_match_form_factors():
    s, V = _closed_box(rho=0.5, n=1)
    o = oracle.OracleScene(s)
    nw = 40000
    v, _ = o.generate_vpls(np.zeros(s.n_tris, np.uint8), n_walks_fixed=nw, rr=0, max_depth=1)
    walls = v["tri"] // 2                                     # room_tris order: floor, ceiling, x0, x2, z2, z0
    frac = np.bincount(walls, minlength=6) / nw
    # floor: signed 4-corner F_c quadrature over the floor (closed form per point)
    H = 1.999
    g = (np.arange(400) + 0.5) / 400 * 2.0
    X, Z = np.meshgrid(g, g)
    x0, x1 = (0.75 - X) / H, (1.25 - X) / H
    z0, z1 = (0.75 - Z) / H, (1.25 - Z) / H
    Fv = np.vectorize(F_c)
    Fpt = Fv(x1, z1) - Fv(x0, z1) - Fv(x1, z0) + Fv(x0, z0)
    floor_frac = (Fpt.mean() * 4.0) / 0.25                    # (1/A_L) * integral F_pt dA
    assert abs(floor_frac - 0.23681) < 2e-4
    se = math.sqrt(floor_frac * (1 - floor_frac) / nw)
    assert abs(frac[0] - floor_frac) < 4 * se
    wall = (1 - floor_frac) / 4
    for k in (2, 3, 4, 5):
        assert abs(frac[k] - wall) < 4 * math.sqrt(wall * (1 - wall) / nw)
    assert frac[1] == 0                                       # ceiling never hit


def test_walk_russian_roulette_unbiased():
    s, _ = _closed_box(rho=0.6)
    o = oracle.OracleScene(s)
    nw = 20000
    v, _ = o.generate_vpls(np.zeros(s.n_tris, np.uint8), n_walks_fixed=nw, rr=1, max_depth=3)
    inc = v["flux"][:, 0].astype(np.float64) * math.pi / 0.6
    phi_tot = math.pi * 0.25 * 10.0
    for d in (2, 3):
        per_walk = np.zeros(nw)
        sel = v["depth"] == d
        np.add.at(per_walk, v["walk"][sel], inc[sel] * nw)    # undo the 1/n division per walk
        m, se = per_walk.mean(), per_walk.std() / math.sqrt(nw)
        assert abs(m - phi_tot * 0.6 ** (d - 1)) < 4 * se + 1e-9


def test_walk_degenerate_cases():
    s, _ = _closed_box()
    o = oracle.OracleScene(s)
    v, info = o.generate_vpls(np.zeros(s.n_tris, np.uint8), M=0, K_near=0)
    assert len(v) == 0 and info["n_walks"] == 0               # count = 0 -> empty
    v, info = o.generate_vpls(np.ones(s.n_tris, np.uint8), n_walks_fixed=100)
    assert len(v) == 0                                        # restrict_to = {} -> empty


def test_budget_rule_first_mfar_deposits():
    s = scenegen.make_scene(1)
    o = oracle.OracleScene(s)
    lab, _ = o.classify()
    v, info = o.generate_vpls(lab)
    K, Mf = info["K"], info["M_far"]
    assert K + Mf == s.M and Mf == s.M - s.K_near
    far = v[K:]
    keys = far["walk"].astype(np.int64) * 16 + far["depth"]
    assert np.all(np.diff(keys) > 0)                          # (w, d) order
    assert far["walk"].max() == info["n_walks"] - 1
    # the same walks in fixed mode, divided by the same count, reproduce the prefix
    fixed, _ = o.generate_vpls(lab, n_walks_fixed=info["n_walks"])
    assert fixed[:Mf].tobytes() == far.tobytes()
    assert len(fixed) >= Mf


# ---------------------------------------------------------------- O12 G-buffer
def test_gbuffer_centre_ray_and_plane_hits():
    V = scenegen.quad_tris([-5, -5, 3.0], [0, 10, 0], [10, 0, 0])       # wall z = 3 facing -z
    cam = scenegen.make_camera([0, 0, 0], [0, 0, 1], 90.0, 5, 5)
    o = oracle.OracleScene(tiny_scene(V, cam=cam, W=5, H=5))
    gb = o.gbuffer(np.arange(25, dtype=np.int32))
    c = gb[12]
    assert c["t"] == np.float32(3.0) and c["pos"].tolist() == [0.0, 0.0, 3.0] and c["front"] == 1
    # pixel (px, py): direction through ((2(px+.5)/W - 1) tan, (1 - 2(py+.5)/H) tan, 1)
    for k in range(25):
        px, py = k % 5, k // 5
        sx = (2 * (px + 0.5) / 5 - 1) * 1.0
        sy = (1 - 2 * (py + 0.5) / 5) * 1.0
        hit = np.array([-sx * 3, sy * 3, 3.0])                # right = -x for this camera
        assert np.allclose(gb[k]["pos"], hit, atol=1e-5)
        assert abs(gb[k]["t"] - 3 * math.sqrt(1 + sx * sx + sy * sy)) < 1e-5


# ---------------------------------------------------------------- O13 gather closed forms
def _gather_setup(half=50.0):
    V = floor_quad(half)                                      # 100 m floor -> diag ~ 141 m, b^2 = 2
    s = tiny_scene(V, albedo=np.full((2, 3), 0.8))
    o = oracle.OracleScene(s)
    return s, o


def _gb(points, rho=0.8, tri=0):
    g = np.zeros(len(points), oracle.GBUF_DTYPE)
    g["pos"] = points
    g["nrm"] = [0, 1, 0]
    g["alb"] = rho
    g["tri"] = tri
    g["front"] = 1
    return g


def _vpl(pos, nrm=(0, -1, 0), flux=(1.0, 2.0, 3.0), tri=5):
    v = np.zeros(1, oracle.VPL_DTYPE)
    v["pos"], v["nrm"], v["flux"], v["tri"] = pos, nrm, flux, tri
    return v


def test_gather_single_vpl_over_plane_closed_form():
    s, o = _gather_setup()
    diag, eps, b2 = o.consts()
    h = 3.0
    assert h * h > b2
    sx = np.array([0.0, 0.5, 1.0, 2.5, 7.0])
    pts = np.stack([sx, np.zeros_like(sx), np.zeros_like(sx)], 1).astype(np.float32)
    r = o.gather(_gb(pts), _vpl([0.0, h, 0.0]))
    for k, x in enumerate(sx):
        expect = 0.8 / math.pi * np.array([1, 2, 3]) * h * h / (h * h + x * x) ** 2
        assert np.allclose(r["rgb64"][k], expect, rtol=1e-6)


def test_gather_clamp_behind_self_and_linearity():
    s, o = _gather_setup()
    diag, eps, b2 = o.consts()
    b2 = float(b2)
    h = 0.5 * math.sqrt(b2)                                   # r < b -> uses b^2 (R12)
    r = o.gather(_gb(np.zeros((1, 3), np.float32)), _vpl([0.0, h, 0.0]))
    h32 = float(np.float32(h))
    expect = 0.8 / math.pi * 1.0 * (h32 * h32) / (float(np.float32(h32 * h32)) * b2)
    assert abs(r["rgb64"][0, 0] - expect) / expect < 1e-6
    unclamped = 0.8 / math.pi / (h32 * h32)
    assert r["rgb64"][0, 0] < unclamped
    r = o.gather(_gb(np.zeros((1, 3), np.float32)), _vpl([0.0, -1.0, 0.0], nrm=(0, 1, 0)))
    assert r["rgb64"].max() == 0 and r["traced"] == 0         # VPL behind receiver
    r = o.gather(_gb(np.zeros((1, 3), np.float32), tri=5), _vpl([0.0, 1.0, 0.0], tri=5))
    assert r["rgb64"].max() == 0                              # self-triangle excluded (R14)
    vs = np.concatenate([_vpl([0.3, 1.0, 0.1]), _vpl([-0.5, 2.0, 0.4], flux=(0.5, 0.1, 0.2))])
    g = _gb(np.array([[0.0, 0, 0], [1.0, 0, 1.0]], np.float32))
    ra, rb, rab = o.gather(g, vs[:1]), o.gather(g, vs[1:]), o.gather(g, vs)
    assert np.allclose(ra["rgb64"] + rb["rgb64"], rab["rgb64"], rtol=1e-12)
    v2 = vs.copy()
    v2["flux"] *= 2
    assert np.allclose(o.gather(g, v2)["rgb64"], 2 * rab["rgb64"], rtol=1e-12)


def test_gather_power_over_square_matches_form_factor():
    """Sum of the pixel radiance * pi / rho over a fine grid on a centred
    square of half-width a integrates the VPL's emitted power onto the square:
    pi * Phi * 4 F_c(a/h, a/h)."""
    s, o = _gather_setup(half=1.0)                            # b^2 = 8e-4 << h^2
    h, a, n = 0.7, 0.4, 160
    g1 = (np.arange(n) + 0.5) / n * 2 * a - a
    X, Z = np.meshgrid(g1, g1)
    pts = np.stack([X.ravel(), np.zeros(X.size), Z.ravel()], 1).astype(np.float32)
    r = o.gather(_gb(pts, rho=1.0), _vpl([0, h, 0], flux=(1.0, 1.0, 1.0)))
    power = (r["rgb64"][:, 0] * math.pi).sum() * (2 * a / n) ** 2
    assert abs(power - math.pi * 4 * F_c(a / h, a / h)) < 2e-4


def test_gather_occluder_blocks():
    V = np.concatenate([floor_quad(5.0), scenegen.quad_tris([-1, 1.0, -1], [2, 0, 0], [0, 0, 2])])
    s = tiny_scene(V)
    o = oracle.OracleScene(s)
    g = _gb(np.array([[0.0, 0, 0], [3.0, 0, 0]], np.float32))
    r = o.gather(g, _vpl([0.0, 2.0, 0.0], nrm=(0, -1, 0)), bits=True)
    assert r["rgb64"][0].max() == 0 and r["rgb64"][1].min() > 0
    assert r["traced_bits"][:, 0].tolist() == [1, 1] and r["vis_bits"][:, 0].tolist() == [0, 1]


# ---------------------------------------------------------------- O14 direct term (reading R21)
def test_direct_irradiance_matches_rectangle_form_factor():
    """Floor point under the centre of the 0.5 x 0.5 light at H = 1.999: the
    direct radiance * pi / rho averaged over independent pixels (each with S
    light samples) equals pi * L * 4 * F_c(0.25/H, 0.25/H) = 0.61286."""
    s = tiny_scene(floor_quad(2.0))
    o = oracle.OracleScene(s)
    n = 4000
    px = np.arange(n, dtype=np.int32)
    g = _gb(np.zeros((n, 3), np.float32), rho=0.5)
    out = o.direct(g, px, 16, seed=9)
    E = out[:, 0].astype(np.float64) * math.pi / 0.5
    closed = math.pi * 10.0 * 4 * F_c(0.25 / 1.999, 0.25 / 1.999)
    m, se = E.mean(), E.std() / math.sqrt(n)
    assert abs(m - closed) < 4 * se + 1e-5, (m, closed, se)
    assert np.array_equal(out[:, 0], out[:, 1]) and np.array_equal(out[:, 0], out[:, 2])   # grey light, grey rho


def test_direct_tiny_light_hand_value_and_zero_cases():
    """SPEC shade_direct example for an area light: a light of area A
    and radiance pi/A at distance 1 straight above, rho = 1 -> 1 (up to the
    light's size); occluded, behind, back-face and grazing cases give 0."""
    size = 1e-3
    L = math.pi / (size * size)
    light = scenegen.make_light([0.0, 1.0, 0.0], size=size, radiance=(L, L, L))
    s = tiny_scene(floor_quad(2.0), lights=light)
    o = oracle.OracleScene(s)
    g = _gb(np.zeros((4, 3), np.float32), rho=1.0)
    out = o.direct(g, np.arange(4, dtype=np.int32), 4, seed=3)
    assert np.allclose(out, 1.0, rtol=1e-5), out
    g2 = g.copy()
    g2["nrm"] = [0, -1, 0]                                    # receiver faces away from the light
    assert o.direct(g2, np.arange(4, dtype=np.int32), 4).max() == 0
    g3 = g.copy()
    g3["front"] = 0                                           # back face
    assert o.direct(g3, np.arange(4, dtype=np.int32), 4).max() == 0
    g4 = g.copy()
    g4["pos"] = [[0.0, 1.0, 3.0]] * 4                         # light exactly edge-on (cl = 0, cx = 0)
    g4["nrm"] = [0, 0, 1]
    assert o.direct(g4, np.arange(4, dtype=np.int32), 4).max() == 0
    blk = np.concatenate([floor_quad(2.0), scenegen.quad_tris([-1, 0.5, -1], [2, 0, 0], [0, 0, 2])])
    ob = oracle.OracleScene(tiny_scene(blk, lights=light))
    assert ob.direct(g, np.arange(4, dtype=np.int32), 4).max() == 0   # blocker between


def test_direct_linear_in_radiance_and_sample_mean():
    """Doubling the light radiance doubles the output bitwise (every term
    scales by 2); with S samples the output is the mean of the S single-
    sample estimates drawn from the same counter slots (draws 2(lS+s), +1)."""
    s1 = tiny_scene(floor_quad(2.0))
    l2 = scenegen.make_light([0.0, 1.999, 0.0], radiance=(20.0, 20.0, 20.0))
    s2 = tiny_scene(floor_quad(2.0), lights=l2)
    g = _gb(np.array([[0.3, 0, -0.2], [1.2, 0, 0.7]], np.float32), rho=0.5)
    px = np.array([5, 77], np.int32)
    a = oracle.OracleScene(s1).direct(g, px, 8, seed=2)
    b = oracle.OracleScene(s2).direct(g, px, 8, seed=2)
    assert np.array_equal(2 * a, b)
    # S = 2 from S = 1 estimates: sample 1 uses draws (2, 3), i.e. the S=1 estimate of a pixel whose
    # draws are shifted by one sample -- checked through the float64 re-evaluation of the same samples
    o = oracle.OracleScene(s1)
    one = o.direct(g, px, 2, seed=2).astype(np.float64)
    Lt = s1.lights.reshape(-1, 16)[0]
    ref = []
    for k, p in enumerate(px):
        x = g["pos"][k].astype(np.float64)
        E = 0.0
        for q in range(2):
            u = (oracle.draw(2, 4, int(p), 2 * q) >> 8) * 2.0 ** -24
            v = (oracle.draw(2, 4, int(p), 2 * q + 1) >> 8) * 2.0 ** -24
            y = Lt[0:3] + u * Lt[3:6] + v * Lt[6:9]
            d = y - x
            r2 = d @ d
            E += 10.0 * Lt[12] * d[1] * d[1] / (r2 * r2)
        ref.append(0.5 * E / 2 / math.pi)
    assert np.allclose(one[:, 0], ref, rtol=1e-5)


# ---------------------------------------------------------------- O15 rejection comparator (reading R23)
def test_rejection_probe_pixels_one_per_block():
    s = scenegen.make_scene(1)
    o = oracle.OracleScene(s)
    for W, H in ((64, 64), (37, 23), (1920, 1080)):
        s2 = scenegen.custom_scene(s.verts, s.albedo, s.lights, s.cam, W, H)
        px = oracle.OracleScene(s2).probe_pixels(seed=4)
        x, y = px % W, px // W
        bx, by = np.arange(64) % 8, np.arange(64) // 8
        assert np.all((x >= bx * W // 8) & (x < (bx + 1) * W // 8))
        assert np.all((y >= by * H // 8) & (y < (by + 1) * H // 8))
    assert not np.array_equal(o.probe_pixels(seed=1), o.probe_pixels(seed=2))


def test_rejection_score_hand_value_and_dominance():
    """One probe under three VPLs: a facing VPL at height h scores
    (1/h^2) lum(Phi) lum(rho) (cx = ci = h, r2 = h^2 > b^2); a VPL facing away
    and one behind the probe score 0.  The facing one has p = 1 and is always
    kept; with every candidate scanned its flux keeps its scale (pilot/scanned
    = 1, 1/p = 1)."""
    s, o = _gather_setup()
    h = 3.0
    g = _gb(np.zeros((1, 3), np.float32), rho=0.8)
    g["alb"] = [0.2, 0.4, 0.6]
    pv = np.concatenate([_vpl([0.0, -1.0, 0.0], nrm=(0, 1, 0)),           # behind the probe
                         _vpl([0.5, h, 0.0], nrm=(0, 1, 0)),               # faces away
                         _vpl([0.0, h, 0.0], flux=(1.0, 2.0, 6.0))])       # facing, straight above
    pv["walk"] = [0, 1, 2]
    expect = (1.0 / (h * h)) * 3.0 * (((0.2 + 0.4) + 0.6) / 3.0)
    for seed in range(20):
        out, info = o.rejection(pv, 3, seed=seed, gb=g)
        assert info["scores"][0] == 0 and info["scores"][1] == 0
        assert abs(info["scores"][2] - expect) < 1e-6 * expect
        assert info["n_scanned"] == 3 and out["walk"][-1] == 2
        assert out["flux"][-1].tolist() == [1.0, 2.0, 6.0]
        if len(out) > 1:                                                  # a p = 0.05 candidate got in
            assert np.allclose(out["flux"][0], pv["flux"][out["walk"][0]] * 20.0, rtol=1e-6)


def test_rejection_ties_keep_generation_order():
    """Identical candidates: every p is 1, so the first `budget` are kept in
    order, the scanned prefix is `budget` long and fluxes scale by pilot/budget."""
    s, o = _gather_setup()
    g = _gb(np.array([[0.0, 0, 0], [1.0, 0, 0.5]], np.float32))
    pv = np.concatenate([_vpl([0.2, 2.0, 0.1])] * 10)
    pv["walk"] = np.arange(10)
    out, info = o.rejection(pv, 4, seed=1, gb=g)
    assert info["accepted"] == 4 and info["n_scanned"] == 4 and out["walk"].tolist() == [0, 1, 2, 3]
    assert np.array_equal(out["flux"], pv["flux"][:4] * np.float32(2.5))


def test_rejection_is_unbiased_in_power():
    """With the whole pilot scanned, E[sum of kept flux] = sum of pilot flux
    (each candidate kept with probability p_i, weighted 1/p_i): the mean over
    400 acceptance seeds (fixed probes) agrees within 4 sigma; the accepted
    count averages sum_i p_i."""
    s1 = scenegen.make_scene(1)
    o1 = oracle.OracleScene(s1)
    pilot, _ = o1.generate_vpls(np.zeros(s1.n_tris, np.uint8), M=512, K_near=0)
    gb = o1.gbuffer(o1.probe_pixels(seed=1))
    tot = pilot["flux"][:, 0].astype(np.float64).sum()
    sums, counts = [], []
    for seed in range(400):
        out, info = o1.rejection(pilot, len(pilot), seed=seed, gb=gb)
        sums.append(out["flux"][:, 0].astype(np.float64).sum())
        counts.append(info["accepted"])
    sc = info["scores"].astype(np.float64)
    p = np.clip(sc / info["mean"], 0.05, 1.0)
    m, se = np.mean(sums), np.std(sums) / math.sqrt(len(sums))
    assert abs(m - tot) < 4 * se + 1e-6 * tot, (m, tot, se)
    assert abs(np.mean(counts) - p.sum()) < 4 * np.std(counts) / math.sqrt(len(counts)) + 1e-9
    assert info["n_scanned"] == len(pilot)


# ---------------------------------------------------------------- O16 Metropolis comparator (reading R24)
def _c1_pilot(M=1024):
    s1 = scenegen.make_scene(1)
    o1 = oracle.OracleScene(s1)
    pilot, _ = o1.generate_vpls(np.zeros(s1.n_tris, np.uint8), M=M, K_near=0)
    return o1, pilot


def test_metropolis_flat_target_accepts_everything():
    """a uniform target gives acceptance rate 1.0 (every ratio is 1)."""
    s, o = _gather_setup()
    g = _gb(np.array([[0.0, 0, 0], [1.0, 0, 0.5]], np.float32))
    pv = np.concatenate([_vpl([0.2, 2.0, 0.1])] * 50)
    out, info = o.metropolis(pv, chains=4, per_chain=10, burn=5, radius=3, seed=1, gb=g)
    assert info["accepted"] == 4 * (5 + 10) and len(out) == 40
    assert np.array_equal(out["flux"], np.repeat(pv["flux"][:1], 40, 0) * np.float32(50 / 40))


def test_metropolis_pool_is_morton_ordered_and_stationary_law_is_f():
    """The pool follows the O4 Morton order of the pilot positions; with a
    wide mutation the chains' visit frequencies over f-quantile bins match
    f (the stationary law) to 5%."""
    o1, pilot = _c1_pilot()
    out, info = o1.metropolis(pilot, chains=64, per_chain=3000, burn=300, radius=300, seed=5)
    pos = pilot["pos"][info["pool"]].astype(np.float32)
    lo, hi = pos.min(0), pos.max(0)
    scale = np.where(hi - lo > 0, np.float32(1024.0) / (hi - lo), 0).astype(np.float32)
    q = np.minimum(((pos - lo).astype(np.float32) * scale).astype(np.uint32), 1023)
    codes = [oracle.morton3(int(a), int(b), int(c)) for a, b, c in q]
    assert all(x <= y for x, y in zip(codes, codes[1:]))
    sc = info["scores"].astype(np.float64)
    f = np.maximum(sc, 0.05 * sc.mean())
    # visited pool index of every emitted record: match by walk/position
    key = {tuple(pilot["pos"][i].tolist()) + (int(pilot["walk"][i]),): i for i in range(len(pilot))}
    vis = np.array([key[tuple(r["pos"].tolist()) + (int(r["walk"]),)] for r in out])
    bins = np.digitize(f, np.quantile(f, [0.25, 0.5, 0.75]))
    for b in range(4):
        expect = f[bins == b].sum() / f.sum()
        got = np.isin(vis, np.flatnonzero(bins == b)).mean()
        assert abs(got - expect) < 0.05 * expect + 0.01, (b, got, expect)


def test_metropolis_is_unbiased_in_power():
    """E[sum of emitted flux] = sum of pilot flux under the stationary law
    (importance weight (pilot / N) * mean_f / f): mean over 60 seeds within 4 sigma."""
    o1, pilot = _c1_pilot(512)
    gb = o1.gbuffer(o1.probe_pixels(seed=1))
    tot = pilot["flux"][:, 0].astype(np.float64).sum()
    sums = []
    for seed in range(60):
        out, _ = o1.metropolis(pilot, chains=32, per_chain=64, burn=64, radius=128, seed=seed, gb=gb)
        sums.append(out["flux"][:, 0].astype(np.float64).sum())
    m, se = np.mean(sums), np.std(sums) / math.sqrt(len(sums))
    assert abs(m - tot) < 4 * se + 1e-3 * tot, (m, tot, se)


def test_any_hit_division_free_matches_float64_segment_triangle():
    """R25 pin: the division-free any-hit of O9 (u, v, t scaled by |det|,
    sign-normalised by det) against a float64 segment-triangle test written
    from geometry (plane crossing point + barycentric coordinates), on random
    segments through one triangle from BOTH sides (det > 0 and det < 0),
    skipping cases within a margin of an edge or of the eps-shrunk ends."""
    T = np.array([[[0.2, 0.1, 0.3], [1.7, 0.4, 0.2], [0.6, 1.5, 1.1]]], np.float32)
    s = scenegen.custom_scene(T, np.full((1, 3), 0.5), scenegen.make_light([0.5, 1.9, 0.5]),
                              scenegen.make_camera([0.5, 0.8, -2.0], [0.5, 0.5, 0.5], 60, 8, 8), 8, 8,
                              M=4, K_near=4, max_depth=1, rr=1, seed=1, T=5.0)
    o = oracle.OracleScene(s)
    eps = float(o.consts()[1])
    v0, v1, v2 = (T[0, i].astype(np.float64) for i in range(3))
    n = np.cross(v1 - v0, v2 - v0)
    rng = np.random.default_rng(25)
    checked = {True: 0, False: 0}
    sides = set()
    for _ in range(4000):
        a = rng.uniform(-0.5, 2.2, 3).astype(np.float32)
        b = rng.uniform(-0.5, 2.2, 3).astype(np.float32)
        A, B = a.astype(np.float64), b.astype(np.float64)
        d = B - A
        L = np.linalg.norm(d)
        if L < 4 * eps:
            continue
        den = n @ d
        if abs(den) < 1e-3 * np.linalg.norm(n) * L:
            continue                                   # nearly parallel: no margin
        t = (n @ (v0 - A)) / den                      # crossing at A + t d
        p = A + t * d
        # barycentrics of p
        m = np.array([v1 - v0, v2 - v0]).T
        uv, *_ = np.linalg.lstsq(m, p - v0, rcond=None)
        u, w = uv
        bary_margin = min(u, w, 1 - u - w)
        end_margin = min(t * L - eps, (1 - t) * L - eps)
        if abs(bary_margin) < 1e-4 or abs(end_margin) < 1e-4:
            continue
        hit = bary_margin > 0 and end_margin > 0
        assert o.occluded(a, b) == hit, (a, b, bary_margin, end_margin)
        checked[hit] += 1
        if hit:
            sides.add(bool(den > 0))
    assert checked[True] > 100 and checked[False] > 1000 and sides == {True, False}
