"""Seeded synthetic scene generator — the ONLY code shared by the oracle side
and the CUDA side (both consume its arrays).  It holds none of the method's
arithmetic: it emits triangles, albedos, area lights, a pinhole camera and the
method knobs of BASELINE.json configs[0..4] (BJ:7-11), following the reading
R0 recorded in DESIGN.md §3.  Everything here is *input*: geometry placement,
colours, light rectangles, camera basis and the VPL budget split.

Conventions:
  * y is up; every triangle is one-sided with normal (v1-v0)x(v2-v0) (P:44
    "one-sided face"); rooms face inward, objects face outward.
  * lights: float32 [nL, 16] = corner(3) e_u(3) e_v(3) normal(3) area(1)
    radiance(3); a light is the parallelogram corner + a*e_u + b*e_v, a,b in
    [0,1], emitting (Lambertian) on the side of `normal`.  Lights are not
    occluders (they are not triangles).
  * camera: float32 [14] = pos(3) fwd(3) up(3) right(3) tan_x tan_y, plus the
    integer resolution (W, H).  tan_y = tan(vfov/2), tan_x = tan_y*W/H.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = ["Scene", "make_scene", "CONFIGS", "custom_scene", "quad_tris", "box_tris",
           "icosphere_tris", "room_tris", "make_light", "make_point_light", "point_lights_of", "make_camera"]


@dataclass
class Scene:
    name: str
    verts: np.ndarray          # float32 [N, 3, 3]
    albedo: np.ndarray         # float32 [N, 3]
    lights: np.ndarray         # float32 [nL, 16]
    cam: np.ndarray            # float32 [14]
    width: int
    height: int
    # method knobs (BJ:7-11; DESIGN.md §3 R0)
    M: int = 0                 # total VPL budget
    K_near: int = 0            # patch-stratified (near-field) VPLs requested
    max_depth: int = 3         # D_max of the sparse-IR walk
    rr: int = 1                # Russian roulette on (R10)
    seed: int = 1
    T: float = 1.0             # near/far distance threshold, metres
    meta: dict = field(default_factory=dict)

    @property
    def n_tris(self) -> int:
        return int(self.verts.shape[0])

    @property
    def n_lights(self) -> int:
        return int(self.lights.shape[0])

    @property
    def M_far(self) -> int:
        return self.M - self.K_near


# --------------------------------------------------------------------------
# geometry builders (float64 construction, rounded once to float32 at the end)
# --------------------------------------------------------------------------

def quad_tris(p, a, b, nu=1, nv=1):
    """Parallelogram p + s*a + t*b split into nu x nv quads, 2 tris each; the
    normal of every triangle is along a x b."""
    p, a, b = (np.asarray(x, np.float64) for x in (p, a, b))
    out = []
    for i in range(nu):
        for j in range(nv):
            q0 = p + a * (i / nu) + b * (j / nv)
            q1 = p + a * ((i + 1) / nu) + b * (j / nv)
            q2 = p + a * ((i + 1) / nu) + b * ((j + 1) / nv)
            q3 = p + a * (i / nu) + b * ((j + 1) / nv)
            out.append((q0, q1, q2))
            out.append((q0, q2, q3))
    return np.array(out, np.float64).reshape(-1, 3, 3)


def box_tris(center, half, yaw=0.0):
    """12 outward-facing triangles of a box with half extents `half`, rotated
    by `yaw` about +y around its centre."""
    c = np.asarray(center, np.float64)
    h = np.asarray(half, np.float64)
    cy, sy = math.cos(yaw), math.sin(yaw)
    ex = np.array([cy, 0.0, -sy]) * (2 * h[0])
    ey = np.array([0.0, 1.0, 0.0]) * (2 * h[1])
    ez = np.array([sy, 0.0, cy]) * (2 * h[2])
    m = c - 0.5 * (ex + ey + ez)
    faces = [
        (m, ez, ey), (m + ex, ey, ez),      # -x, +x
        (m, ex, ez), (m + ey, ez, ex),      # -y, +y
        (m, ey, ex), (m + ez, ex, ey),      # -z, +z
    ]
    return np.concatenate([quad_tris(p, a, b) for p, a, b in faces])


def _icosphere_unit(level):
    t = (1.0 + math.sqrt(5.0)) / 2.0
    v = [(-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0), (0, -1, t), (0, 1, t),
         (0, -1, -t), (0, 1, -t), (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1)]
    v = [np.array(x, np.float64) / np.linalg.norm(x) for x in v]
    f = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4),
         (11, 10, 2), (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8),
         (3, 8, 9), (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    for _ in range(level):
        cache = {}

        def mid(i, j):
            key = (min(i, j), max(i, j))
            if key not in cache:
                m = v[i] + v[j]
                v.append(m / np.linalg.norm(m))
                cache[key] = len(v) - 1
            return cache[key]
        nf = []
        for a, b, c in f:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            nf += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        f = nf
    V = np.array(v)
    return V[np.array(f)]          # [F, 3, 3], outward (CCW seen from outside)


_ICO2 = None


def icosphere_tris(center, radius):
    """Level-2 icosphere (320 faces, R18), outward-facing."""
    global _ICO2
    if _ICO2 is None:
        _ICO2 = _icosphere_unit(2)
    return _ICO2 * float(radius) + np.asarray(center, np.float64)


def room_tris(lo, hi, n=1, open_front=False, ny=None):
    """Inward-facing walls of the axis-aligned room [lo, hi]; each wall split
    into n x n quads (ny for the vertical direction if given)."""
    lo, hi = np.asarray(lo, np.float64), np.asarray(hi, np.float64)
    L = hi - lo
    X, Y, Z = (np.array([L[0], 0, 0]), np.array([0, L[1], 0]), np.array([0, 0, L[2]]))
    nv = n if ny is None else ny
    walls = [
        quad_tris(lo, Z, X, n, n),                                  # floor  (+y)
        quad_tris(np.array([lo[0], hi[1], lo[2]]), X, Z, n, n),     # ceiling (-y)
        quad_tris(lo, Y, Z, nv, n),                                 # x = lo (+x)
        quad_tris(np.array([hi[0], lo[1], lo[2]]), Z, Y, n, nv),    # x = hi (-x)
        quad_tris(np.array([lo[0], lo[1], hi[2]]), Y, X, nv, n),    # z = hi (-z)
    ]
    if not open_front:
        walls.append(quad_tris(lo, X, Y, n, nv))                    # z = lo (+z)
    return np.concatenate(walls)


def make_light(center, size=0.5, radiance=(10.0, 10.0, 10.0)):
    """0.5 x 0.5 m ceiling light facing -y (R0).  e_u = (s,0,0), e_v = (0,0,s)
    so normal = normalize(e_u x e_v) = (0,-1,0); area = s*s."""
    c = np.asarray(center, np.float64)
    corner = c - np.array([size / 2, 0.0, size / 2])
    return np.concatenate([corner, [size, 0, 0], [0, 0, size], [0, -1, 0],
                           [size * size], list(radiance)]).astype(np.float32)


def make_point_light(position, power=(10.0, 10.0, 10.0)):
    """Isotropic point light (reading R27, "the light sources are all
    point lights"): the light row with e_u = e_v = 0 and area = 0, `power`
    (W per channel) in the radiance field."""
    return np.concatenate([np.asarray(position, np.float64), [0, 0, 0], [0, 0, 0], [0, -1, 0], [0.0],
                           list(power)]).astype(np.float32)


def point_lights_of(lights, drop=0.2):
    """The paper-literal variant of a config (R27): every area light becomes a
    point light `drop` m below its centre with the area light's total power
    pi * A * L (so the two variants carry the same energy)."""
    out = []
    for L in np.asarray(lights, np.float64):
        c = L[0:3] + 0.5 * L[3:6] + 0.5 * L[6:9] + drop * L[9:12]
        out.append(make_point_light(c, np.pi * L[12] * L[13:16]))
    return np.stack(out)


def make_camera(pos, target, vfov_deg, W, H, up=(0.0, 1.0, 0.0)):
    p = np.asarray(pos, np.float64)
    f = np.asarray(target, np.float64) - p
    f /= np.linalg.norm(f)
    r = np.cross(f, np.asarray(up, np.float64))
    r /= np.linalg.norm(r)
    u = np.cross(r, f)
    ty = math.tan(math.radians(vfov_deg) / 2.0)
    tx = ty * W / H
    return np.concatenate([p, f, u, r, [tx, ty]]).astype(np.float32)


def _k_near(M, frac):
    return int(math.floor(frac * M + 0.5))


# --------------------------------------------------------------------------
# BASELINE.json configs (BJ:7-11) — reading R0
# --------------------------------------------------------------------------

def _config1(seed=1):
    rng = np.random.default_rng(seed)
    tris = [room_tris([0, 0, 0], [2, 2, 2], open_front=True)]        # 10 tris
    for _ in range(2):
        e = rng.uniform(0.3, 0.7, 3)
        cx, cz = rng.uniform(0.4, 1.6, 2)
        tris.append(box_tris([cx, e[1] / 2, cz], e / 2))               # resting on the floor
    V = np.concatenate(tris)
    alb = rng.uniform(0.2, 0.8, (V.shape[0], 3))                       # per patch (R17)
    lights = np.stack([make_light([1.0, 2.0 - 1e-3, 1.0])])
    cam = make_camera([0.35, 1.2, 0.25], [2.0, 0.0, 2.0], 60.0, 64, 64)
    M = 256
    return dict(name="C1", verts=V, albedo=alb, lights=lights, cam=cam, width=64, height=64,
                M=M, K_near=192, max_depth=3, rr=1, seed=seed, T=1.75)


def _config2(seed=2):
    rng = np.random.default_rng(seed)
    eye, tgt = np.array([0.25, 1.1, 0.2]), np.array([1.3, 0.75, 1.5])
    seg = 0.7 * (tgt - eye)
    tris = [room_tris([0, 0, 0], [2, 2, 2], open_front=True)]
    alb = [rng.uniform(0.2, 0.8, (10, 3))]
    placed = 0
    while placed < 200:
        e = rng.uniform(0.05, 0.4, 3)
        yaw = rng.uniform(0.0, 2 * math.pi)
        c = rng.uniform([0.2, 0.2, 0.2], [1.8, 1.4, 1.8])      # keep the ceiling light clear
        col = rng.uniform(0.1, 0.9, (1, 3))
        tt = np.clip((c - eye) @ seg / (seg @ seg), 0.0, 1.0)
        if np.linalg.norm(c - (eye + tt * seg)) <= 0.5 * np.linalg.norm(e) + 0.1:
            continue                                           # keep the camera's line of sight clear
        tris.append(box_tris(c, e / 2, yaw))
        alb.append(np.repeat(col, 12, axis=0))
        placed += 1
    V = np.concatenate(tris)
    lights = np.stack([make_light([1.0, 2.0 - 1e-3, 1.0])])
    cam = make_camera(eye, tgt, 45.0, 512, 512)
    M = 4096
    return dict(name="C2", verts=V, albedo=np.concatenate(alb), lights=lights, cam=cam,
                width=512, height=512, M=M, K_near=_k_near(M, 0.75), max_depth=3, rr=1,
                seed=seed, T=1.75)


def _scatter_objects(rng, n_box, n_sph, lo, hi, tris, alb, clear=None):
    """Random boxes and level-2 icospheres, log-uniform size in [0.02, 1] m,
    uniformly placed in [lo, hi], per-object albedo U[0.1, 0.9]^3.  `clear` =
    (p0, p1): objects whose bounding sphere comes within 0.1 m of the segment
    p0-p1 are rejected (a line-of-sight corridor from the camera toward its
    target, so the view is not filled by one object in front of the lens)."""
    lo, hi = np.asarray(lo, np.float64), np.asarray(hi, np.float64)
    n_tot = n_box + n_sph
    cand = int(n_tot * 1.25) + 64
    kinds = np.array([0] * int(cand * n_box / n_tot) + [1] * (cand - int(cand * n_box / n_tot)))
    rng.shuffle(kinds)
    sizes = np.exp(rng.uniform(math.log(0.02), math.log(1.0), kinds.size))
    cents = rng.uniform(lo, hi, (kinds.size, 3))
    cols = rng.uniform(0.1, 0.9, (kinds.size, 3))
    yaws = rng.uniform(0.0, 2 * math.pi, kinds.size)
    shp = rng.uniform(0.5, 1.0, (kinds.size, 3))
    keep = np.ones(kinds.size, bool)
    if clear is not None:
        p0, p1 = (np.asarray(x, np.float64) for x in clear)
        seg = p1 - p0
        tt = np.clip(((cents - p0) @ seg) / (seg @ seg), 0.0, 1.0)
        dist = np.linalg.norm(cents - (p0 + tt[:, None] * seg), axis=1)
        keep &= dist > (0.87 * sizes + 0.1)
    # first n_box boxes and n_sph spheres that survive, in candidate order
    sel = np.zeros(kinds.size, bool)
    for k, n in ((0, n_box), (1, n_sph)):
        idx = np.nonzero(keep & (kinds == k))[0]
        if idx.size < n:
            raise RuntimeError("scene generator: not enough candidates")
        sel[idx[:n]] = True
    order = np.nonzero(sel)[0]
    unit_box = box_tris([0, 0, 0], [0.5, 0.5, 0.5])                    # [12,3,3] unit cube
    global _ICO2
    if _ICO2 is None:
        _ICO2 = _icosphere_unit(2)
    b = order[kinds[order] == 0]
    sp = order[kinds[order] == 1]
    pieces = {}
    if b.size:
        s = sizes[b, None] * shp[b]                                   # edges per axis
        cy, sy = np.cos(yaws[b]), np.sin(yaws[b])
        R = np.zeros((b.size, 3, 3))
        R[:, 0, 0], R[:, 0, 2] = cy, sy
        R[:, 1, 1] = 1.0
        R[:, 2, 0], R[:, 2, 2] = -sy, cy
        local = unit_box[None] * s[:, None, None, :]
        world = np.einsum("oij,otvj->otvi", R, local) + cents[b, None, None, :]
        pieces.update({int(o): world[k] for k, o in enumerate(b)})
    if sp.size:
        world = _ICO2[None] * (sizes[sp, None, None, None] / 2) + cents[sp, None, None, :]
        pieces.update({int(o): world[k] for k, o in enumerate(sp)})
    for o in order:
        w = pieces[int(o)]
        tris.append(w)
        alb.append(np.repeat(cols[o:o + 1], w.shape[0], axis=0))


def _config3(seed=3):
    rng = np.random.default_rng(seed)
    tris = [room_tris([0, 0, 0], [8, 3, 8], n=16)]                    # 3,072 tris
    alb = [rng.uniform(0.1, 0.9, (3072, 3))]
    tgt = np.array([4.0, 0.6, 4.0])
    eye = tgt + np.array([-0.9, 0.9, -1.15])                          # ~1.7 m from the target
    _scatter_objects(rng, 1763, 237, [0.3, 0.0, 0.3], [7.7, 2.7, 7.7], tris, alb,
                     clear=(eye, eye + 0.7 * (tgt - eye)))
    V = np.concatenate(tris)
    lights = np.stack([make_light([2.75, 3.0 - 1e-3, 4.0]), make_light([5.25, 3.0 - 1e-3, 4.0])])
    cam = make_camera(eye, tgt, 60.0, 1920, 1080)
    M = 16384
    return dict(name="C3", verts=V, albedo=np.concatenate(alb), lights=lights, cam=cam,
                width=1920, height=1080, M=M, K_near=_k_near(M, 0.8), max_depth=3, rr=1,
                seed=seed, T=3.0)


def _config4(seed=4):
    rng = np.random.default_rng(seed)
    tris = [room_tris([0, 0, 0], [20, 5, 20], n=16)]                  # 6 x 512 tris
    alb = [rng.uniform(0.1, 0.9, (3072, 3))]
    tgt = np.array([6.0, 0.9, 6.0])
    eye = tgt + np.array([-0.9, 0.9, -1.15])
    _scatter_objects(rng, 27932, 2068, [0.3, 0.0, 0.3], [19.7, 1.8, 19.7], tris, alb,
                     clear=(eye, eye + 0.7 * (tgt - eye)))
    V = np.concatenate(tris)
    lights = np.stack([make_light([x, 5.0 - 1e-3, z]) for x in (5.0, 15.0) for z in (5.0, 15.0)])
    cam = make_camera(eye, tgt, 60.0, 1920, 1080)
    M = 65536
    return dict(name="C4", verts=V, albedo=np.concatenate(alb), lights=lights, cam=cam,
                width=1920, height=1080, M=M, K_near=_k_near(M, 0.8), max_depth=5, rr=1,
                seed=seed, T=3.0)


def _config5(seed=5, near_frac=0.5):
    rng = np.random.default_rng(seed)
    tris = [room_tris([0, 0, 0], [40, 3, 40], n=64, ny=8)]            # shell
    alb = [rng.uniform(0.1, 0.9, (tris[0].shape[0], 3))]
    # internal walls: 3 lines along x and 3 along z, 4 segments each, one 1 m
    # door (2.1 m tall) per segment -> 3 slabs per segment
    for axis in (0, 2):
        for k in (1, 2, 3):
            for seg in range(4):
                a0, a1 = seg * 10.0, seg * 10.0 + 10.0
                d0, d1 = a0 + 4.5, a0 + 5.5
                parts = [(a0, d0, 0.0, 3.0), (d1, a1, 0.0, 3.0), (d0, d1, 2.1, 3.0)]
                for (s0, s1, y0, y1) in parts:
                    c = [0.0, (y0 + y1) / 2, 0.0]
                    h = [0.0, (y1 - y0) / 2, 0.0]
                    c[axis] = (s0 + s1) / 2
                    h[axis] = (s1 - s0) / 2
                    other = 2 - axis
                    c[other] = 10.0 * k
                    h[other] = 0.05
                    t = box_tris(c, h)
                    tris.append(t)
                    alb.append(np.repeat(rng.uniform(0.1, 0.9, (1, 3)), 12, axis=0))
    tgt = np.array([15.0, 0.8, 15.0])
    eye = tgt + np.array([-0.9, 0.9, -1.15])
    _scatter_objects(rng, 111848, 8152, [0.3, 0.0, 0.3], [39.7, 1.6, 39.7], tris, alb,
                     clear=(eye, eye + 0.7 * (tgt - eye)))
    V = np.concatenate(tris)
    lights = []
    for i in range(4):
        for j in range(4):
            if (i + j) % 2 == 0:
                lights.append(make_light([10.0 * i + 5.0, 3.0 - 1e-3, 10.0 * j + 5.0]))
    lights = np.stack(lights)
    cam = make_camera(eye, tgt, 60.0, 3840, 2160)
    M = 262144
    return dict(name=f"C5@{int(round(near_frac * 100))}", verts=V, albedo=np.concatenate(alb),
                lights=lights, cam=cam, width=3840, height=2160, M=M,
                K_near=_k_near(M, near_frac), max_depth=5, rr=1, seed=seed, T=3.0)


CONFIGS = {1: _config1, 2: _config2, 3: _config3, 4: _config4, 5: _config5}


def _finish(d):
    V = np.ascontiguousarray(np.asarray(d.pop("verts"), np.float64).astype(np.float32))
    A = np.ascontiguousarray(np.asarray(d.pop("albedo"), np.float64).astype(np.float32))
    L = np.ascontiguousarray(np.asarray(d.pop("lights"), np.float32))
    C = np.ascontiguousarray(np.asarray(d.pop("cam"), np.float32))
    return Scene(verts=V, albedo=A, lights=L, cam=C, **d)


def make_scene(config: int, seed: int | None = None, point_lights: bool = False, **kw) -> Scene:
    """Build BASELINE.json configs[config-1] with its seed (BJ:7-11);
    point_lights=True gives the paper-literal variant lit by point lights
    (reading R27) of the same geometry and light power."""
    fn = CONFIGS[config]
    d = fn(**kw) if seed is None else fn(seed=seed, **kw)
    if point_lights:
        d["lights"] = point_lights_of(d["lights"])
        d["name"] = d["name"] + "-point"
    return _finish(d)


def custom_scene(verts, albedo, lights, cam, width, height, name="custom", **knobs) -> Scene:
    """Hand-built scenes for pins and edge cases."""
    d = dict(name=name, verts=verts, albedo=albedo, lights=np.atleast_2d(lights), cam=cam,
             width=width, height=height)
    d.update(knobs)
    return _finish(d)
