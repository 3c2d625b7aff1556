"""The gather's plane-side cull (gather.cuh `plane_cull`) drops a candidate triangle
before its exact MT tests when no pending segment can cross the triangle's plane inside O9's
(eps, L - eps).  The CUDA path applies it inside the list filter; the GPU tests check in situ that
no visibility bit moves (whole-frame counters, tests/test_gpu_fullsize.py).  This CPU test pins the
*criterion itself* against the oracle's exact O9 segment test: the criterion is restated here in
numpy float32, operation by operation, and on thousands of adversarial configurations — receivers
lying in the triangle's own plane, the VPL lying in it, grazing segments, endpoints a few ulps
off the plane — a culled triangle must never occlude any of the segments the oracle tests.

One scene holds a grid of well-separated cells with one triangle each (plus tiny markers at the
corners of [-5, 5]^3 that fix the scene's eps and box padding at realistic values); every segment
stays inside its cell, so the oracle's brute-force occlusion of a segment can only come from the
cell's own triangle."""
import numpy as np
import pytest

import oracle
import scenegen

F = np.float32


def _fma(a, b, c):
    # single-rounding fused multiply-add of float32 operands (exact in float64 up to the final rounding)
    return F(np.float64(a) * np.float64(b) + np.float64(c))


def plane_of(v0, e1, e2):
    """k_emit_tris: unit normal and offset in float64, rounded once."""
    n = np.cross(e1.astype(np.float64), e2.astype(np.float64))
    ln = np.linalg.norm(n)
    n = n / ln
    return n.astype(F), F(np.dot(n, v0.astype(np.float64)))


def plane_cull(n, off, y, xs, eps, mu):
    """gather.cuh make_beam (D box of the pending segments, s_lo) + plane_cull, float32."""
    D = (xs - y).astype(F)                      # D = x - y per receiver (fp32 subtraction)
    Dn, Dm = D.min(axis=0), D.max(axis=0)
    l2 = (D[:, 0] * D[:, 0] + D[:, 1] * D[:, 1]).astype(F) + (D[:, 2] * D[:, 2]).astype(F)
    lmax = F(np.sqrt(l2.max()))
    s = F(F(0.5) * eps) / lmax                  # Beam::s_lo = (VPL_SCAP * eps) * rcp(lmax)
    dc = (F(0.5) * (Dn + Dm)).astype(F)
    de = (F(0.5) * (Dm - Dn) + F(2e-7) * np.maximum(np.abs(Dn), np.abs(Dm))).astype(F)
    a = _fma(n[0], y[0], _fma(n[1], y[1], _fma(n[2], y[2], -off)))
    c = _fma(n[0], dc[0], _fma(n[1], dc[1], F(n[2] * dc[2])))
    e = _fma(abs(n[0]), de[0], _fma(abs(n[1]), de[1], _fma(abs(n[2]), de[2], F(mu + mu))))
    a_lo, a_hi = F(a - mu), F(a + mu)
    b_lo, b_hi = F(F(a + c) - e), F(F(a + c) + e)
    pos = (max(a_lo, b_lo) > 0) and (_fma(s, a_lo, b_lo) >= 0) and (_fma(s, b_lo, a_lo) >= 0)
    neg = (min(a_hi, b_hi) < 0) and (_fma(s, a_hi, b_hi) <= 0) and (_fma(s, b_hi, a_hi) <= 0)
    return bool(pos or neg)


def _scene(rng, cells):
    tris, meta = [], []
    for c in cells:
        ctr = c + rng.uniform(-0.05, 0.05, 3)
        # varied shapes: regular, needle, tiny, axis-aligned
        kind = rng.integers(0, 4)
        if kind == 0:
            e1, e2 = rng.normal(size=3) * 0.15, rng.normal(size=3) * 0.15
        elif kind == 1:
            e1 = rng.normal(size=3) * 0.2
            e2 = e1 * rng.uniform(0.2, 0.9) + rng.normal(size=3) * 0.004
        elif kind == 2:
            e1, e2 = rng.normal(size=3) * 0.01, rng.normal(size=3) * 0.01
        else:
            ax = rng.permutation(3)
            e1, e2 = np.zeros(3), np.zeros(3)
            e1[ax[0]], e2[ax[1]] = rng.uniform(0.05, 0.25), rng.uniform(0.05, 0.25)
        v0 = ctr - (e1 + e2) / 3
        tris.append(np.stack([v0, v0 + e1, v0 + e2]))
        meta.append(ctr)
    # markers: tiny triangles at the corners of [-5, 5]^3 (never near a test segment)
    for sx in (-5.0, 5.0):
        for sy in (-5.0, 5.0):
            for sz in (-5.0, 5.0):
                p = np.array([sx, sy, sz])
                q = p - np.sign(p) * 1e-3
                tris.append(np.stack([p, [q[0], p[1], p[2]], [p[0], q[1], p[2]]]))
    verts = np.asarray(tris, np.float32)
    alb = np.full((len(verts), 3), 0.5, np.float32)
    light = scenegen.make_light([0, 4.9, 0], 0.1)
    cam = scenegen.make_camera([0, 0, 4.5], [0, 0, 0], 60.0, 8, 8)
    return scenegen.custom_scene(verts, alb, light, cam, 8, 8, name="plane-cull cells", M=0, K_near=0)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_culled_triangle_never_occludes(seed):
    rng = np.random.default_rng(seed)
    g = np.arange(-3.5, 4.0, 1.0)
    cells = np.array([[x, y, z] for x in g for y in g for z in g])
    s = _scene(rng, cells)
    o = oracle.OracleScene(s)
    _, eps, _ = o.consts()
    eps = F(eps)
    mu = F(np.abs(s.verts).max()) * F(2.0 ** -16)       # SceneHdr::box_pad (scene.cu k_scene_consts)
    segs_a, segs_b, owner = [], [], []
    n_cull = n_case = 0
    kinds = np.zeros(6, int)
    for ci in range(len(cells)):
        v = s.verts[ci].astype(F)
        v0, e1, e2 = v[0], (v[1] - v[0]).astype(F), (v[2] - v[0]).astype(F)    # the triangle MT sees (k_emit_tris)
        n, off = plane_of(v0, e1, e2)
        n64 = n.astype(np.float64)
        inpl = lambda: (v0 + rng.uniform(-0.3, 1.3) * e1 + rng.uniform(-0.3, 1.3) * e2).astype(np.float64)
        for _ in range(6):
            kind = rng.integers(0, 6)
            nrec = rng.integers(1, 9)
            h = rng.choice([1e-7, 1e-6, 1e-5, 1e-4, 1e-3, 1e-2, 0.1]) * rng.choice([-1, 1])
            if kind == 0:      # receivers in the triangle's own plane (a few ulps off), VPL off it
                xs = np.array([inpl() + n64 * rng.normal() * 2e-7 for _ in range(nrec)])
                y = inpl() + n64 * rng.uniform(0.002, 0.3) * rng.choice([-1, 1]) + rng.normal(size=3) * 0.05
            elif kind == 1:    # the VPL in the plane, receivers off it (same side)
                y = inpl() + n64 * rng.normal() * 2e-7
                sd = rng.choice([-1, 1])
                xs = np.array([inpl() + n64 * sd * rng.uniform(0.002, 0.3) + rng.normal(size=3) * 0.03 for _ in range(nrec)])
            elif kind == 2:    # both ends close to the plane on either side: crossings near the ends
                y = inpl() + n64 * h
                xs = np.array([inpl() + n64 * rng.choice([-1, 1]) * abs(h) * rng.uniform(0.1, 10) for _ in range(nrec)])
            elif kind == 3:    # grazing: long in-plane offset, tiny normal offset
                y = inpl() + n64 * h
                t = e1.astype(np.float64) / np.linalg.norm(e1) * rng.uniform(0.2, 0.4)
                xs = np.array([y + t + n64 * rng.normal() * abs(h) + rng.normal(size=3) * 1e-3 for _ in range(nrec)])
            elif kind == 4:    # generic same-side / opposite-side
                y = inpl() + n64 * rng.uniform(-0.3, 0.3)
                xs = np.array([inpl() + n64 * rng.uniform(-0.3, 0.3) for _ in range(nrec)])
            else:              # receivers spread around one point of a curved patch near the plane
                base = inpl() + n64 * rng.uniform(-0.01, 0.01)
                xs = np.array([base + rng.normal(size=3) * 0.01 for _ in range(nrec)])
                y = inpl() + n64 * rng.uniform(0.01, 0.3) * rng.choice([-1, 1])
            ctr = cells[ci]
            y = np.clip(y, ctr - 0.45, ctr + 0.45).astype(F)
            xs = np.clip(xs, ctr - 0.45, ctr + 0.45).astype(F)
            n_case += 1
            if plane_cull(n, off, y, xs, eps, mu):
                n_cull += 1
                kinds[kind] += 1
                for x in xs:
                    segs_a.append(x); segs_b.append(y); owner.append(ci)
    assert n_cull > 0.2 * n_case, (n_cull, n_case)        # the criterion fires on these configurations
    assert (kinds > 0).all(), kinds                       # ... in every family, incl. own-plane and grazing ones
    occ = o.occluded_batch(np.asarray(segs_a, F), np.asarray(segs_b, F))
    bad = np.flatnonzero(occ)
    assert len(bad) == 0, f"{len(bad)} of {len(occ)} segments of culled triangles are occluded (O9), first: cell {owner[bad[0]]}"
