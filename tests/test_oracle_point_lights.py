"""Pins for the oracle's point lights (reading R27: "the light sources
are all point lights"; Eq. 2's literal point form P:51-56 with R1/R3 —
L_e = the light's power Phi, omega and r relative to the light):
closed forms, symmetry and energy invariants, not the oracle's own formulas.
CPU only; both oracle builds (default and frozen O0)."""
from __future__ import annotations

import math

import numpy as np
import pytest

import oracle
import scenegen


@pytest.fixture(autouse=True, params=["default", "o0"])
def oracle_variant(request):
    oracle.set_default_variant(request.param)
    yield request.param
    oracle.set_default_variant("default")


def tiny_scene(verts, lights, albedo=None, cam=None, W=8, H=8, **kw):
    verts = np.asarray(verts, np.float64).reshape(-1, 3, 3)
    if albedo is None:
        albedo = np.full((verts.shape[0], 3), 0.5)
    if cam is None:
        cam = scenegen.make_camera([0.0, 1.0, -3.0], [0.0, 0.0, 0.0], 60.0, W, H)
    return scenegen.custom_scene(verts, albedo, lights, cam, W, H, **kw)


def floor_quad(half=2.0, y=0.0):
    return scenegen.quad_tris([-half, y, -half], [0, 0, 2 * half], [2 * half, 0, 0])   # normal +y


def _gb(points, rho=0.5):
    g = np.zeros(len(points), oracle.GBUF_DTYPE)
    g["pos"] = points
    g["nrm"] = [0, 1, 0]
    g["alb"] = rho
    g["tri"] = 0
    g["front"] = 1
    return g


def _near_flux(light_pos, power, h=1e-3, rho=0.5, K=4000):
    """Near VPLs on a tiny horizontal patch at the origin (normal +y) lit by one point light."""
    V = [[[-h, 0, -h], [-h, 0, h], [h, 0, -h]]]
    cam = scenegen.make_camera([0.0, 1.0, -1.0], [0, 0, 0], 60.0, 8, 8)
    light = scenegen.make_point_light(light_pos, (power, power, power))
    s = tiny_scene(V, light, albedo=[[rho, rho, rho]], cam=cam, T=5.0, M=K, K_near=K, seed=5)
    o = oracle.OracleScene(s)
    lab, nn = o.classify()
    assert nn == 1 and o.lit(lab)[0] == 1
    v, info = o.generate_vpls(lab)
    assert info["K"] == K
    D = float(o.tri_data()["area"][0]) / K
    return v["flux"][:, 0].astype(np.float64) / D           # flux per unit represented area


def test_eq2_point_form_hand_value():
    """SPEC S:240 restated (R5): Phi_light = 4 pi, r = 1, cos omega = 1, rho = 0.5 ->
    Phi_in / D = 1 and the VPL flux / D = rho / pi = 0.159155 (tiny patch, so r and cos
    are 1 to 1e-6)."""
    f = _near_flux([0.0, 1.0, 0.0], 4 * math.pi)
    assert np.allclose(f, 0.5 / math.pi, rtol=1e-5), (f.min(), f.max())
    assert abs(0.5 / math.pi - 0.159155) < 1e-6


def test_eq2_point_form_inverse_square_and_lambert():
    """Moving the light to r = 2 quarters the flux; moving it to 60 degrees off the normal
    at r = 1 halves it (cos 60 = 1/2); behind the patch (cos < 0) gives no lit patch."""
    base = _near_flux([0.0, 1.0, 0.0], 4 * math.pi).mean()
    far = _near_flux([0.0, 2.0, 0.0], 4 * math.pi).mean()
    assert abs(far / base - 0.25) < 1e-4
    tilt = _near_flux([math.sin(math.pi / 3), math.cos(math.pi / 3), 0.0], 4 * math.pi).mean()
    assert abs(tilt / base - 0.5) < 1e-3
    V = [[[-1e-3, 0, -1e-3], [-1e-3, 0, 1e-3], [1e-3, 0, -1e-3]]]
    cam = scenegen.make_camera([0.0, 1.0, -1.0], [0, 0, 0], 60.0, 8, 8)
    s = tiny_scene(V, scenegen.make_point_light([0.0, -1.0, 0.0]), cam=cam, T=5.0, M=16, K_near=16, seed=5)
    o = oracle.OracleScene(s)
    lab, _ = o.classify()
    assert o.lit(lab)[0] == 0                                  # the light is behind the patch


def test_point_light_walk_energy_and_sphere_symmetry():
    """Closed 2 m cube, point light at its centre, every patch FAR (plain IR, fixed walks):
    (i) every walk's first hit deposits, and the depth-1 incident powers sum to Phi exactly
    (up to fp32); (ii) uniform emission on the sphere: each of the 6 faces gets 1/6 of the
    first hits (binomial 4 sigma)."""
    V = scenegen.room_tris([0, 0, 0], [2, 2, 2], n=1)
    cam = scenegen.make_camera([1.0, 1.0, 0.1], [1, 1, 2], 60.0, 8, 8)
    phi = 7.0
    s = tiny_scene(V, scenegen.make_point_light([1.0, 1.0, 1.0], (phi, phi, phi)), albedo=np.full((len(V), 3), 0.5),
                   cam=cam, T=0.01, M=0, K_near=0, max_depth=1, rr=0, seed=33)
    o = oracle.OracleScene(s)
    nw = 60000
    v, info = o.generate_vpls(np.zeros(s.n_tris, np.uint8), n_walks_fixed=nw, rr=0, max_depth=1)
    assert info["n_walks"] == nw and len(v) == nw
    inc = v["flux"][:, 0].astype(np.float64) * math.pi / 0.5
    assert abs(inc.sum() - phi) < 1e-4 * phi
    frac = np.bincount(v["tri"] // 2, minlength=6) / nw
    se = math.sqrt((1 / 6) * (5 / 6) / nw)
    assert np.all(np.abs(frac - 1 / 6) < 4 * se), frac


def test_point_light_direct_term_closed_form():
    """O14 for a point light of power Phi at height h above a floor point at horizontal
    offset s: irradiance Phi h / (4 pi (h^2 + s^2)^(3/2)), pixel = rho/pi * E; no samples,
    so every S gives the same value; a blocker zeroes it."""
    phi, h = 5.0, 1.5
    light = scenegen.make_point_light([0.0, h, 0.0], (phi, 2 * phi, 3 * phi))
    s = tiny_scene(floor_quad(3.0), light)
    o = oracle.OracleScene(s)
    offs = np.array([0.0, 0.3, 0.9, 2.0])
    g = _gb(np.stack([offs, np.zeros(4), np.zeros(4)], 1).astype(np.float32), rho=0.5)
    px = np.arange(4, dtype=np.int32)
    a = o.direct(g, px, 1, seed=1)
    b = o.direct(g, px, 16, seed=7)
    assert np.array_equal(a, b)
    E = phi * h / (4 * math.pi * (h * h + offs * offs) ** 1.5)
    assert np.allclose(a[:, 0], 0.5 / math.pi * E, rtol=2e-6)
    assert np.allclose(a[:, 2], 3 * a[:, 0], rtol=1e-6)
    blk = np.concatenate([floor_quad(3.0), scenegen.quad_tris([-2, 0.7, -2], [4, 0, 0], [0, 0, 4])])
    assert oracle.OracleScene(tiny_scene(blk, light)).direct(g, px, 1).max() == 0


def test_point_variant_of_a_config_keeps_power():
    s = scenegen.make_scene(3, point_lights=True)
    a = scenegen.make_scene(3)
    La, Lp = a.lights.reshape(-1, 16), s.lights.reshape(-1, 16)
    assert np.all(Lp[:, 12] == 0) and np.all(Lp[:, 3:9] == 0)
    assert np.allclose(Lp[:, 13:16], math.pi * La[:, 12:13] * La[:, 13:16], rtol=1e-6)
    assert np.array_equal(s.verts, a.verts)
