"""GPU parity of SURVEY §8(f) row f4's paper-literal point-light scenes
("the light sources are all point lights"; Eq. 2's point form P:51-56;
reading R27): C1-C3 geometry with every area light replaced by a point light
of the same power.  Bitwise: labels, the lit set through the whole VPL set
(near strata with Eq. 2's point form, sparse-IR walks emitted uniformly on
the sphere), the direct term; the indirect image and the production gather's
own visibility bits on sampled pixels within BJ:5's tolerances."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_2203_11484_b200 as V
import scenegen
from gpu_helpers import (MRE_TOL, PIXEL_TOL, VIS_TOL, GpuScene, assert_vpls_bitwise, compare_images,
                         gbuf_to_oracle, sample_pixels, vis_disagreement, vpls_to_oracle)

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg,n_px", [(1, None), (2, 256), (3, 64)])
def test_point_light_frame_parity(cfg, n_px):
    s = scenegen.make_scene(cfg, point_lights=True)
    assert np.all(s.lights.reshape(-1, 16)[:, 12] == 0)
    r = V.Renderer(s)
    r.frame()
    o = oracle.OracleScene(s)
    lab, nn = o.classify()
    assert np.array_equal(r.labels.cpu().numpy(), lab)
    ov, oinfo = o.generate_vpls(lab)
    assert r.info == oinfo and oinfo["K"] > 0 and oinfo["M_far"] > 0
    gv = V.decode_vpls(r.vpls)
    assert_vpls_bitwise(gv, ov)
    px = np.arange(s.width * s.height, dtype=np.int32) if n_px is None else sample_pixels(s.width, s.height, n_px)
    gpx = gbuf_to_oracle(V.decode_gbuf(r.gbuf)[px])
    og = o.gbuffer(px)
    assert np.array_equal(gpx["tri"], og["tri"])
    # direct term: no light samples for a point light, bitwise
    d = V.render_direct(r.scene, r.bvh, r.gbuf, r.tiles, s.width, s.height, samples=4, seed=3)
    dg = d.view(-1, 3).cpu().numpy()[px]
    do = o.direct(gpx, px, 4, seed=3)
    assert np.array_equal(dg.view(np.uint32), do.view(np.uint32))
    assert dg.max() > 0
    # indirect image with the production gather's own visibility bits
    rgb, _, tb, vb = V.gather_dump(r.scene, r.bvh, r.gbuf, r.vpls, r.tiles, s.width, s.height, px)
    res = o.gather(gpx, vpls_to_oracle(gv), bits=True)
    tmis, vmis, ntr, agree = vis_disagreement(tb, vb, res["traced_bits"], res["vis_bits"])
    mre, prel = compare_images(rgb.view(-1, 3).cpu().numpy()[px], res["rgb64"], agree)
    print(f"{s.name}: traced {ntr} tmis {tmis} vmis {vmis} mre {mre:.2e} prel {prel:.2e}")
    assert tmis == 0 and vmis <= VIS_TOL * max(ntr, 1) + 1
    assert mre <= MRE_TOL and prel <= PIXEL_TOL


def test_point_light_ir_walks_fixed_mode():
    """Plain IR (every patch FAR, fixed walk count) from point lights: the walk set bitwise."""
    s = scenegen.make_scene(2, point_lights=True)
    gs, o = GpuScene(s), oracle.OracleScene(s)
    far = np.zeros(s.n_tris, np.uint8)
    v, info = gs.generate(labels=far, K_near=0, n_walks_fixed=512)
    ov, oinfo = o.generate_vpls(far, K_near=0, n_walks_fixed=512)
    assert info == oinfo
    assert_vpls_bitwise(V.decode_vpls(v), ov)
