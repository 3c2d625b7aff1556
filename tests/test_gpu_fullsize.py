"""GPU parity at BASELINE.json's full sizes (configs[2..4], BJ:9-11), in the
launch configuration bench.py times (whole frame, 16x16 tiles, persistent
gather), on outputs the brute-force oracle can compute: near/far labels and
(C3, C4) the whole VPL set bitwise; G-buffer bitwise on sampled pixels; the
indirect image and every pixel x VPL visibility bit on sampled pixels; C5
(3,972,160 triangles, 262,144 VPLs) checks sampled strata-free quantities:
labels, sampled walks, G-buffer samples and a VPL-subset gather."""
from __future__ import annotations

import os

import numpy as np
import pytest
import torch

import oracle
import paper_2203_11484_b200 as V
import scenegen
from gpu_helpers import (MRE_TOL, PIXEL_TOL, VIS_TOL, assert_vpls_bitwise, compare_images, gbuf_to_oracle,
                         sample_pixels, vis_disagreement, vpls_to_oracle)

pytestmark = pytest.mark.gpu


def _frame(s):
    r = V.Renderer(s)
    r.frame(counters=True)
    torch.cuda.synchronize()
    return r


def _check_gather(r, o, px):
    s = r.s
    gpx = gbuf_to_oracle(V.decode_gbuf(r.gbuf)[px])
    ov = vpls_to_oracle(V.decode_vpls(r.vpls))
    res = o.gather(gpx, ov, bits=True)
    tb, vb = V.visibility_dump(r.scene, r.bvh, r.gbuf, r.vpls, px)
    tmis, vmis, ntr, agree = vis_disagreement(tb.cpu().numpy(), vb.cpu().numpy(), res["traced_bits"],
                                              res["vis_bits"])
    img = r.rgb.view(-1, 3).cpu().numpy()[px]
    mre, prel = compare_images(img, res["rgb64"], agree)
    return dict(tmis=tmis, vmis=vmis, ntr=ntr, mre=mre, prel=prel, agree=float(agree.mean()))


@pytest.mark.parametrize("cfg,n_px", [(3, 256), (4, 36)])
def test_full_frame_parity(cfg, n_px):
    s = scenegen.make_scene(cfg)
    r = _frame(s)
    o = oracle.OracleScene(s)
    lab, nn = o.classify()
    assert np.array_equal(r.labels.cpu().numpy(), lab) and int(r.n_near.item()) == nn
    ov, oinfo = o.generate_vpls(lab)
    assert r.info == oinfo
    assert_vpls_bitwise(V.decode_vpls(r.vpls), ov)
    # G-buffer on 4096 stratified pixels
    px = sample_pixels(s.width, s.height, 4096, seed=cfg)
    g = gbuf_to_oracle(V.decode_gbuf(r.gbuf)[px])
    og = o.gbuffer(px)
    assert np.array_equal(g["tri"], og["tri"])
    hit = og["tri"] >= 0
    for k in ("pos", "nrm", "alb", "t"):
        assert np.array_equal(g[k][hit].view(np.uint32), og[k][hit].view(np.uint32)), k
    # gather + visibility bits on sampled pixels (BJ:5 tolerances)
    n_px *= int(os.environ.get("VPLGI_PARITY_SCALE", "1"))    # extended runs (profiles/r01_extended_parity.txt)
    c = _check_gather(r, o, sample_pixels(s.width, s.height, n_px, seed=100 + cfg))
    print(f"C{cfg} {n_px} px: {c}")
    assert c["tmis"] == 0, c
    assert c["vmis"] <= VIS_TOL * max(c["ntr"], 1) + 1, c
    assert c["mre"] <= MRE_TOL and c["prel"] <= PIXEL_TOL, c


def test_c5_sampled_parity():
    s = scenegen.make_scene(5, near_frac=0.5)
    r = V.Renderer(s)
    r.upload()
    r.bvh, r._bwork = V.build_bvh(r.scene, r.n)
    r.labels, r.n_near = V.classify_near_far(r.scene, r.n, s.T)
    r.vpls, r.info, _ = V.generate_vpls(r.scene, r.bvh, r.labels, r.n, s.M, s.K_near, s.max_depth, s.rr, s.seed,
                                        max_out=s.M)
    torch.cuda.synchronize()
    o = oracle.OracleScene(s)
    lab, nn = o.classify()
    assert np.array_equal(r.labels.cpu().numpy(), lab)
    info = r.info
    assert info["K"] + info["M_far"] == s.M and info["flags"] == 0
    gv = V.decode_vpls(r.vpls)
    # sampled walks: the oracle's raw deposits of walks [w0, w0 + 64) divided by the walk count
    far = gv[info["K"]:]
    n_w = info["n_walks"]
    for w0 in (0, n_w // 2, max(n_w - 64, 0)):
        w1 = min(w0 + 64, n_w)
        dep = o.walk_range(lab, w0, w1)
        sel = (far["walk"] >= w0) & (far["walk"] < w1)
        mine = far[sel]
        dep = dep[:len(mine)]                                  # the last walk may be cut (R11)
        assert len(mine) == len(dep)
        assert np.array_equal(mine["tri"], dep["tri"])
        assert np.array_equal(mine["pos"].view(np.uint32), dep["pos"].view(np.uint32))
        fl = (dep["flux"] / np.float32(n_w)).astype(np.float32)
        assert np.array_equal(mine["flux"].view(np.uint32), fl.view(np.uint32))
    # sampled strata of the near part
    for k0 in (0, info["K"] // 2, info["K"] - 32):
        ns = o.near_strata(lab, info["K"], k0, k0 + 32)
        go = vpls_to_oracle(gv[k0:k0 + 32])
        for k in ("pos", "nrm", "flux"):
            assert np.array_equal(go[k].view(np.uint32), ns[k].view(np.uint32)), k
    # G-buffer and a VPL-subset gather on the tiles holding 8 sampled pixels
    px = sample_pixels(s.width, s.height, 9, seed=55)[:8]
    tx = (s.width + 15) // 16
    tiles = torch.tensor(sorted({int((p // s.width) // 16 * tx + (p % s.width) // 16) for p in px}),
                         dtype=torch.int32, device="cuda")
    gb = V.render_gbuffer(r.scene, r.bvh, tiles, s.width, s.height)
    og = o.gbuffer(px)
    g = gbuf_to_oracle(V.decode_gbuf(gb)[px])
    assert np.array_equal(g["tri"], og["tri"])
    idx = np.sort(np.random.default_rng(5).choice(len(gv), 4096, replace=False))
    sub = r.vpls[torch.from_numpy(idx).cuda()].contiguous()
    rgb, _ = V.gather_indirect(r.scene, r.bvh, gb, sub, tiles, s.width, s.height)
    res = o.gather(g, vpls_to_oracle(V.decode_vpls(sub)), bits=True)
    tb, vb = V.visibility_dump(r.scene, r.bvh, gb, sub, px)
    tmis, vmis, ntr, agree = vis_disagreement(tb.cpu().numpy(), vb.cpu().numpy(), res["traced_bits"],
                                              res["vis_bits"])
    assert tmis == 0 and vmis <= VIS_TOL * max(ntr, 1) + 1
    mre, prel = compare_images(rgb.view(-1, 3).cpu().numpy()[px], res["rgb64"], agree)
    assert mre <= MRE_TOL and prel <= PIXEL_TOL
