"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Bit-exact for labels, VPL sets, G-buffers, closest hits;
BJ:5 tolerances for the gather.  All tests need a B200 (-m gpu)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import paper_2203_11484_b200 as V
import scenegen
from gpu_helpers import (GpuScene, MRE_TOL, PIXEL_TOL, VIS_TOL, assert_vpls_bitwise, compare_images,
                         gbuf_to_oracle, sample_pixels, vis_disagreement)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def scenes():
    return {c: scenegen.make_scene(c) for c in (1, 2, 3)}


@pytest.fixture(scope="module")
def gpu(scenes):
    return {c: GpuScene(s) for c, s in scenes.items()}


@pytest.fixture(scope="module")
def orc(scenes):
    return {c: oracle.OracleScene(s) for c, s in scenes.items()}


def test_device_is_sm100():
    info = V.device_info()
    assert info["cc"] == (10, 0) and info["sm_count"] >= 100


def test_philox_matches_oracle():
    rng = np.random.default_rng(1)
    x = rng.integers(0, 2**32, (4096, 6), dtype=np.uint64).astype(np.uint32)
    g = V.philox_batch(x)
    for i in range(0, 4096, 97):
        assert g[i].tolist() == oracle.philox(x[i, :4], x[i, 4:]).tolist()


@pytest.mark.parametrize("c", [1, 2, 3])
def test_scene_prep_bitwise(c, gpu, orc):
    g = V.scene_tri_data(gpu[c].scene, gpu[c].n)
    o = orc[c].tri_data()
    for k in ("normal", "centroid", "area"):
        assert np.array_equal(g[k].view(np.uint32), o[k].view(np.uint32)), k
    assert np.array_equal(g["aq"], o["aq"])
    assert V.scene_consts(gpu[c].scene) == orc[c].consts()
    assert int(gpu[c].bad.item()) == -1


def test_degenerate_triangle_reported():
    V_ = np.array([[[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0, 0, 0], [1, 1, 1], [2, 2, 2]],
                   [[0, 0, 0], [0, 0, 1], [1, 0, 0]], [[0, 0, 0], [0, 0, 0], [1, 0, 0]]], np.float32)
    s = scenegen.custom_scene(V_, np.full((4, 3), 0.5), scenegen.make_light([0, 2, 0]),
                              scenegen.make_camera([0, 1, -3], [0, 0, 0], 60, 8, 8), 8, 8)
    g = GpuScene(s)
    assert int(g.bad.item()) == 1 == oracle.OracleScene(s).bad


def _random_rays(s, n, seed):
    rng = np.random.default_rng(seed)
    lo, hi = s.verts.reshape(-1, 3).min(0), s.verts.reshape(-1, 3).max(0)
    o = rng.uniform(lo, hi, (n, 3)).astype(np.float32)
    d = rng.normal(size=(n, 3)).astype(np.float32)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return o, d.astype(np.float32)


@pytest.mark.parametrize("c", [1, 2, 3])
def test_closest_hit_bitwise(c, scenes, gpu, orc):
    s = scenes[c]
    o, d = _random_rays(s, 4000 if c < 3 else 1500, seed=c)
    tri, t = V.closest_hit_batch(gpu[c].scene, gpu[c].bvh, o, d, 1e-4, float("inf"))
    oi, ot = orc[c].closest_batch(o, d, 1e-4, np.inf)
    tri, t = tri.cpu().numpy(), t.cpu().numpy()
    bad = np.nonzero(tri != oi)[0]
    assert bad.size == 0, (bad[:10], tri[bad[:5]], oi[bad[:5]])
    hit = oi >= 0
    assert np.array_equal(t[hit].view(np.uint32), ot[hit].view(np.uint32))


@pytest.mark.parametrize("c", [1, 2, 3])
def test_segment_occlusion_matches(c, scenes, gpu, orc):
    s = scenes[c]
    rng = np.random.default_rng(10 + c)
    lo, hi = s.verts.reshape(-1, 3).min(0), s.verts.reshape(-1, 3).max(0)
    n = 4000 if c < 3 else 1500
    a = rng.uniform(lo, hi, (n, 3)).astype(np.float32)
    b = rng.uniform(lo, hi, (n, 3)).astype(np.float32)
    g = V.occluded_batch(gpu[c].scene, gpu[c].bvh, a, b).cpu().numpy().astype(bool)
    o = orc[c].occluded_batch(a, b)
    assert np.array_equal(g, o), np.nonzero(g != o)[0][:10]


@pytest.mark.parametrize("c", [1, 2, 3])
def test_classify_bitwise(c, gpu, orc):
    g, gn = gpu[c].labels()
    o, on = orc[c].classify()
    assert np.array_equal(g, o) and gn == on


@pytest.mark.parametrize("c", [1, 2, 3])
def test_generate_vpls_bitwise(c, scenes, gpu, orc):
    v, info = gpu[c].generate()
    lab, _ = orc[c].classify()
    ov, oinfo = orc[c].generate_vpls(lab)
    assert info == oinfo
    gv = V.decode_vpls(v)
    assert_vpls_bitwise(gv, ov)
    n = scenes[c].n_tris
    assert np.array_equal(np.bincount(gv["tri"], minlength=n), np.bincount(ov["tri"], minlength=n))


def test_generate_plain_ir_fixed_walks(scenes, gpu, orc):
    s = scenes[2]
    lab = np.zeros(s.n_tris, np.uint8)
    v, info = gpu[2].generate(labels=lab, n_walks_fixed=3000)
    ov, oinfo = orc[2].generate_vpls(lab, n_walks_fixed=3000)
    assert info == oinfo
    assert_vpls_bitwise(V.decode_vpls(v), ov)


def test_generate_degenerate_budgets(scenes, gpu, orc):
    s = scenes[1]
    for kw in [dict(K_near=0), dict(K_near=s.M), dict(M=0, K_near=0), dict(M=1, K_near=1), dict(max_depth=1)]:
        lab, _ = orc[1].classify()
        v, info = gpu[1].generate(**kw)
        ov, oinfo = orc[1].generate_vpls(lab, **kw)
        assert info == oinfo, kw
        assert_vpls_bitwise(V.decode_vpls(v), ov)


@pytest.mark.parametrize("c", [1, 3])
def test_gbuffer_bitwise(c, scenes, gpu, orc):
    s = scenes[c]
    gb, _ = gpu[c].gbuffer()
    g = V.decode_gbuf(gb)
    px = np.arange(s.width * s.height, dtype=np.int32) if c == 1 else sample_pixels(s.width, s.height, 4096)
    o = orc[c].gbuffer(px)
    gg = gbuf_to_oracle(g[px])
    assert np.array_equal(gg["tri"], o["tri"])
    hit = o["tri"] >= 0
    assert np.array_equal(gg["front"][hit], o["front"][hit])
    for k in ("pos", "nrm", "alb"):
        assert np.array_equal(gg[k][hit].view(np.uint32), o[k][hit].view(np.uint32)), k
    assert np.array_equal(gg["t"][hit].view(np.uint32), o["t"][hit].view(np.uint32))


def _gather_case(gs: GpuScene, os_: oracle.OracleScene, px, vpls_t, tw=16, th=16):
    s = gs.s
    gb, tiles = gs.gbuffer(tw, th)
    rgb, ctr = V.gather_indirect(gs.scene, gs.bvh, gb, vpls_t, tiles, s.width, s.height, tw, th, counters=True)
    rgb = rgb.view(-1, 3).cpu().numpy()
    gpx = gbuf_to_oracle(V.decode_gbuf(gb)[px])
    ov = V.decode_vpls(vpls_t)
    from gpu_helpers import vpls_to_oracle
    o = os_.gather(gpx, vpls_to_oracle(ov), bits=True)
    tb, vb = V.visibility_dump(gs.scene, gs.bvh, gb, vpls_t, px)
    tmis, vmis, ntr, agree = vis_disagreement(tb.cpu().numpy(), vb.cpu().numpy(), o["traced_bits"], o["vis_bits"])
    mre, prel = compare_images(rgb[px], o["rgb64"], agree)
    return dict(mre=mre, prel=prel, tmis=tmis, vmis=vmis, ntr=ntr, agree=agree.mean(), ctr=ctr.cpu().numpy(),
                rgb=rgb, o=o)


def test_gather_c1_all_pixels(scenes, gpu, orc):
    s = scenes[1]
    v, info = gpu[1].generate()
    px = np.arange(s.width * s.height, dtype=np.int32)
    r = _gather_case(gpu[1], orc[1], px, v)
    assert r["tmis"] == 0
    assert r["vmis"] <= VIS_TOL * r["ntr"]
    assert r["mre"] <= MRE_TOL and r["prel"] <= PIXEL_TOL, r
    assert r["ctr"][1] == r["ntr"]                      # traced pairs: GPU counter == oracle count
    assert r["rgb"].max() > 0


def test_gather_c2_sampled(scenes, gpu, orc):
    s = scenes[2]
    v, info = gpu[2].generate()
    px = sample_pixels(s.width, s.height, 1024)
    r = _gather_case(gpu[2], orc[2], px, v)
    assert r["tmis"] == 0
    assert r["vmis"] <= max(1, VIS_TOL * r["ntr"])
    assert r["mre"] <= MRE_TOL and r["prel"] <= PIXEL_TOL, {k: r[k] for k in ("mre", "prel", "vmis", "ntr")}


def test_gather_ragged_tiles_and_tile_subsets():
    """W, H not multiples of the tile size; the union of disjoint tile subsets
    equals the full-frame image bitwise (the multi-GPU sharding invariant)."""
    base = scenegen.make_scene(1)
    s = scenegen.custom_scene(base.verts, base.albedo, base.lights,
                              scenegen.make_camera([0.35, 1.2, 0.25], [2.0, 0.0, 2.0], 60.0, 37, 23), 37, 23,
                              M=base.M, K_near=base.K_near, max_depth=3, rr=1, seed=1, T=1.75)
    gs, os_ = GpuScene(s), oracle.OracleScene(s)
    v, _ = gs.generate()
    px = np.arange(37 * 23, dtype=np.int32)
    r = _gather_case(gs, os_, px, v, tw=8, th=4)
    assert r["tmis"] == 0 and r["mre"] <= MRE_TOL and r["prel"] <= PIXEL_TOL
    gb, tiles = gs.gbuffer(8, 4)
    full, _ = V.gather_indirect(gs.scene, gs.bvh, gb, v, tiles, 37, 23, 8, 4)
    parts = torch.zeros_like(full)
    for r_ in range(3):
        sub = tiles[r_::3].contiguous()
        V.gather_indirect(gs.scene, gs.bvh, gb, v, sub, 37, 23, 8, 4, rgb=parts)
    assert torch.equal(full, parts)


def test_empty_vpl_list_is_black(gpu, scenes):
    s = scenes[1]
    gb, tiles = gpu[1].gbuffer()
    empty = torch.zeros((0, 48), dtype=torch.uint8, device="cuda")
    rgb, _ = V.gather_indirect(gpu[1].scene, gpu[1].bvh, gb, empty, tiles, s.width, s.height)
    assert float(rgb.abs().max()) == 0.0


def test_empty_tile_list_writes_nothing(gpu, scenes):
    """n_tiles = 0 (a rank with no tiles): every per-tile call is a no-op
    (include/vplgi.h), also when the empty tile tensor has a null data pointer."""
    s = scenes[1]
    gb, tiles = gpu[1].gbuffer()
    v, _ = gpu[1].generate()
    none = torch.zeros(0, dtype=torch.int32, device="cuda")
    rgb = torch.full((s.height * s.width * 3,), 7.0, device="cuda")
    V.gather_indirect(gpu[1].scene, gpu[1].bvh, gb, v, none, s.width, s.height, rgb=rgb)
    V.render_direct(gpu[1].scene, gpu[1].bvh, gb, none, s.width, s.height, rgb=rgb, accumulate=True)
    assert bool((rgb == 7.0).all())


def test_single_triangle_scene():
    V_ = np.array([[[-1, 0, -1], [-1, 0, 1], [1, 0, -1]]], np.float32)
    s = scenegen.custom_scene(V_, np.full((1, 3), 0.5), scenegen.make_light([0, 1.999, 0]),
                              scenegen.make_camera([0, 1.0, -1.5], [0, 0, 0], 60, 16, 8), 16, 8,
                              M=8, K_near=8, max_depth=2, rr=1, seed=3, T=5.0)
    gs, os_ = GpuScene(s), oracle.OracleScene(s)
    o, d = _random_rays(s, 200, 5)
    tri, t = V.closest_hit_batch(gs.scene, gs.bvh, o, d, 0.0, float("inf"))
    oi, ot = os_.closest_batch(o, d, 0.0, np.inf)
    assert np.array_equal(tri.cpu().numpy(), oi)
    lab, _ = os_.classify()
    v, info = gs.generate()
    ov, oinfo = os_.generate_vpls(lab)
    assert info == oinfo
    assert_vpls_bitwise(V.decode_vpls(v), ov)
    r = _gather_case(gs, os_, np.arange(128, dtype=np.int32), v)
    assert r["rgb"].max() == 0.0                         # every VPL is on the receiver's own triangle (R14)


def test_gather_chunked_items_are_tile_split_invariant(scenes, gpu):
    """C2 (M = 4096 -> 16 VPL chunks folded in-kernel): the union of disjoint
    tile subsets equals the full frame bitwise, and repeated launches agree
    bitwise (the fold order is fixed, the queue order is not)."""
    s = scenes[2]
    v, _ = gpu[2].generate()
    gb, tiles = gpu[2].gbuffer()
    full, _ = V.gather_indirect(gpu[2].scene, gpu[2].bvh, gb, v, tiles, s.width, s.height)
    again, _ = V.gather_indirect(gpu[2].scene, gpu[2].bvh, gb, v, tiles, s.width, s.height)
    assert torch.equal(full, again)
    parts = torch.zeros_like(full)
    for r in range(4):
        V.gather_indirect(gpu[2].scene, gpu[2].bvh, gb, v, tiles[r::4].contiguous(), s.width, s.height, rgb=parts)
    assert torch.equal(full, parts)
    assert float(full.abs().max()) > 0


@pytest.mark.parametrize("M", [257, 511, 1000])
def test_gather_chunk_boundaries_against_oracle(M, scenes, orc):
    """VPL counts just above a chunk multiple (2 chunks of 256 + 1, ...):
    every chunk partial is folded, the image matches the oracle (C1, all
    pixels) and the tile-split invariance holds."""
    s0 = scenes[1]
    s = scenegen.custom_scene(s0.verts, s0.albedo, s0.lights, s0.cam, s0.width, s0.height, M=M,
                              K_near=int(0.75 * M + 0.5), max_depth=3, rr=1, seed=7, T=1.75)
    gs = GpuScene(s)
    v, info = gs.generate()
    assert v.shape[0] == M
    px = np.arange(s.width * s.height, dtype=np.int32)
    r = _gather_case(gs, orc[1], px, v)
    assert r["tmis"] == 0 and r["vmis"] <= max(1, VIS_TOL * r["ntr"])
    assert r["mre"] <= MRE_TOL and r["prel"] <= PIXEL_TOL, {k: r[k] for k in ("mre", "prel")}
    gb, tiles = gs.gbuffer()
    full, _ = V.gather_indirect(gs.scene, gs.bvh, gb, v, tiles, s.width, s.height)
    parts = torch.zeros_like(full)
    for k in range(3):
        V.gather_indirect(gs.scene, gs.bvh, gb, v, tiles[k::3].contiguous(), s.width, s.height, rgb=parts)
    assert torch.equal(full, parts)
