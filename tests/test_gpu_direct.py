"""GPU parity of NEXT row f2 — the direct term L_e of Eq. 1 (
DESIGN.md O14, reading R21) — against the CPU oracle: the same exact-fp32
Eq. 2-form sum with exact visibility, so the images must match bitwise."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import paper_2203_11484_b200 as V
import scenegen
from gpu_helpers import GpuScene, gbuf_to_oracle, sample_pixels

pytestmark = pytest.mark.gpu


def _direct_case(s, gs, os_, px, S, seed, tw=16, th=16):
    gb, tiles = gs.gbuffer(tw, th)
    rgb = V.render_direct(gs.scene, gs.bvh, gb, tiles, s.width, s.height, tw, th, samples=S, seed=seed)
    g = rgb.view(-1, 3).cpu().numpy()[px]
    o = os_.direct(gbuf_to_oracle(V.decode_gbuf(gb)[px]), px, S, seed=seed)
    return g, o, gb, tiles, rgb


@pytest.mark.parametrize("cfg,n_px,S", [(1, None, 8), (2, 1024, 4), (3, 64, 2)])
def test_direct_bitwise(cfg, n_px, S):
    s = scenegen.make_scene(cfg)
    gs, os_ = GpuScene(s), oracle.OracleScene(s)
    px = np.arange(s.width * s.height, dtype=np.int32) if n_px is None else sample_pixels(s.width, s.height, n_px)
    g, o, *_ = _direct_case(s, gs, os_, px, S, seed=s.seed)
    assert np.array_equal(g.view(np.uint32), o.view(np.uint32)), np.abs(g - o).max()
    assert g.max() > 0 and (g == 0).any()                   # lit and shadowed / back-facing pixels


def test_direct_c4_sampled_bitwise():
    s = scenegen.make_scene(4)
    gs, os_ = GpuScene(s), oracle.OracleScene(s)
    px = sample_pixels(s.width, s.height, 16)
    g, o, *_ = _direct_case(s, gs, os_, px, 2, seed=11)
    assert np.array_equal(g.view(np.uint32), o.view(np.uint32))


def test_direct_accumulates_onto_indirect_and_ragged_tiles():
    """accumulate=1 adds (fp32) onto the gather's indirect image; a ragged
    frame (37 x 23, 8 x 4 tiles) split into tile subsets equals the full frame."""
    base = scenegen.make_scene(1)
    s = scenegen.custom_scene(base.verts, base.albedo, base.lights,
                              scenegen.make_camera([0.35, 1.2, 0.25], [2.0, 0.0, 2.0], 60.0, 37, 23), 37, 23,
                              M=base.M, K_near=base.K_near, max_depth=3, rr=1, seed=1, T=1.75)
    gs, os_ = GpuScene(s), oracle.OracleScene(s)
    px = np.arange(37 * 23, dtype=np.int32)
    g, o, gb, tiles, direct = _direct_case(s, gs, os_, px, 4, seed=5, tw=8, th=4)
    assert np.array_equal(g.view(np.uint32), o.view(np.uint32))
    v, _ = gs.generate()
    ind, _ = V.gather_indirect(gs.scene, gs.bvh, gb, v, tiles, 37, 23, 8, 4)
    full = ind.clone()
    V.render_direct(gs.scene, gs.bvh, gb, tiles, 37, 23, 8, 4, samples=4, seed=5, rgb=full, accumulate=True)
    expect = ind.cpu().numpy() + direct.cpu().numpy()              # fp32 adds, same operands
    assert np.array_equal(full.cpu().numpy(), expect)
    parts = torch.zeros_like(direct)
    for r in range(3):
        V.render_direct(gs.scene, gs.bvh, gb, tiles[r::3].contiguous(), 37, 23, 8, 4, samples=4, seed=5,
                        rgb=parts)
    assert torch.equal(parts, direct)


def test_direct_rejects_bad_arguments():
    s = scenegen.make_scene(1)
    gs = GpuScene(s)
    gb, tiles = gs.gbuffer()
    with pytest.raises(V.VplError):
        V.render_direct(gs.scene, gs.bvh, gb, tiles, s.width, s.height, samples=0)
