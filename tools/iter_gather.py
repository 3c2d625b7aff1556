"""Kernel-iteration driver for the gather (a8): for each config, run one
frame, time `reps` gather launches with CUDA events, run the counter build,
and cross-check the gather's warp traversal (vpl_visibility_dump) against
the per-thread binary-BVH traversal (vpl_occluded_batch) on sampled pixels x
all VPLs.  This is a fast GPU self-consistency check for kernel work; the
parity tests against the oracle are tests/test_gpu_*.py.

  python tools/iter_gather.py --configs 3 4 --reps 2 --pixels 64
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2203_11484_b200 as V  # noqa: E402
import scenegen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", type=int, nargs="+", default=[3, 4])
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--pixels", type=int, default=64)
ap.add_argument("--no-counters", action="store_true")
a = ap.parse_args()

for cfg in a.configs:
    s = scenegen.make_scene(cfg)
    r = V.Renderer(s)
    r.frame()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(a.reps):
        e0.record()
        V.gather_indirect(r.scene, r.bvh, r.gbuf, r.vpls, r.tiles, s.width, s.height, 16, 16, r.rgb)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    out = {"config": cfg, "gather_ms": ts}
    img = r.rgb.clone()
    if not a.no_counters:
        rgb2, ctr = V.gather_indirect(r.scene, r.bvh, r.gbuf, r.vpls, r.tiles, s.width, s.height, 16, 16,
                                      counters=True)
        torch.cuda.synchronize()
        c = V.counters_dict(ctr)
        out["counters"] = c
        out["counter_build_image_equal"] = bool(torch.equal(rgb2, img))
        wr = max(c.get("warp_rays", 1), 1)
        out["steps_per_packet"] = c.get("warp_steps", 0) / wr
        out["tri_per_traced"] = c["tri_tests"] / max(c["traced"], 1)
    # visibility self-check on sampled pixels
    g = V.decode_gbuf(r.gbuf)
    rng = np.random.default_rng(cfg)
    cand = np.flatnonzero((g["tri"] >= 0) & (g["front"] != 0))
    px = np.sort(rng.choice(cand, size=min(a.pixels, len(cand)), replace=False)).astype(np.int32)
    tb, vb = V.visibility_dump(r.scene, r.bvh, r.gbuf, r.vpls.view(-1, V.VPL_RECORD_BYTES), px)
    vp = V.decode_vpls(r.vpls)
    M = len(vp)
    tbits = np.unpackbits(tb.cpu().numpy().view(np.uint8), bitorder="little").reshape(len(px), -1)[:, :M]
    vbits = np.unpackbits(vb.cpu().numpy().view(np.uint8), bitorder="little").reshape(len(px), -1)[:, :M]
    pi, vi = np.nonzero(tbits)
    A = g["pos"][px[pi]].astype(np.float32)
    B = vp["pos"][vi].astype(np.float32)
    occ = V.occluded_batch(r.scene, r.bvh, A, B).cpu().numpy().astype(bool)
    dis = int(np.count_nonzero(vbits[pi, vi].astype(bool) == occ))
    out["vis_check"] = {"pixels": len(px), "traced": int(len(pi)), "disagree": dis}
    print(json.dumps(out), flush=True)
