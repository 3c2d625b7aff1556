"""One pass over every entry point of libvplgi.so, meant for the bounds-
checked build (SURVEY §6 "race detection / sanitizers"; compute-sanitizer is
not available on the GPU pool, so the library's own VPL_DEBUG device checks
stand in for memcheck):

  python tools/variants.py debug VPL_DEBUG=1
  VPLGI_LIB=paper_2203_11484_b200/libvplgi_debug.so python tools/exercise_all.py --config 4

Runs a1-a8 (upload, BVH, classification, VPL generation, G-buffer, gather
with counters, ragged 8x4 tiles), the direct term, the visibility dump, the
batch ray queries, the image error and the two comparators."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2203_11484_b200 as V  # noqa: E402
import scenegen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--vpls", type=int, default=0, help="cap M (0 = the config's)")
a = ap.parse_args()

s = scenegen.make_scene(a.config)
M = a.vpls or s.M
K = min(s.K_near, M)
r = V.Renderer(s)
rgb = r.frame(counters=True)
scene, bvh, n = r.scene, r.bvh, r.n
lab, _ = V.classify_near_far(scene, n, s.T)
v, info, _ = V.generate_vpls(scene, bvh, lab, n, M, K, s.max_depth, s.rr, s.seed)
# ragged 8x4 tiles, two chunk layouts
tiles = V.all_tiles(s.width, s.height, 8, 4)
gb = V.render_gbuffer(scene, bvh, tiles, s.width, s.height, 8, 4)
img, ctr = V.gather_indirect(scene, bvh, gb, v, tiles, s.width, s.height, 8, 4, counters=True)
img2, _ = V.gather_indirect(scene, bvh, gb, v[: max(1, v.shape[0] // 3)], tiles, s.width, s.height, 8, 4)
V.gather_indirect(scene, bvh, gb, v, tiles[:0], s.width, s.height, 8, 4)
V.render_direct(scene, bvh, gb, tiles, s.width, s.height, 8, 4, samples=4, rgb=img, accumulate=True)
px = torch.arange(0, s.width * s.height, 97, dtype=torch.int32, device="cuda")
V.visibility_dump(scene, bvh, gb, v, px)
rng = np.random.default_rng(0)
o = torch.from_numpy(rng.uniform(-1, 1, (256, 3)).astype(np.float32)).cuda()
d = torch.from_numpy(rng.normal(size=(256, 3)).astype(np.float32)).cuda()
V.closest_hit_batch(scene, bvh, o, d)
V.occluded_batch(scene, bvh, o, o + d)
V.image_error(img, img2)
pilot, _, _ = V.generate_vpls(scene, bvh, torch.zeros_like(lab), n, 4 * M, 0, s.max_depth, s.rr, s.seed + 1)
V.generate_rejection(scene, bvh, pilot, M, 7)
V.generate_metropolis(scene, bvh, pilot, 16, max(1, M // 16), burn=8, radius=4, seed=3)
torch.cuda.synchronize()
print("ok", s.name, "M", M, "launches", V.launch_count(), V.counters_dict(ctr))
