"""Run the hot path once on config C (untimed), then launch the gather
`--reps` times on a tile subset — a bounded command for ncu captures
(`ncu -k regex:k_gather ... python tools/profile_gather.py --config 3`)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2203_11484_b200 as V  # noqa: E402
import scenegen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--tile-frac", type=float, default=1.0, help="fraction of tiles (evenly strided)")
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--counters", action="store_true")
a = ap.parse_args()
s = scenegen.make_scene(a.config)
r = V.Renderer(s)
r.frame()
torch.cuda.synchronize()
step = max(1, int(round(1 / a.tile_frac)))
tiles = r.tiles[::step].contiguous()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(a.reps):
    e0.record()
    rgb, ctr = V.gather_indirect(r.scene, r.bvh, r.gbuf, r.vpls, tiles, s.width, s.height, 16, 16, r.rgb,
                                 counters=a.counters)
    e1.record()
    torch.cuda.synchronize()
    print(f"gather C{a.config} tiles {tiles.numel()}/{r.tiles.numel()}: {e0.elapsed_time(e1):.2f} ms"
          + (f" ctr {ctr.tolist()}" if ctr is not None else ""))
