"""Does the order of the tile list matter for the gather?  (The image does not depend on it.)  Times the C3 / C4
gather with the default row-major list, a Morton-ordered list and 4x4-tile super-blocks in row-major order.

  python tools/tile_order.py --configs 3 4
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


def spread(v):
    v = v.astype(np.uint32)
    v = (v | (v << 8)) & 0x00FF00FF
    v = (v | (v << 4)) & 0x0F0F0F0F
    v = (v | (v << 2)) & 0x33333333
    v = (v | (v << 1)) & 0x55555555
    return v


ap = argparse.ArgumentParser()
ap.add_argument("--configs", type=int, nargs="+", default=[3, 4])
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
for cfg in a.configs:
    s = scenegen.make_scene(cfg)
    r = V.Renderer(s)
    r.frame()
    torch.cuda.synchronize()
    ref = r.rgb.clone()
    tx, ty = (s.width + 15) // 16, (s.height + 15) // 16
    t = np.arange(tx * ty, dtype=np.int32)
    x, y = t % tx, t // tx
    orders = {
        "row-major": t,
        "morton": t[np.argsort(spread(x) | (spread(y) << 1), kind="stable")],
        "super4x4": t[np.lexsort((x % 4, y % 4, x // 4, y // 4))],
        "super8x8": t[np.lexsort((x % 8, y % 8, x // 8, y // 8))],
        "column-major": t[np.lexsort((y, x))],
        "random": np.random.default_rng(7).permutation(t).astype(np.int32),
        "random-eighth": np.sort(np.random.default_rng(7).permutation(t)[: len(t) // 8]).astype(np.int32),
        "super4x4-eighth": t[((x // 4 + (y // 4) * ((tx + 3) // 4)) % 8) == 0],
    }
    out = {"config": cfg}
    for name, order in orders.items():
        tiles = torch.from_numpy(np.ascontiguousarray(order)).to(r.tiles.device)
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            V.gather_indirect(r.scene, r.bvh, r.gbuf, r.vpls, tiles, s.width, s.height, 16, 16, r.rgb)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        out[name] = {"ms": min(ts), "tiles": int(len(order)),
                     "bitwise_equal": bool(torch.equal(r.rgb, ref)) if len(order) == len(t) else None}
    print(json.dumps(out), flush=True)
