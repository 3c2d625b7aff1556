"""C5 (BASELINE.json configs[4]: 3840x2160, ~4M tris, 262,144 VPLs) on one
GPU, near fraction swept over 50/80/95% (BJ:11): one frame of a1-a8, the
gather timed with CUDA events, counters from the counter build.  BJ runs C5
across 8 GPUs; this pod has one, so these are the per-GPU numbers."""
import os
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2203_11484_b200 as V  # noqa: E402
import scenegen  # noqa: E402

for f in [float(x) for x in os.environ.get("VPLGI_C5_FRACS", "0.5,0.8,0.95").split(",")]:
    s = scenegen.make_scene(5, near_frac=f)
    r = V.Renderer(s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    r.frame()
    torch.cuda.synchronize()
    e0.record()
    V.gather_indirect(r.scene, r.bvh, r.gbuf, r.vpls, r.tiles, s.width, s.height, 16, 16, r.rgb)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1)
    _, ctr = V.gather_indirect(r.scene, r.bvh, r.gbuf, r.vpls, r.tiles, s.width, s.height, 16, 16, counters=True)
    c = V.counters_dict(ctr.cpu())
    print(json.dumps({"config": s.name, "n_tris": s.n_tris, "M": int(r.vpls.shape[0]), "K": r.info["K"],
                      "gather_ms": t, "pairs_per_s": c["pairs"] / (t * 1e-3),
                      "traced_per_s": c["traced"] / (t * 1e-3), "counters": c}), flush=True)
    del r
    torch.cuda.empty_cache()
