"""Time the C4 gather on the near VPLs only and on the far VPLs only (tools/ analysis)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2203_11484_b200 as V, scenegen
s = scenegen.make_scene(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
r = V.Renderer(s); r.frame(); torch.cuda.synchronize()
K = r.info["K"]
vp = r.vpls.view(-1, V.VPL_RECORD_BYTES)
for name, sub in (("all", vp), ("near", vp[:K]), ("far", vp[K:])):
    sub = sub.contiguous()
    V.gather_indirect(r.scene, r.bvh, r.gbuf, sub, r.tiles, s.width, s.height, 16, 16)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _, ctr = V.gather_indirect(r.scene, r.bvh, r.gbuf, sub, r.tiles, s.width, s.height, 16, 16, counters=False)
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1)
    _, ctr = V.gather_indirect(r.scene, r.bvh, r.gbuf, sub, r.tiles, s.width, s.height, 16, 16, counters=True)
    c = V.counters_dict(ctr.cpu())
    print(name, sub.shape[0], f"{t:.1f} ms", "traced", c["traced"], "vis", c["visible"], "packets", c["warp_rays"],
          "steps", c["warp_steps"], "tri", c["tri_tests"], "cache", c["cache_hits"], flush=True)
