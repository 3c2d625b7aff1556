"""Per-stage times of one frame ("ms/frame ... plus per-stage
times for a1-a9"), CUDA events around each C-ABI call, best of 3."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2203_11484_b200 as V  # noqa: E402
import scenegen  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
s = scenegen.make_scene(cfg)
r = V.Renderer(s)
r.frame()
torch.cuda.synchronize()


def t(fn, reps=3):
    best = None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = e0.elapsed_time(e1) if best is None else min(best, e0.elapsed_time(e1))
    return best


out = {"config": s.name}
out["a1_scene_upload_ms"] = t(lambda: r.upload())
out["a2_build_bvh_ms"] = t(lambda: V.build_bvh(r.scene, r.n, r._bvh, r._bwork))
out["a3_classify_ms"] = t(lambda: V.classify_near_far(r.scene, r.n, s.T, labels=r.labels))
out["a4_a6_generate_vpls_ms"] = t(lambda: V.generate_vpls(r.scene, r.bvh, r.labels, r.n, s.M, s.K_near, s.max_depth,
                                                          s.rr, s.seed, max_out=r.max_out, vpls=r._vbuf, work=r._gwork))
out["a7_gbuffer_ms"] = t(lambda: V.render_gbuffer(r.scene, r.bvh, r.tiles, s.width, s.height, 16, 16, r.gbuf))
out["a8_gather_ms"] = t(lambda: V.gather_indirect(r.scene, r.bvh, r.gbuf, r.vpls, r.tiles, s.width, s.height, 16, 16,
                                                  r.rgb), reps=2)
out["f2_direct_16spp_ms"] = t(lambda: V.render_direct(r.scene, r.bvh, r.gbuf, r.tiles, s.width, s.height, samples=16,
                                                      seed=s.seed))
print(json.dumps(out))
