"""Multi-GPU scaling estimate on one GPU: the G ranks of the
pixel-tile sharding do not wait on one another (each gathers its own tiles
with the replicated scene, BVH and VPLs), so each rank's gather can be timed
alone, one after the other, on a single B200.  Reports, per G, every rank's
gather time, the load-balance efficiency T(1) / (G * max_r T_r) of the
gather, the frame efficiency of SURVEY §8(e) — T = VPL generation on rank 0
+ VPL broadcast + G-buffer of the rank's tiles + gather + framebuffer gather
(collectives at the measured 770 GB/s NVLink bus bandwidth of
B200_PROFILING.md) — and the step efficiency with the replicated scene setup
(upload, BVH build, scene broadcast) added, which §8(e) reports separately.  This is an emulation:
the driver's `bench.py --gpus N` runs are the measurement.

  python tools/shard_sim.py --config 4 --gpus 2 4 8
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2203_11484_b200 as V  # noqa: E402
import scenegen  # noqa: E402
from paper_2203_11484_b200.parallel import tiles_for_rank  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--gpus", type=int, nargs="+", default=[2, 4, 8])
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--tile", type=int, nargs=2, default=[16, 16], help="partition tile w h (multiples of 8, 4)")
a = ap.parse_args()

s = scenegen.make_scene(a.config)
tw, th = a.tile
r = V.Renderer(s, tw=tw, th=th)
torch.cuda.synchronize()
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def timed(fn):
    best = None
    for _ in range(a.reps):
        e0, e1 = ev(), ev()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1)
        best = t if best is None else min(best, t)
    return best


# scene setup (replicated on every rank, reported separately) and the per-frame VPL generation (rank 0)
def setup():
    r.upload()
    r.bvh, r._bwork = V.build_bvh(r.scene, r.n, r._bvh, r._bwork)
    r._bvh = r.bvh


def vplgen():
    r.labels, r.n_near = V.classify_near_far(r.scene, r.n, s.T)
    r.vpls, r.info, r._gwork = V.generate_vpls(r.scene, r.bvh, r.labels, r.n, s.M, s.K_near, s.max_depth, s.rr,
                                               s.seed, max_out=r.max_out, vpls=r._vbuf, work=r._gwork)


t_setup = timed(setup)
t_gen = timed(vplgen)
t_gb = timed(lambda: V.render_gbuffer(r.scene, r.bvh, r.tiles, s.width, s.height, tw, th, r.gbuf))
t1 = timed(lambda: V.gather_indirect(r.scene, r.bvh, r.gbuf, r.vpls, r.tiles, s.width, s.height, tw, th, r.rgb))
bw = 770e9
scene_bcast_ms = (s.verts.nbytes + s.albedo.nbytes) / bw * 1e3
vpl_bcast_ms = r.vpls.numel() / bw * 1e3
fb_ms = (s.width * s.height * 12) / bw * 1e3           # every pixel crosses NVLink once into rank 0
out = {"config": s.name, "tile": [tw, th], "t1_gather_ms": t1, "scene_setup_ms": t_setup, "vplgen_ms": t_gen,
       "gbuffer_full_ms": t_gb, "scene_bcast_ms_est": scene_bcast_ms, "vpl_bcast_ms_est": vpl_bcast_ms,
       "fb_gather_ms_est": fb_ms, "runs": []}
frame1 = t_gen + t_gb + t1
step1 = t_setup + frame1
for G in a.gpus:
    tr = []
    for rank in range(G):
        tiles = tiles_for_rank(s.width, s.height, tw, th, rank, G, device="cuda")
        tr.append(timed(lambda: V.gather_indirect(r.scene, r.bvh, r.gbuf, r.vpls, tiles, s.width, s.height, tw, th,
                                                  r.rgb)))
    tmax = max(tr)
    frameG = t_gen + vpl_bcast_ms + t_gb / G + tmax + fb_ms
    stepG = t_setup + scene_bcast_ms + frameG
    out["runs"].append({"G": G, "rank_gather_ms": tr, "gather_efficiency": t1 / (G * tmax),
                        "frame_ms_est": frameG, "frame_efficiency_est": frame1 / (G * frameG),
                        "step_ms_est": stepG, "step_efficiency_est": step1 / (G * stepG)})
print(json.dumps(out), flush=True)
