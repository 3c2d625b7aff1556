"""bench.py — one step = one pass of the whole hot path (SURVEY §8(a) rows
a1-a8, plus a9 assembly for N > 1) over BASELINE.json's C4 workload
(configs[3]: 1080p, ~1M triangles, 65,536 VPLs, BJ:10).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]

Headline metric (BJ:2): pixel x VPL shadow-tested contributions per second =
(front-hit pixels x M) / step time, whole job.  The reference arm
(--impl reference) times the CPU oracle (oracle/, the only other place this
file executes it) on a bounded pixel sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "pixel×VPL shadow-tested contributions/sec; ms/frame at 1080p, 64k VPLs"
UNIT = "pairs/s"


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return json.loads(p.read_text()), "measured"
        except Exception:
            pass
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index=0, period_ms=200):
        self.index, self.period_ms = index, period_ms
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", f"-lms={self.period_ms}"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for k, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(k)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------- algorithmic op counts
# Per-unit thread-op counts: the arithmetic the method itself prescribes per
# unit of work, split by the SM pipe that executes it.  The
# exact fp32 contract (O0) forbids FMA contraction in the Eq. 1 terms and the
# segment setup, so those count as separate FMUL/FADD; the any-hit MT counts
# the fused form of reading R26; square roots and divisions count as one MUFU
# op each.  (fma, alu, mufu) per unit:
OPS = {"pairs": (14, 3, 0),       # d (3), r^2 (5), cx (3, fused), ci (3, fused) | tri, cx, ci tests (O13, R26)
       "traced": (9, 2, 2),       # tmax, cx*ci, r2*max, 3 FFMA, d*inv (3) | test, max | sqrt, 1/dist  (O9, O13, R25)
       "box_tests": (12, 5, 0),   # per-ray slab (centre/half-extent): 3 FFMA + 3 FMUL + 6 FADD | 4 min/max + cmp
       "cone_tests": (6, 11, 0),  # beam x child box: 6 FFMA | 6 SEL + 4 min/max + 1 cmp (gather.cuh beam_box)
       "tri_tests": (30, 9, 0)}   # exact MT any hit (O9, R25, R26): 27 FMUL/FFMA/FADD + a_u+a_v, tmin*D, tmax*D | 6 compares + 3 sign flips

# Pipe rates in thread-ops per clock per SM, measured on this pool's B200
# (tools/pipebench.cu, profiles/r01_pipebench.jsonl): FFMA/FMUL/FADD 126,
# FMNMX/FSETP/FSEL/LOP3 64, MUFU.RCP 14.6; instruction issue 4 warps x 32.
PIPE = {"fma": 128.0, "alu": 64.0, "mufu": 16.0, "issue": 128.0}


def algorithmic_ops(c: dict) -> int:
    return sum(c[k] * sum(v) for k, v in OPS.items())


def roof_seconds(c: dict, sms: int, f_hz: float) -> tuple[float, str]:
    """T_roof = max over pipes of ops / (rate * SMs * f); returns (T, binding pipe)."""
    fma = sum(c[k] * v[0] for k, v in OPS.items())
    alu = sum(c[k] * v[1] for k, v in OPS.items())
    mufu = sum(c[k] * v[2] for k, v in OPS.items())
    t = {"fma": fma / PIPE["fma"], "alu": alu / PIPE["alu"], "mufu": mufu / PIPE["mufu"],
         "issue": (fma + alu + mufu) / PIPE["issue"]}
    k = max(t, key=t.get)
    return t[k] / (sms * f_hz), k


def measured_traffic():
    """dram read + write bytes of one C4 gather launch from the committed ncu
    capture (profiles/r01_gather_c4_dram.csv), or None."""
    import csv
    f = ROOT / "profiles" / "r01_gather_c4_dram.csv"
    if not f.exists():
        return None
    tot, seen = 0.0, 0
    for r in csv.reader(f.read_text().splitlines()):
        if len(r) > 14 and r[12] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            tot += float(r[14].replace(",", ""))
            seen += 1
    return tot if seen == 2 else None


# ---------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2203_11484_b200 as V
    import scenegen

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one GPU per rank; VPLGI_BENCH_BACKEND=gloo + fewer GPUs than ranks is a functional
    # check of the multi-rank path only (ranks share a GPU, timings are not scaling numbers)
    backend = os.environ.get("VPLGI_BENCH_BACKEND", "nccl")
    gpu = local % torch.cuda.device_count() if backend != "nccl" else local
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    V.load_library()
    s = scenegen.make_scene(args.config)
    W, H, tw, th = s.width, s.height, 16, 16
    from paper_2203_11484_b200.parallel import tiles_for_rank
    tiles = tiles_for_rank(W, H, tw, th, rank, world, device=dev)
    stream = torch.cuda.current_stream()

    # inputs resident in HBM (rank 0 owns the scene; others receive it by broadcast each step)
    d_verts = torch.from_numpy(s.verts.reshape(-1)).to(dev)
    d_alb = torch.from_numpy(s.albedo.reshape(-1)).to(dev)
    r = V.Renderer(s, device=dev, tw=tw, th=th, tiles=tiles)
    vbuf = torch.empty(max(s.M, 1) * V.VPL_RECORD_BYTES, dtype=torch.uint8, device=dev)
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)   # > 126 MB L2

    ev = {k: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for k in ("step", "gather")}
    state = {}

    def step(counters=False):
        if world > 1:
            # the frame is assembled by an in-place SUM all-reduce, so every rank's buffer
            # holds the other ranks' tiles afterwards: they must start from zero every step
            r.rgb.zero_()
            dist.broadcast(d_verts, 0)
            dist.broadcast(d_alb, 0)
        r.upload(d_verts, d_alb, stream)
        r.bvh, r._bwork = V.build_bvh(r.scene, r.n, r._bvh, r._bwork, stream)
        r._bvh = r.bvh
        if rank == 0:
            r.labels, r.n_near = V.classify_near_far(r.scene, r.n, s.T, stream=stream)
            r.vpls, r.info, r._gwork = V.generate_vpls(r.scene, r.bvh, r.labels, r.n, s.M, s.K_near, s.max_depth,
                                                      s.rr, s.seed, max_out=r.max_out, vpls=vbuf, work=r._gwork,
                                                      stream=stream)
            nv = torch.tensor([r.info["n_out"]], dtype=torch.int64, device=dev)
        else:
            nv = torch.zeros(1, dtype=torch.int64, device=dev)
        if world > 1:
            dist.broadcast(nv, 0)
            n_out = int(nv.item())
            dist.broadcast(vbuf[: n_out * V.VPL_RECORD_BYTES], 0)
            r.vpls = vbuf[: n_out * V.VPL_RECORD_BYTES].view(-1, V.VPL_RECORD_BYTES)
        V.render_gbuffer(r.scene, r.bvh, r.tiles, W, H, tw, th, r.gbuf, stream)
        ev["gather"][0].record(stream)
        r.rgb, r.ctr = V.gather_indirect(r.scene, r.bvh, r.gbuf, r.vpls, r.tiles, W, H, tw, th, r.rgb, counters,
                                         stream=stream)
        ev["gather"][1].record(stream)
        if world > 1:
            dist.all_reduce(r.rgb, op=dist.ReduceOp.SUM)     # disjoint tiles: exact assembly on every rank
        return r.rgb

    # pairs per step: front-hit pixels of the whole frame x VPLs
    def hit_pixels():
        g = r.gbuf.view(torch.int32).view(-1, 12)
        mine = ((g[:, 3] >= 0) & (g[:, 7] != 0)).sum()
        if world > 1:
            dist.all_reduce(mine)
        return int(mine.item())

    # counter pass (untimed): algorithmic work of the gather on these inputs
    step(counters=True)
    torch.cuda.synchronize()
    ctr = r.ctr.clone()
    if world > 1:
        dist.all_reduce(ctr)
    ctr = V.counters_dict(ctr.cpu())
    n_hit = hit_pixels()
    M = int(r.vpls.shape[0])
    pairs_per_step = n_hit * M

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    launches0 = V.launch_count()
    step_ms, gather_ms = [], []
    with ClockSampler(gpu) as clk:
        for _ in range(args.steps):
            flush.zero_()                                   # L2 flush between timed steps (untimed)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            ev["step"][0].record(stream)
            step()
            ev["step"][1].record(stream)
            torch.cuda.synchronize()
            step_ms.append(ev["step"][0].elapsed_time(ev["step"][1]))
            gather_ms.append(ev["gather"][0].elapsed_time(ev["gather"][1]))
    launches = (V.launch_count() - launches0) / max(args.steps, 1)
    t_step = sum(step_ms) / len(step_ms)
    t_gather = sum(gather_ms) / len(gather_ms)
    if world > 1:
        tt = torch.tensor([t_step, t_gather], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step, t_gather = (float(x) for x in tt.cpu())

    # e2e through the public API with host buffers: pinned H2D of the scene, D2H of the image
    h_verts = torch.from_numpy(s.verts.reshape(-1)).pin_memory()
    h_alb = torch.from_numpy(s.albedo.reshape(-1)).pin_memory()
    h_rgb = torch.empty(W * H * 3, dtype=torch.float32).pin_memory()
    e2e_ms = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(max(1, min(args.steps, 2))):
        flush.zero_()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        if rank == 0:
            d_verts.copy_(h_verts, non_blocking=True)
            d_alb.copy_(h_alb, non_blocking=True)
        step()
        if rank == 0:
            h_rgb.copy_(r.rgb, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
    t_e2e = sum(e2e_ms) / len(e2e_ms)
    if world > 1:
        tt = torch.tensor([t_e2e], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_e2e = float(tt.item())

    cpu_base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu_base = cpu_baseline(s, r, args.cpu_seconds)

    if rank == 0:
        peaks, peak_src = _peaks()
        sm_count = V.device_info()["sm_count"]
        clocks = clk.summary()
        f_max = (clocks.get("sm_max_mhz") or peaks.get("sm_max_mhz", 1965.0)) * 1e6
        ops = algorithmic_ops(ctr) / max(world, 1)              # per launch (one rank's share)
        share = {k: v / max(world, 1) for k, v in ctr.items()}
        t_roof, binding = roof_seconds(share, sm_count, f_max)
        achieved = ops / (t_gather * 1e-3)
        peak_ops = ops / t_roof                                  # the pipe roof for this op mix
        c = ctr
        pairs, traced = c["pairs"], c["traced"]
        out = {
            "metric": METRIC, "value": pairs_per_step / (t_step * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded scenegen)",
            "config": {"workload": f"C{args.config} (BASELINE.json configs[{args.config - 1}])",
                       "width": W, "height": H, "n_tris": s.n_tris, "n_lights": s.n_lights, "M": M,
                       "K_near": r.info.get("K") if rank == 0 else None, "hit_pixels": n_hit,
                       "pairs_per_step": pairs_per_step, "parallelism": f"pixel-tiles x{world}",
                       "l2": "flushed between timed steps (512 MiB write)"},
            "gather_ms": t_gather, "gather_pairs_per_s": pairs_per_step / (t_gather * 1e-3),
            "traced_fraction": traced / max(pairs, 1),
            "traced_pairs_per_s": traced / (t_gather * 1e-3),
            "counters": dict(c, tri_tests_per_traced=c["tri_tests"] / max(traced, 1),
                             steps_per_packet=c["warp_steps"] / max(c["warp_rays"], 1),
                             cone_packet_fraction=c["cone_packets"] / max(c["warp_rays"], 1),
                             cache_hit_fraction=c["cache_hits"] / max(traced, 1),
                             cache_tests_per_traced=c["cache_tests"] / max(traced, 1)),
            "roofline": {"bound": "alu", "kernel": "k_gather", "achieved": achieved / 1e12,
                         "peak": peak_ops / 1e12, "unit": "Tops/s", "frac": achieved / peak_ops,
                         "binding_pipe": binding, "t_roof_ms": t_roof * 1e3,
                         "traffic": measured_traffic() if args.config == 4 else None,
                         "traffic_unit": "bytes per launch (dram read + write, profiles/r01_gather_c4_dram.csv)",
                         "peak_source": f"derived: {sm_count} SMs x {f_max / 1e6:.0f} MHz x measured pipe rates "
                                        f"(FMA 128, ALU 64, MUFU 16, issue 128 thread-ops/clk/SM; "
                                        f"profiles/r01_pipebench.jsonl), max over pipes for this op mix "
                                        f"(DESIGN.md §5)"},
            "e2e": {"value": pairs_per_step / (t_e2e * 1e-3), "unit": UNIT, "ms": t_e2e,
                    "h2d_bytes_per_step": int(s.verts.nbytes + s.albedo.nbytes),
                    "d2h_bytes_per_step": int(W * H * 3 * 4)},
            "gpu_launches": int(round(launches)),
            "clocks": clocks,
            "cpu_baseline": cpu_base,
        }
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


def cpu_baseline(s, r, budget_s=15.0, sample_pixels=None):
    """The oracle gather, as it stands, on a bounded pixel sample of the same
    frame (its own G-buffer points; the frame's VPL array), OpenMP over the
    host cores.  Returns pairs/s over the sample."""
    import oracle
    import paper_2203_11484_b200 as V

    o = oracle.OracleScene(s)
    gv = V.decode_vpls(r.vpls)
    ov = np.zeros(len(gv), oracle.VPL_DTYPE)
    for k in ("pos", "nrm", "flux", "tri"):
        ov[k] = gv[k]
    th = oracle.threads()
    rng = np.random.default_rng(7)
    done_px, t_used = 0, 0.0
    chunk = max(th, 8)
    while t_used < budget_s and done_px < 4096:
        px = rng.integers(0, s.width * s.height, chunk).astype(np.int32)
        gb = o.gbuffer(px)
        t0 = time.perf_counter()
        o.gather(gb, ov)
        t_used += time.perf_counter() - t0
        done_px += chunk
    pairs = done_px * len(ov)
    return {"value": pairs / t_used, "unit": UNIT, "cores": th, "kind": "oracle",
            "sample": f"oracle gather of {done_px} random pixels x {len(ov)} VPLs of C4 (brute-force "
                      f"visibility over {s.n_tris} tris), {t_used:.1f} s"}


# ---------------------------------------------------------------------------- reference arm (the oracle)
def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    import scenegen

    s = scenegen.make_scene(args.config)
    o = oracle.OracleScene(s)
    lab, _ = o.classify()
    # bounded sample of the workload: the oracle's own VPL generation is
    # C4-sized (~1 min); the timed steps are pixel samples of its gather
    t0 = time.perf_counter()
    v, info = o.generate_vpls(lab)
    t_gen = time.perf_counter() - t0
    th = oracle.threads()
    rng = np.random.default_rng(11)
    per_step = max(th, 8)
    for _ in range(args.warmup):
        pass                                                # the oracle has nothing to warm
    times = []
    for _ in range(args.steps):
        px = rng.integers(0, s.width * s.height, per_step).astype(np.int32)
        gb = o.gbuffer(px)
        t0 = time.perf_counter()
        o.gather(gb, v)
        times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    val = per_step * len(v) / t
    out = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded scenegen)",
           "config": {"workload": f"C{args.config} (BASELINE.json configs[{args.config - 1}])",
                      "width": s.width, "height": s.height, "n_tris": s.n_tris, "M": len(v),
                      "sample_pixels_per_step": per_step},
           "cpu_baseline": {"value": val, "unit": UNIT, "cores": th, "kind": "oracle",
                            "sample": f"{per_step} random pixels x {len(v)} VPLs per step; oracle VPL "
                                      f"generation {t_gen:.1f} s untimed"},
           "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("note: warmup raised to the 3-step minimum", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
