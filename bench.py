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
# SURVEY §8(d)'s per-unit algorithmic cost (what the method must compute,
# excluding traversal control), thread-ops split by SM pipe, and bytes the
# unit requests from L2:   unit: (FMA pipe, ALU pipe, MUFU, L2 bytes)
OPS = {"pairs": (12, 2, 0, 0),        # every pair: d, r^2, 2 dots, cull (VPL record from smem / L1, amortised)
       "traced": (14, 1, 5, 0),       # traced pair: G, shadow-ray setup, accumulate
       "box_tests": (6, 11, 0, 32),   # per-ray child-box test (4-wide node: 32 B per child)
       "cone_tests": (6, 11, 0, 32),  # beam x child box (16-wide node child, or a list entry: 32 B)
       "tri_tests": (27, 7, 1, 48)}   # exact Moller-Trumbore test (triangle: 48 B)

# Roof rates: thread-ops per clock per SM — FMA pipe 128, ALU
# pipe 64 (FMNMX/FSETP/FSEL/LOP3, tools/pipebench.cu measured 63.7-64.0),
# MUFU 16, instruction issue 4 x 32; L2 read bandwidth measured by
# tools/pipebench.cu on this pool's B200 (profiles/r02_pipebench.jsonl).
PIPE = {"fma": 128.0, "alu": 64.0, "mufu": 16.0, "issue": 128.0}
FP32_PEAK_TFLOPS = 74.4   # BJ:5: 148 SMs x 128 FMA lanes x 2 flop x 1.965 GHz


def l2_bandwidth():
    f = ROOT / "profiles" / "r02_pipebench.jsonl"
    if f.exists():
        for line in f.read_text().splitlines():
            try:
                d = json.loads(line)
            except ValueError:
                continue
            if "GB_per_s" in d:
                return float(d["GB_per_s"]) * 1e9
    return None


def pipe_ops(c: dict) -> dict:
    return {p: sum(c[k] * v[i] for k, v in OPS.items()) for i, p in enumerate(("fma", "alu", "mufu", "l2_bytes"))}


def roof_terms(c: dict, sms: int, f_hz: float, l2_bps) -> dict:
    """T_roof = max(FMA/(128 SMs f), ALU/(64 SMs f), MUFU/(16 SMs f), L2 bytes/BW_L2);
    plus the issue limit (all ops / (128 SMs f)) that binds an issue-bound kernel."""
    o = pipe_ops(c)
    t = {"fma": o["fma"] / (PIPE["fma"] * sms * f_hz), "alu": o["alu"] / (PIPE["alu"] * sms * f_hz),
         "mufu": o["mufu"] / (PIPE["mufu"] * sms * f_hz)}
    if l2_bps:
        t["l2"] = o["l2_bytes"] / l2_bps
    t["issue"] = (o["fma"] + o["alu"] + o["mufu"]) / (PIPE["issue"] * sms * f_hz)
    return t


def sources_sha() -> str:
    """Hash of the CUDA sources and the ABI header: stamps which kernel version a committed ncu capture measured."""
    import hashlib
    h = hashlib.sha256()
    files = sorted((ROOT / "paper_2203_11484_b200" / "csrc").glob("*.cu*")) + [ROOT / "include" / "vplgi.h"]
    for f in files:
        h.update(f.name.encode())
        h.update(f.read_bytes())
    return h.hexdigest()[:12]


def measured_traffic():
    """dram read + write bytes of one C4 gather launch from the committed ncu
    capture (profiles/gather_c4_dram.csv) and the source hash it was taken on
    (profiles/gather_c4_dram.sha), or (None, None)."""
    import csv
    f, st = ROOT / "profiles" / "gather_c4_dram.csv", ROOT / "profiles" / "gather_c4_dram.sha"
    if not f.exists():
        return None, None
    tot, seen = 0.0, 0
    for r in csv.reader(f.read_text().splitlines()):
        if len(r) > 14 and r[12] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            tot += float(r[14].replace(",", ""))
            seen += 1
    return (tot if seen == 2 else None), (st.read_text().strip() if st.exists() else None)


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
    # VPLGI_BENCH_FORCE_DIST=1 (tests): take the collective path even with one rank, so that the NCCL
    # broadcasts / gather / reductions of the multi-rank frame execute on a one-GPU box
    use_dist = world > 1 or os.environ.get("VPLGI_BENCH_FORCE_DIST", "0") == "1"
    if use_dist:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    V.load_library()
    s = scenegen.make_scene(args.config)
    W, H, tw, th = s.width, s.height, 16, 16
    from paper_2203_11484_b200.parallel import FrameAssembler, tiles_for_rank
    tiles = tiles_for_rank(W, H, tw, th, rank, world, device=dev)
    assembler = FrameAssembler(W, H, tw, th, world, device=dev, force=use_dist)
    stream = torch.cuda.current_stream()

    # inputs resident in HBM (rank 0 owns the scene; the others receive it by broadcast)
    d_verts = torch.from_numpy(s.verts.reshape(-1)).to(dev)
    d_alb = torch.from_numpy(s.albedo.reshape(-1)).to(dev)
    r = V.Renderer(s, device=dev, tw=tw, th=th, tiles=tiles)
    vbuf = torch.empty(max(s.M, 1) * V.VPL_RECORD_BYTES, dtype=torch.uint8, device=dev)
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)   # > 126 MB L2

    ev = {k: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for k in ("step", "setup", "frame", "gather")}

    def setup():
        """scene setup (reported separately): broadcast, a1 upload, a2 BVH build"""
        if use_dist:
            dist.broadcast(d_verts, 0)
            dist.broadcast(d_alb, 0)
        r.upload(d_verts, d_alb, stream)
        r.bvh, r._bwork = V.build_bvh(r.scene, r.n, r._bvh, r._bwork, stream)
        r._bvh = r.bvh

    def frame(counters=False):
        """per frame: a3-a6 on rank 0 + VPL broadcast, a7 G-buffer and a8 gather of the rank's tiles,
        a9 framebuffer gather to rank 0"""
        if rank == 0:
            r.labels, r.n_near = V.classify_near_far(r.scene, r.n, s.T, stream=stream)
            r.vpls, r.info, r._gwork = V.generate_vpls(r.scene, r.bvh, r.labels, r.n, s.M, s.K_near, s.max_depth,
                                                      s.rr, s.seed, max_out=r.max_out, vpls=vbuf, work=r._gwork,
                                                      stream=stream)
        if use_dist:
            nv = torch.tensor([r.info["n_out"] if rank == 0 else 0], dtype=torch.int64, device=dev)
            dist.broadcast(nv, 0)
            n_out = int(nv.item())
            dist.broadcast(vbuf[: n_out * V.VPL_RECORD_BYTES], 0)
            r.vpls = vbuf[: n_out * V.VPL_RECORD_BYTES].view(-1, V.VPL_RECORD_BYTES)
        V.render_gbuffer(r.scene, r.bvh, r.tiles, W, H, tw, th, r.gbuf, stream)
        ev["gather"][0].record(stream)
        r._gawork = V.gather_work(r.vpls, W, H, dev, getattr(r, "_gawork", None))   # persistent scratch
        r.rgb, r.ctr = V.gather_indirect(r.scene, r.bvh, r.gbuf, r.vpls, r.tiles, W, H, tw, th, r.rgb, counters,
                                         work=r._gawork, stream=stream)
        ev["gather"][1].record(stream)
        assembler(r.rgb, rank, dst=0)
        return r.rgb

    def step(counters=False):
        """one pass of every §8(a) row: a1-a2 (setup) then a3-a9 (frame)"""
        ev["setup"][0].record(stream)
        setup()
        ev["setup"][1].record(stream)
        ev["frame"][0].record(stream)
        frame(counters)
        ev["frame"][1].record(stream)
        return r.rgb

    # pairs per step: front-hit pixels of the whole frame x VPLs
    def hit_pixels():
        g = r.gbuf.view(torch.int32).view(-1, 12)
        mine = ((g[:, 3] >= 0) & (g[:, 7] != 0)).sum()
        if use_dist:
            dist.all_reduce(mine)
        return int(mine.item())

    # counter pass (untimed): algorithmic work of the gather on these inputs
    step(counters=True)
    torch.cuda.synchronize()
    ctr = r.ctr.clone()
    if use_dist:
        dist.all_reduce(ctr)
    ctr = V.counters_dict(ctr.cpu())
    n_hit = hit_pixels()
    M = int(r.vpls.shape[0])
    pairs_per_step = n_hit * M

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    launches0 = V.launch_count()
    times = {k: [] for k in ("step", "setup", "frame", "gather")}
    with ClockSampler(gpu) as clk:
        for _ in range(args.steps):
            flush.zero_()                                   # L2 flush between timed steps (untimed)
            if use_dist:
                dist.barrier()
            torch.cuda.synchronize()
            ev["step"][0].record(stream)
            step()
            ev["step"][1].record(stream)
            torch.cuda.synchronize()
            for k in times:
                times[k].append(ev[k][0].elapsed_time(ev[k][1]))
    launches = (V.launch_count() - launches0) / max(args.steps, 1)
    t = {k: sum(v) / len(v) for k, v in times.items()}
    if use_dist:   # max over ranks
        tt = torch.tensor([t[k] for k in times], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = dict(zip(times, (float(x) for x in tt.cpu())))
    t_step, t_gather = t["step"], t["gather"]
    if rank == 0 and os.environ.get("VPLGI_BENCH_DUMP"):     # assembled frame (tests compare 1 vs N ranks)
        np.save(os.environ["VPLGI_BENCH_DUMP"], r.rgb.cpu().numpy())

    # e2e through the public API with host buffers: pinned H2D of the scene, D2H of the image
    h_verts = torch.from_numpy(s.verts.reshape(-1)).pin_memory()
    h_alb = torch.from_numpy(s.albedo.reshape(-1)).pin_memory()
    h_rgb = torch.empty(W * H * 3, dtype=torch.float32).pin_memory()
    e2e_ms = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(max(1, min(args.steps, 2))):
        flush.zero_()
        if use_dist:
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
    if use_dist:
        tt = torch.tensor([t_e2e], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_e2e = float(tt.item())

    cpu_base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu_base = cpu_baseline(s, r, args.cpu_seconds)

    if rank == 0:
        sm_count = V.device_info()["sm_count"]
        clocks = clk.summary()
        f_max = (clocks.get("sm_max_mhz") or _peaks()[0].get("sm_max_mhz", 1965.0)) * 1e6
        share = {k: v / max(world, 1) for k, v in ctr.items()}   # one rank's launch (equal shares)
        l2_bps = l2_bandwidth()
        terms = roof_terms(share, sm_count, f_max, l2_bps)
        o = pipe_ops(share)
        ops = o["fma"] + o["alu"] + o["mufu"]
        # headline: SM pipes + issue.  The L2 term of §8(d) counts every node / triangle byte the
        # algorithm requests; ~92% of those requests hit L1 (profiles/), so it is reported beside the
        # roof (frac_with_l2_requests) rather than taken as the bound.
        core = {k: v for k, v in terms.items() if k != "l2"}
        t_roof = max(core.values())
        t_roof_pipes = max(v for k, v in core.items() if k != "issue")
        binding = max(core, key=core.get)
        t_g = t_gather * 1e-3
        traffic, traffic_sha = measured_traffic() if args.config == 4 else (None, None)
        cur_sha = sources_sha()
        c = ctr
        pairs, traced = c["pairs"], c["traced"]
        out = {
            "metric": METRIC, "value": pairs_per_step / (t_step * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded scenegen)",
            "config": {"workload": f"C{args.config} (BASELINE.json configs[{args.config - 1}])",
                       "width": W, "height": H, "n_tris": s.n_tris, "n_lights": s.n_lights, "M": M,
                       "K_near": r.info.get("K"), "hit_pixels": n_hit,
                       "pairs_per_step": pairs_per_step, "parallelism": f"pixel-tiles x{world}",
                       "step": "a1-a2 scene setup + a3-a9 frame (SURVEY §8(a))",
                       "l2": "flushed between timed steps (512 MiB write)"},
            "scene_setup_ms": t["setup"], "frame_ms": t["frame"],
            "frame_pairs_per_s": pairs_per_step / (t["frame"] * 1e-3),
            "gather_ms": t_gather, "gather_pairs_per_s": pairs_per_step / t_g,
            "traced_fraction": traced / max(pairs, 1),
            "traced_pairs_per_s": traced / t_g,
            "counters": dict(c, tri_tests_per_traced=c["tri_tests"] / max(traced, 1),
                             steps_per_packet=c["warp_steps"] / max(c["warp_rays"], 1),
                             cone_packet_fraction=c["cone_packets"] / max(c["warp_rays"], 1),
                             cache_hit_fraction=c["cache_hits"] / max(traced, 1),
                             cache_tests_per_traced=c["cache_tests"] / max(traced, 1)),
            "roofline": {"bound": "alu", "binding_pipe": binding, "kernel": "k_gather",
                         "achieved": ops / t_g / 1e12, "peak": ops / t_roof / 1e12, "unit": "Tops/s",
                         "frac": t_roof / t_g, "frac_pipes_only": t_roof_pipes / t_g,
                         "frac_with_l2_requests": max(terms.values()) / t_g,
                         "t_roof_ms": {k: v * 1e3 for k, v in terms.items()},
                         "ops": {k: float(v) for k, v in o.items()},
                         "per_unit": {k: dict(zip(("fma", "alu", "mufu", "l2_bytes"), v)) for k, v in OPS.items()},
                         "fp32_flops_per_s": 2 * o["fma"] / t_g, "fp32_peak_flops_per_s": FP32_PEAK_TFLOPS * 1e12,
                         "fp32_note": "FMA-pipe algorithmic ops counted as FFMA (2 flop each): an upper bound",
                         "l2_bw_bytes_per_s": l2_bps, "sm_clock_hz": f_max, "sms": sm_count,
                         "traffic": traffic, "traffic_unit": "dram read + write bytes per launch "
                                                             "(profiles/gather_c4_dram.csv, ncu)",
                         "traffic_kernel_sha": traffic_sha, "kernel_sha": cur_sha,
                         "traffic_matches_build": traffic_sha == cur_sha,
                         "peak_source": "SURVEY §8(d) roof: per-unit algorithmic ops x counter-build counts of the "
                                        "same kernel; pipe rates FMA 128, ALU 64, MUFU 16, issue 128 "
                                        "thread-ops/clk/SM at the sampled max SM clock; L2 BW measured "
                                        "(tools/pipebench.cu, profiles/r02_pipebench.jsonl)"},
            "e2e": {"value": pairs_per_step / (t_e2e * 1e-3), "unit": UNIT, "ms": t_e2e,
                    "h2d_bytes_per_step": int(s.verts.nbytes + s.albedo.nbytes),
                    "d2h_bytes_per_step": int(W * H * 3 * 4)},
            "gpu_launches": int(round(launches)),
            "clocks": clocks,
            "cpu_baseline": cpu_base,
        }
        print(json.dumps(out))
    if use_dist:
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
