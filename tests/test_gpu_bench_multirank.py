"""Functional check of bench.py's multi-rank path (broadcast of scene and
VPLs, per-rank tile gather, framebuffer gather to rank 0, max-over-ranks
timing, rank-0 JSON line): two ranks launched by torch.distributed.run share
the one GPU of the test box over gloo (VPLGI_BENCH_BACKEND=gloo).  The ranks
never wait on one another inside a kernel; the timings are not scaling
numbers.  The assembled 2-rank frame must equal the 1-rank frame bitwise
(SURVEY §8(e))."""
from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _run(n, port, dump, cfg, backend="gloo", force_dist=False):
    env = dict(os.environ, VPLGI_BENCH_BACKEND=backend, VPLGI_BENCH_DUMP=str(dump),
               VPLGI_BENCH_FORCE_DIST="1" if force_dist else "0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"), "--gpus", str(n),
           "--steps", "1", "--warmup", "3", "--config", str(cfg), "--no-cpu-baseline"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0]), np.load(dump)


@pytest.mark.parametrize("cfg", [1, 2])
def test_two_ranks_match_one_rank(cfg, tmp_path):
    (one, img1) = _run(1, 29531 + 10 * cfg, tmp_path / "one.npy", cfg)
    (two, img2) = _run(2, 29532 + 10 * cfg, tmp_path / "two.npy", cfg)
    assert np.array_equal(img1.view(np.uint32), img2.view(np.uint32))      # assembled frame, bitwise
    assert np.abs(img1).sum() > 0
    assert two["n_gpus"] == 2 and two["config"]["parallelism"] == "pixel-tiles x2"
    for k in ("pairs", "traced", "visible"):
        assert two["counters"][k] == one["counters"][k], k      # the tiles of both ranks cover the frame once
    assert two["config"]["hit_pixels"] == one["config"]["hit_pixels"]
    assert two["value"] > 0 and two["e2e"]["value"] > 0


@pytest.mark.parametrize("cfg", [1, 2])
def test_nccl_collective_path_one_rank(cfg, tmp_path):
    """The NCCL code path of the multi-rank frame — scene and VPL broadcasts, hit-pixel / counter / timing
    all-reduces, barriers, the framebuffer gather on CUDA tensors — executed with a one-rank NCCL
    communicator on the test GPU (NCCL refuses two ranks on one device, so this is what a one-GPU box can
    run of it): the frame must equal the plain one-rank frame bitwise."""
    (plain, img1) = _run(1, 29571 + 10 * cfg, tmp_path / "plain.npy", cfg)
    (nccl, img2) = _run(1, 29572 + 10 * cfg, tmp_path / "nccl.npy", cfg, backend="nccl", force_dist=True)
    assert np.array_equal(img1.view(np.uint32), img2.view(np.uint32))
    for k in ("pairs", "traced", "visible"):
        assert nccl["counters"][k] == plain["counters"][k], k
    assert nccl["n_gpus"] == 1 and nccl["value"] > 0 and nccl["e2e"]["value"] > 0
