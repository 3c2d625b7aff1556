"""Shared helpers for the -m gpu parity tests: run the CUDA path through the
C ABI (paper_2203_11484_b200) and the oracle on the same seeded scene and
compare.  Tolerances follow BJ:5."""
from __future__ import annotations

import numpy as np
import torch

import oracle
import paper_2203_11484_b200 as V

MRE_TOL = 1e-4          # mean relative error of the indirect image (BJ:5)
PIXEL_TOL = 1e-3        # per-pixel relative error where visibility agrees (BJ:5)
VIS_TOL = 1e-4          # pixel x VPL visibility disagreements / traced pairs (BJ:5)


class GpuScene:
    def __init__(self, s, device="cuda"):
        self.s = s
        self.scene, self.bad, self.n = V.scene_upload(s.verts, s.albedo, s.lights, s.cam, s.width, s.height, device)
        self.bvh, _ = V.build_bvh(self.scene, self.n)
        torch.cuda.synchronize()

    def labels(self, T=None):
        lab, nn = V.classify_near_far(self.scene, self.n, self.s.T if T is None else T)
        return lab.cpu().numpy(), int(nn.item())

    def generate(self, labels=None, **kw):
        s = self.s
        if labels is None:
            lab, _ = V.classify_near_far(self.scene, self.n, s.T)
        else:
            lab = torch.from_numpy(np.ascontiguousarray(labels, np.uint8)).cuda()
        args = dict(M=s.M, K_near=s.K_near, max_depth=s.max_depth, rr=s.rr, seed=s.seed)
        args.update(kw)
        v, info, _ = V.generate_vpls(self.scene, self.bvh, lab, self.n, **args)
        return v, info

    def gbuffer(self, tw=16, th=16):
        tiles = V.all_tiles(self.s.width, self.s.height, tw, th)
        return V.render_gbuffer(self.scene, self.bvh, tiles, self.s.width, self.s.height, tw, th), tiles


def vpls_to_oracle(v: np.ndarray) -> np.ndarray:
    out = np.zeros(len(v), oracle.VPL_DTYPE)
    out["pos"], out["nrm"], out["flux"] = v["pos"], v["nrm"], v["flux"]
    out["tri"] = v["tri"]
    out["tag"] = v["tag_depth"] & 0xFF
    out["depth"] = v["tag_depth"] >> 8
    out["walk"] = v["walk"]
    return out


def gbuf_to_oracle(g: np.ndarray) -> np.ndarray:
    out = np.zeros(len(g), oracle.GBUF_DTYPE)
    for k in ("pos", "nrm", "alb", "t", "tri", "front"):
        out[k] = g[k]
    return out


def assert_vpls_bitwise(gv: np.ndarray, ov: np.ndarray):
    assert len(gv) == len(ov), (len(gv), len(ov))
    go = vpls_to_oracle(gv)
    for k in ("tri", "tag", "depth", "walk"):
        bad = np.nonzero(go[k] != ov[k])[0]
        assert bad.size == 0, (k, bad[:10], go[k][bad[:5]], ov[k][bad[:5]])
    for k in ("pos", "nrm", "flux"):
        a, b = go[k].view(np.uint32), ov[k].view(np.uint32)
        bad = np.nonzero(np.any(a != b, axis=1))[0]
        assert bad.size == 0, (k, bad[:10], go[k][bad[:3]], ov[k][bad[:3]])


def compare_images(g_rgb: np.ndarray, o_rgb64: np.ndarray, agree: np.ndarray | None = None):
    """g_rgb, o_rgb64: [P, 3] on the compared pixels; agree: [P] bool (visibility identical)."""
    den = np.abs(o_rgb64).sum()
    mre = np.abs(g_rgb.astype(np.float64) - o_rgb64).sum() / max(den, 1e-300)
    floor = 1e-3 * np.abs(o_rgb64).mean()
    rel = np.abs(g_rgb - o_rgb64).max(1) / np.maximum(np.abs(o_rgb64).max(1), max(floor, 1e-30))
    if agree is not None:
        rel = rel[agree]
    return mre, (rel.max() if rel.size else 0.0)


def vis_disagreement(gt, gv, ot, ov):
    """bit arrays [P, words] (int32 / uint32): returns (#traced-bit mismatches,
    #visible-bit mismatches among pairs both traced, #traced pairs)."""
    gt, gv = gt.view(np.uint32), gv.view(np.uint32)
    ot, ov = ot.view(np.uint32), ov.view(np.uint32)
    popc = np.vectorize(lambda x: bin(int(x)).count("1"))
    traced_mis = int(popc(gt ^ ot).sum())
    both = gt & ot
    vis_mis = int(popc((gv ^ ov) & both).sum())
    n_traced = int(popc(ot).sum())
    per_pixel_agree = np.all(gt == ot, axis=1) & np.all(((gv ^ ov) & both) == 0, axis=1)
    return traced_mis, vis_mis, n_traced, per_pixel_agree


def sample_pixels(W, H, P, seed=3):
    """P pixels: one per block of a sqrt(P) x sqrt(P) grid, seeded offset (§8(c))."""
    g = int(round(np.sqrt(P)))
    rng = np.random.default_rng(seed)
    out = []
    for by in range(g):
        for bx in range(g):
            x0, x1 = bx * W // g, (bx + 1) * W // g
            y0, y1 = by * H // g, (by + 1) * H // g
            out.append(int(rng.integers(y0, y1)) * W + int(rng.integers(x0, x1)))
    return np.array(out, np.int32)
