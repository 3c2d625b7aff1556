"""NEXT row f1 — the paper's equal-sample comparison on the
seeded synthetic scenes: the hybrid VPL set against plain instant
radiosity (the IR comparator: the same walk with every patch FAR, P:15, P:46
step 3 unrestricted) at the same VPL count M, both scored by RMS error against
a dense IR reference with > 200k VPLs ("more than 200k VPLs"), indirect
lighting only.  Every step is a libvplgi call: VPL generation,
G-buffer, gather and the error sums (vpl_image_error); this module only
orders the calls and times them.
"""
from __future__ import annotations

import torch

from . import (Renderer, all_tiles, gather_indirect, generate_metropolis, generate_rejection, generate_vpls,
               image_error)


def _timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = fn()
    e1.record()
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1)


def compare_estimators(scene, M_list=(1024, 4096), ref_M=262144, ref_seed=None, device="cuda", return_images=False,
                       pilot_factor=4, mh_burn=64, mh_radius=16):
    """Returns {"ref": {...}, "ref_hybrid": {...}, "runs": [{"M", "hybrid",
    "hybrid_vs_own", "ir", "rejection"}]}.  Rejection (f3, O15): an IR pilot of
    pilot_factor * M candidates scored at 64 probe pixels, M kept.  Metropolis
    (f4, O16): min(256, M) chains over the same pilot pool, burn-in mh_burn,
    mutation radius mh_radius, M states emitted.  Hybrid: near fraction K_near/M of the scene's
    own configuration; IR: all patches FAR (K = 0, M_far = M, budget rule O10).
    References (independent seed ref_seed, default scene.seed + 1000): dense
    IR with ref_M VPLs (the paper's reference) and the dense hybrid with
    ref_M VPLs — "hybrid_vs_own" scores the hybrid against its own limit (its
    variance alone); ref_hybrid's error against the IR reference is the
    hybrid's bias (the restricted walk drops every deposit on a near patch,
    P:46 step 3, so light reaching near patches after two or more bounces is
    not carried by any VPL)."""
    s = scene
    r = Renderer(s, device=device)
    r.frame()                                    # scene, BVH, labels, G-buffer (and one hybrid image)
    torch.cuda.synchronize()
    W, H = s.width, s.height
    tiles = all_tiles(W, H, 16, 16, r.device)
    frac = s.K_near / max(s.M, 1)
    far = torch.zeros_like(r.labels)             # IR comparator: every patch FAR

    def render(labels, M, K, seed):
        (v, info, _), t_gen = _timed(lambda: generate_vpls(r.scene, r.bvh, labels, r.n, M, K, s.max_depth, s.rr,
                                                           seed, max_out=max(M, 1)))
        (img, _), t_gat = _timed(lambda: gather_indirect(r.scene, r.bvh, r.gbuf, v, tiles, W, H, 16, 16))
        return img, info, t_gen, t_gat

    images = {}
    ref_seed = s.seed + 1000 if ref_seed is None else ref_seed
    ref_img, ref_info, tg, tt = render(far, ref_M, 0, ref_seed)
    refh_img, refh_info, thg, tht = render(r.labels, ref_M, int(frac * ref_M + 0.5), ref_seed)
    out = {"scene": s.name, "width": W, "height": H, "n_tris": s.n_tris,
           "ref": {"M": ref_M, "kind": "IR (all FAR)", "seed": ref_seed, "n_walks": ref_info["n_walks"],
                   "gen_ms": tg, "gather_ms": tt, "mean": float(ref_img.double().mean())},
           "ref_hybrid": dict(image_error(refh_img, ref_img), M=ref_M, K=refh_info["K"], gen_ms=thg, gather_ms=tht,
                              mean=float(refh_img.double().mean())),
           "runs": []}
    for M in M_list:
        K = int(frac * M + 0.5)
        h_img, h_info, hg, ht = render(r.labels, M, K, s.seed)
        i_img, i_info, ig, it = render(far, M, 0, s.seed)
        # rejection comparator (f3): IR pilot of pilot_factor * M candidates, keep M by probe score
        (pv, p_info, _), pg = _timed(lambda: generate_vpls(r.scene, r.bvh, far, r.n, pilot_factor * M, 0,
                                                           s.max_depth, s.rr, s.seed, max_out=pilot_factor * M))
        (rv, r_info), rg = _timed(lambda: generate_rejection(r.scene, r.bvh, pv, M, s.seed))
        (j_img, _), jt = _timed(lambda: gather_indirect(r.scene, r.bvh, r.gbuf, rv, tiles, W, H, 16, 16))
        # Metropolis comparator (f4): chains over the same pilot, M states emitted
        chains = min(256, M)
        (mv, m_info), mg = _timed(lambda: generate_metropolis(r.scene, r.bvh, pv, chains, M // chains, mh_burn,
                                                              mh_radius, s.seed))
        (k_img, _), kt = _timed(lambda: gather_indirect(r.scene, r.bvh, r.gbuf, mv, tiles, W, H, 16, 16))
        if return_images:
            images[M] = (h_img.clone(), i_img.clone(), j_img.clone(), k_img.clone())
        out["runs"].append({
            "M": M,
            "hybrid": dict(image_error(h_img, ref_img), K=h_info["K"], M_far=h_info["M_far"], gen_ms=hg,
                           gather_ms=ht),
            "hybrid_vs_own": image_error(h_img, refh_img),
            "ir": dict(image_error(i_img, ref_img), K=i_info["K"], M_far=i_info["M_far"], gen_ms=ig, gather_ms=it),
            "rejection": dict(image_error(j_img, ref_img), pilot=pilot_factor * M, accepted=r_info["accepted"],
                              n_scanned=r_info["n_scanned"], gen_ms=pg + rg, gather_ms=jt),
            "metropolis": dict(image_error(k_img, ref_img), pilot=pilot_factor * M, chains=chains,
                               per_chain=M // chains, accept_rate=m_info["accepted"] / (chains * (mh_burn + M // chains)),
                               gen_ms=pg + mg, gather_ms=kt),
        })
    if return_images:
        images["ref"] = ref_img
        images["ref_hybrid"] = refh_img
        return out, images
    return out
