"""Pixel-tile sharding across ranks (BJ:5 "work is partitioned
by pixel tiles, scene and VPLs replicated").  Tile t goes to rank
perm(t) mod G with perm a fixed seeded permutation, so every rank gets a
spatially interleaved, load-balanced share; each pixel's VPL loop is
independent of the map, so any G reproduces the 1-GPU image bitwise.
Host logic only; the collectives are torch.distributed (NCCL on GPUs, gloo in
the CPU tests)."""
from __future__ import annotations

import numpy as np
import torch

TILE_PERM_SEED = 0x5EED


def n_tiles(W, H, tw=16, th=16):
    return ((W + tw - 1) // tw) * ((H + th - 1) // th)


def tile_owner(W, H, tw, th, world):
    """owner[t] = rank of tile t."""
    nt = n_tiles(W, H, tw, th)
    perm = np.random.default_rng(TILE_PERM_SEED).permutation(nt)
    owner = np.empty(nt, np.int32)
    owner[perm] = np.arange(nt) % world
    return owner


def tiles_for_rank(W, H, tw, th, rank, world, device="cpu"):
    owner = tile_owner(W, H, tw, th, world)
    t = np.nonzero(owner == rank)[0].astype(np.int32)
    return torch.from_numpy(t).to(device)


def tile_pixel_mask(W, H, tw, th, tiles):
    """bool [H*W] mask of the pixels covered by `tiles`."""
    tx = (W + tw - 1) // tw
    m = np.zeros((H, W), bool)
    for t in np.asarray(tiles.cpu() if isinstance(tiles, torch.Tensor) else tiles):
        x0, y0 = (t % tx) * tw, (t // tx) * th
        m[y0:y0 + th, x0:x0 + tw] = True
    return m.reshape(-1)


def assemble(rgb_local: torch.Tensor, group=None, dst=0):
    """Framebuffer assembly: every rank holds a zero-initialised full frame
    with only its own tiles written; a SUM reduce to `dst` is bitwise equal to
    gathering the tiles (x + 0 = x exactly).  The reduce is in place: `dst`'s
    buffer then holds every rank's tiles, so zero it before the next frame."""
    import torch.distributed as dist
    dist.reduce(rgb_local, dst, op=dist.ReduceOp.SUM, group=group)
    return rgb_local
