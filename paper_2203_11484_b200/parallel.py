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


class FrameAssembler:
    """Framebuffer assembly by gather (BJ:5 "framebuffer assembled
    with NCCL gather"): each rank packs the pixels of its own tiles (in-image
    pixels, tile order) into a compact buffer, `dist.gather` brings the G
    buffers to `dst`, which scatters every other rank's pixels into its frame.
    Pure data movement (no arithmetic): `dst`'s frame equals composing the
    tiles directly, bitwise.  Buffers are padded to the largest share (tile
    counts differ by at most one); the pad repeats a valid pixel and is
    dropped on unpacking.  Works on CUDA (NCCL) and CPU (gloo) tensors."""

    def __init__(self, W, H, tw, th, world, device="cpu", force=False):
        self.world = world
        self.force = force   # run the gather even with one rank (tests: the NCCL path on a one-GPU box)
        owner = tile_owner(W, H, tw, th, world)
        tx = (W + tw - 1) // tw
        ys, xs = np.meshgrid(np.arange(th), np.arange(tw), indexing="ij")
        self.idx, self.n = [], []
        for r in range(world):
            t = np.nonzero(owner == r)[0]
            x = (t % tx)[:, None, None] * tw + xs[None]
            y = (t // tx)[:, None, None] * th + ys[None]
            ok = (x < W) & (y < H)
            self.idx.append((y * W + x)[ok].astype(np.int64))
            self.n.append(int(ok.sum()))
        self.n_max = max(self.n) if self.n else 0
        self.idx_pad = []
        for r in range(world):
            a = self.idx[r]
            pad = np.full(self.n_max - len(a), a[0] if len(a) else 0, np.int64)
            self.idx_pad.append(torch.from_numpy(np.concatenate([a, pad])).to(device))
        self.idx = [torch.from_numpy(a).to(device) for a in self.idx]
        self.bytes_per_rank = self.n_max * 12

    def __call__(self, rgb: torch.Tensor, rank: int, group=None, dst=0):
        import torch.distributed as dist
        if self.world == 1 and not self.force:
            return rgb
        v = rgb.view(-1, 3)
        send = v.index_select(0, self.idx_pad[rank])
        # gloo gathers host tensors only (the functional multi-rank check on one GPU); NCCL gathers in HBM
        host = dist.get_backend(group) == "gloo" and send.is_cuda
        if host:
            send = send.cpu()
        recv = [torch.empty_like(send) for _ in range(self.world)] if rank == dst else None
        dist.gather(send, recv, dst=dst, group=group)
        if rank == dst:
            for r in range(self.world):
                if r != dst and self.n[r]:
                    v.index_copy_(0, self.idx[r], recv[r][: self.n[r]].to(v.device))
        return rgb
