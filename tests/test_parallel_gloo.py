"""Multi-rank host logic on CPU (gloo, world_size 2 and 3): the pixel-tile
partition covers every tile exactly once, every rank's share is balanced,
and the framebuffer assembly (gather of each rank's packed tile pixels to
rank 0, §8(e); the code bench.py runs under NCCL) equals composing the tiles
directly, bitwise.  The per-tile "render" here is a
deterministic stand-in (CPU), because the CUDA kernels need a GPU; the
partition/assembly code is the one bench.py runs under NCCL."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2203_11484_b200.parallel import FrameAssembler, n_tiles, tile_owner, tile_pixel_mask, tiles_for_rank


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def fake_render(W, H, tiles, tw, th):
    """stand-in for render_gbuffer + gather_indirect on a tile list: a
    pixel-dependent value written only on the listed tiles"""
    rgb = torch.zeros(H * W * 3, dtype=torch.float32)
    m = torch.from_numpy(tile_pixel_mask(W, H, tw, th, tiles))
    px = torch.arange(H * W, dtype=torch.float64)
    val = (torch.sin(px * 0.37) ** 2 + 1e-3).to(torch.float32)
    v3 = rgb.view(-1, 3)
    v3[m] = torch.stack([val[m], 2 * val[m], 3 * val[m]], 1)
    return rgb


def _worker(rank, world, port, W, H, tw, th, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    tiles = tiles_for_rank(W, H, tw, th, rank, world)
    rgb = fake_render(W, H, tiles, tw, th)
    rgb.view(-1, 3)[~torch.from_numpy(tile_pixel_mask(W, H, tw, th, tiles))] = -7.0   # other ranks' pixels: stale
    counts = torch.tensor([tiles.numel()], dtype=torch.int64)
    dist.all_reduce(counts)
    asm = FrameAssembler(W, H, tw, th, world)
    assert sum(asm.n) == W * H
    asm(rgb, rank, dst=0)
    if rank == 0:
        q.put((rgb.numpy().copy(), int(counts.item())))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_tile_sharding_and_assembly_gloo(world):
    W, H, tw, th = 150, 70, 16, 8              # ragged: neither dimension divides the tile size
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, W, H, tw, th, q)) for r in range(world)]
    for p in procs:
        p.start()
    img, count = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert count == n_tiles(W, H, tw, th)
    all_tiles = torch.arange(n_tiles(W, H, tw, th), dtype=torch.int32)
    ref = fake_render(W, H, all_tiles, tw, th).numpy()
    assert np.array_equal(img.view(np.uint32), ref.view(np.uint32))


def test_partition_is_exact_cover_and_balanced():
    for (W, H, tw, th) in [(1920, 1080, 16, 16), (3840, 2160, 16, 16), (37, 23, 8, 4)]:
        for world in (1, 2, 4, 8):
            owner = tile_owner(W, H, tw, th, world)
            nt = n_tiles(W, H, tw, th)
            assert owner.shape == (nt,) and owner.min() >= 0 and owner.max() < world
            per = np.bincount(owner, minlength=world)
            assert per.max() - per.min() <= 1                    # balanced to one tile
            cover = np.zeros(W * H, int)
            for r in range(world):
                cover += tile_pixel_mask(W, H, tw, th, tiles_for_rank(W, H, tw, th, r, world))
            assert np.all(cover == 1)                            # every pixel exactly once
