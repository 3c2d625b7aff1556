"""Dump one frame's VPLs and a sample of 8x4 receiver blocks (tools/ analysis only)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2203_11484_b200 as V, scenegen
cfg = int(sys.argv[1]); out = sys.argv[2]
s = scenegen.make_scene(cfg)
r = V.Renderer(s); r.frame(); torch.cuda.synchronize()
g = V.decode_gbuf(r.gbuf).reshape(s.height, s.width)
rng = np.random.default_rng(0)
bx = rng.integers(0, s.width // 8, 2000); by = rng.integers(0, s.height // 4, 2000)
blocks = np.stack([g[y*4:(y+1)*4, x*8:(x+1)*8] for x, y in zip(bx, by)])
np.savez_compressed(out, vpls=V.decode_vpls(r.vpls), blocks=blocks, cam=s.cam)
print("ok", len(V.decode_vpls(r.vpls)))
