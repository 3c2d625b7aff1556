"""paper_2203_11484_b200 — thin ctypes binding of libvplgi.so, the sm_100a
hybrid-VPL many-light gather (arXiv 2203.11484).  Argument marshalling only:
every step of the path runs in the library's CUDA kernels (include/vplgi.h).
torch is used for device memory and streams.  There is no CPU fallback: a
missing or unloadable library raises ImportError/RuntimeError.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np
import torch

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libvplgi.so"

VPL_OK, VPL_EINVAL, VPL_ESMALL, VPL_ECUDA, VPL_EARCH = 0, -1, -2, -3, -4
FLAG_EMPTY_NEAR, FLAG_EMPTY_FAR, FLAG_WALK_BUDGET_UNMET = 1, 2, 4

# every symbol include/vplgi.h declares (checked by tests/test_abi.py)
EXPORTS = ["vpl_abi_version", "vpl_status_string", "vpl_last_error", "vpl_launch_count", "vpl_device_info", "vpl_scene_bytes",
           "vpl_scene_upload", "vpl_scene_consts", "vpl_scene_tri_data", "vpl_bvh_bytes", "vpl_build_bvh", "vpl_classify_near_far",
           "vpl_generate_bytes", "vpl_generate_vpls", "vpl_render_gbuffer", "vpl_gather_bytes",
           "vpl_gather_indirect", "vpl_render_direct", "vpl_image_error", "vpl_rejection_bytes",
           "vpl_generate_rejection", "vpl_generate_metropolis", "vpl_visibility_dump", "vpl_gather_dump", "vpl_closest_hit_batch", "vpl_occluded_batch",
           "vpl_philox_batch"]


class vpl_light(C.Structure):
    _fields_ = [("corner", C.c_float * 3), ("e_u", C.c_float * 3), ("e_v", C.c_float * 3),
                ("normal", C.c_float * 3), ("area", C.c_float), ("radiance", C.c_float * 3)]


class vpl_camera(C.Structure):
    _fields_ = [("pos", C.c_float * 3), ("fwd", C.c_float * 3), ("up", C.c_float * 3), ("right", C.c_float * 3),
                ("tan_x", C.c_float), ("tan_y", C.c_float), ("width", C.c_int32), ("height", C.c_int32)]


class vpl_gen_params(C.Structure):
    _fields_ = [("M", C.c_int64), ("K_near", C.c_int64), ("max_depth", C.c_int64), ("rr", C.c_int64),
                ("n_walks_fixed", C.c_int64), ("seed", C.c_uint64)]


class vpl_gen_info(C.Structure):
    _fields_ = [("n_near", C.c_int64), ("n_lit", C.c_int64), ("K", C.c_int64), ("M_far", C.c_int64),
                ("n_walks", C.c_int64), ("flags", C.c_int64), ("n_far_tris", C.c_int64), ("n_out", C.c_int64)]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


COUNTER_NAMES = ["pairs", "traced", "visible", "box_tests", "tri_tests", "warp_rays", "warp_steps", "cone_tests",
                 "cone_packets", "ray_packets", "cache_hits", "cache_tests", "cand_lists", "cand_entries", "cand_fails",
                 "filter_steps", "cand_steps", "filter_mt", "filter_mt_hits", "plane_culled"]


class vpl_counters(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in COUNTER_NAMES]


def counters_dict(ctr) -> dict:
    """vpl_counters tensor (int64[len(COUNTER_NAMES)]) -> {name: int}"""
    vals = ctr.tolist() if hasattr(ctr, "tolist") else list(ctr)
    return {k: int(v) for k, v in zip(COUNTER_NAMES, vals)}


VPL_RECORD_BYTES = 48
GPOINT_BYTES = 48

_lib = None


def load_library(path: str | os.PathLike | None = None):
    """Load libvplgi.so (raises if absent — there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    p = Path(path) if path else Path(os.environ.get("VPLGI_LIB", LIB_PATH))   # VPLGI_LIB: tuning variants (tools/)
    if not p.exists():
        raise ImportError(f"libvplgi.so not built at {p}; run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(str(p))
    P, I32, I64, F, D, SZ = C.c_void_p, C.c_int32, C.c_int64, C.c_float, C.c_double, C.c_size_t
    sig = {
        "vpl_abi_version": (I32, []),
        "vpl_status_string": (C.c_char_p, [I32]),
        "vpl_last_error": (C.c_char_p, []),
        "vpl_launch_count": (C.c_uint64, []),
        "vpl_device_info": (I32, [P, P, P]),
        "vpl_scene_bytes": (I32, [I64, I32, P]),
        "vpl_scene_upload": (I32, [P, P, I64, P, I32, P, P, SZ, P, P]),
        "vpl_scene_consts": (I32, [P, P, P, P, P]),
        "vpl_scene_tri_data": (I32, [P, P, P, P, P, P]),
        "vpl_bvh_bytes": (I32, [I64, P, P]),
        "vpl_build_bvh": (I32, [P, P, SZ, P, SZ, P]),
        "vpl_classify_near_far": (I32, [P, D, P, P, P]),
        "vpl_generate_bytes": (I32, [P, I64, I64, P]),
        "vpl_generate_vpls": (I32, [P, P, P, P, P, I64, P, P, SZ, P]),
        "vpl_render_gbuffer": (I32, [P, P, P, I32, I32, I32, P, P]),
        "vpl_gather_bytes": (I32, [I32, I32, I32, P]),
        "vpl_gather_indirect": (I32, [P, P, P, P, I32, P, I32, I32, I32, P, P, P, SZ, P]),
        "vpl_render_direct": (I32, [P, P, P, P, I32, I32, I32, I32, C.c_uint64, I32, P, P]),
        "vpl_image_error": (I32, [P, P, I64, P, P, SZ, P]),
        "vpl_rejection_bytes": (I32, [I64, P]),
        "vpl_generate_metropolis": (I32, [P, P, P, I64, I64, I64, I64, I64, C.c_uint64, P, P, P, P, P, SZ, P]),
        "vpl_generate_rejection": (I32, [P, P, P, I64, I64, C.c_uint64, P, P, P, P, P, P, P, SZ, P]),
        "vpl_visibility_dump": (I32, [P, P, P, P, I32, P, I32, P, P, P]),
        "vpl_gather_dump": (I32, [P, P, P, P, I32, P, I32, I32, I32, P, P, P, SZ, P, P, P, I32, P]),
        "vpl_closest_hit_batch": (I32, [P, P, P, P, I64, F, F, P, P, P]),
        "vpl_occluded_batch": (I32, [P, P, P, P, I64, P, P]),
        "vpl_philox_batch": (I32, [P, I64, P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


class VplError(RuntimeError):
    pass


def _check(st: int, what: str):
    if st != VPL_OK:
        L = load_library()
        raise VplError(f"{what}: {L.vpl_status_string(st).decode()} ({L.vpl_last_error().decode()})")


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _dev(x, dtype, device):
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(x)).to(device=device, dtype=dtype)


# ---------------------------------------------------------------- low-level calls (same names as the C ABI)
def abi_version() -> int:
    return int(load_library().vpl_abi_version())


def launch_count() -> int:
    """kernels launched by libvplgi.so so far (CUB's internal launches excluded)"""
    return int(load_library().vpl_launch_count())


def device_info():
    a, b, c = C.c_int32(), C.c_int32(), C.c_int32()
    _check(load_library().vpl_device_info(C.byref(a), C.byref(b), C.byref(c)), "vpl_device_info")
    return dict(sm_count=a.value, cc=(b.value, c.value))


def make_lights(lights: np.ndarray):
    lights = np.asarray(lights, np.float32).reshape(-1, 16)
    arr = (vpl_light * len(lights))()
    C.memmove(arr, lights.tobytes(), lights.nbytes)
    return arr


def make_camera(cam: np.ndarray, W: int, H: int):
    c = np.asarray(cam, np.float32)
    out = vpl_camera()
    C.memmove(C.addressof(out), c.tobytes(), 14 * 4)
    out.width, out.height = int(W), int(H)
    return out


def scene_upload(verts, albedo, lights, cam, W, H, device="cuda", stream=None):
    """a1: returns (scene blob tensor, device int64 bad-triangle tensor)."""
    L = load_library()
    d_v = _dev(verts, torch.float32, device).reshape(-1)
    d_a = _dev(albedo, torch.float32, device).reshape(-1)
    n = d_v.numel() // 9
    lt = make_lights(lights)
    nbytes = C.c_size_t()
    _check(L.vpl_scene_bytes(n, len(lt), C.byref(nbytes)), "vpl_scene_bytes")
    scene = torch.empty(nbytes.value, dtype=torch.uint8, device=device)
    bad = torch.empty(1, dtype=torch.int64, device=device)
    camst = make_camera(cam, W, H)
    _check(L.vpl_scene_upload(_ptr(d_v), _ptr(d_a), n, lt, len(lt), C.byref(camst), _ptr(scene), nbytes.value,
                              _ptr(bad), _stream(stream)), "vpl_scene_upload")
    return scene, bad, n


def scene_consts(scene, stream=None):
    d, e, b = C.c_double(), C.c_float(), C.c_float()
    _check(load_library().vpl_scene_consts(_ptr(scene), C.byref(d), C.byref(e), C.byref(b), _stream(stream)),
           "vpl_scene_consts")
    return d.value, np.float32(e.value), np.float32(b.value)


def scene_tri_data(scene, n, stream=None):
    dev = scene.device
    nrm = torch.empty(n * 3, dtype=torch.float32, device=dev)
    cen = torch.empty(n * 3, dtype=torch.float32, device=dev)
    area = torch.empty(n, dtype=torch.float32, device=dev)
    aq = torch.empty(n, dtype=torch.int64, device=dev)
    _check(load_library().vpl_scene_tri_data(_ptr(scene), _ptr(nrm), _ptr(cen), _ptr(area), _ptr(aq),
                                             _stream(stream)), "vpl_scene_tri_data")
    return dict(normal=nrm.view(n, 3).cpu().numpy(), centroid=cen.view(n, 3).cpu().numpy(),
                area=area.cpu().numpy(), aq=aq.cpu().numpy().view(np.uint64))


def bvh_bytes(n):
    a, b = C.c_size_t(), C.c_size_t()
    _check(load_library().vpl_bvh_bytes(n, C.byref(a), C.byref(b)), "vpl_bvh_bytes")
    return a.value, b.value


def build_bvh(scene, n, bvh=None, work=None, stream=None):
    nb, wb = bvh_bytes(n)
    dev = scene.device
    bvh = bvh if bvh is not None else torch.empty(nb, dtype=torch.uint8, device=dev)
    work = work if work is not None else torch.empty(wb, dtype=torch.uint8, device=dev)
    _check(load_library().vpl_build_bvh(_ptr(scene), _ptr(bvh), bvh.numel(), _ptr(work), work.numel(),
                                        _stream(stream)), "vpl_build_bvh")
    return bvh, work


def classify_near_far(scene, n, T, labels=None, stream=None):
    dev = scene.device
    labels = labels if labels is not None else torch.empty(n, dtype=torch.uint8, device=dev)
    n_near = torch.zeros(1, dtype=torch.int64, device=dev)
    _check(load_library().vpl_classify_near_far(_ptr(scene), float(T), _ptr(labels), _ptr(n_near),
                                                _stream(stream)), "vpl_classify_near_far")
    return labels, n_near


def generate_bytes(params: vpl_gen_params, n, max_out):
    w = C.c_size_t()
    _check(load_library().vpl_generate_bytes(C.byref(params), n, max_out, C.byref(w)), "vpl_generate_bytes")
    return w.value


def generate_vpls(scene, bvh, labels, n, M, K_near, max_depth, rr, seed, n_walks_fixed=0, max_out=None,
                  vpls=None, work=None, stream=None):
    """a4-a6: returns (vpl tensor uint8 [n_out, 48] view, info dict).  Synchronises."""
    dev = scene.device
    p = vpl_gen_params(M=M, K_near=K_near, max_depth=max_depth, rr=rr, n_walks_fixed=n_walks_fixed, seed=seed)
    if max_out is None:
        max_out = max(M, 1) + n_walks_fixed * max(max_depth, 1)
    wb = generate_bytes(p, n, max_out)
    work = work if work is not None and work.numel() >= wb else torch.empty(wb, dtype=torch.uint8, device=dev)
    vpls = vpls if vpls is not None and vpls.numel() >= max_out * VPL_RECORD_BYTES else \
        torch.empty(max(max_out, 1) * VPL_RECORD_BYTES, dtype=torch.uint8, device=dev)
    info = vpl_gen_info()
    _check(load_library().vpl_generate_vpls(_ptr(scene), _ptr(bvh), _ptr(labels), C.byref(p), _ptr(vpls), max_out,
                                            C.byref(info), _ptr(work), work.numel(), _stream(stream)),
           "vpl_generate_vpls")
    d = info.as_dict()
    return vpls[: d["n_out"] * VPL_RECORD_BYTES].view(-1, VPL_RECORD_BYTES), d, work


def all_tiles(W, H, tw=16, th=16, device="cuda"):
    nt = ((W + tw - 1) // tw) * ((H + th - 1) // th)
    return torch.arange(nt, dtype=torch.int32, device=device)


def render_gbuffer(scene, bvh, tiles, W, H, tw=16, th=16, gbuf=None, stream=None):
    dev = scene.device
    gbuf = gbuf if gbuf is not None else torch.zeros(W * H * GPOINT_BYTES, dtype=torch.uint8, device=dev)
    _check(load_library().vpl_render_gbuffer(_ptr(scene), _ptr(bvh), _ptr(tiles), tiles.numel(), tw, th,
                                             _ptr(gbuf), _stream(stream)), "vpl_render_gbuffer")
    return gbuf


def gather_work(vpls, W, H, device, work=None):
    """The gather's scratch buffer (vpl_gather_bytes) for the VPL tensor `vpls`: `work` if it is large enough,
    else a new tensor."""
    nv = vpls.shape[0] if vpls.dim() == 2 else vpls.numel() // VPL_RECORD_BYTES
    wb = C.c_size_t()
    _check(load_library().vpl_gather_bytes(int(nv), W, H, C.byref(wb)), "vpl_gather_bytes")
    if work is None or work.numel() < wb.value:
        work = torch.empty(wb.value, dtype=torch.uint8, device=device)
    return work


def gather_indirect(scene, bvh, gbuf, vpls, tiles, W, H, tw=16, th=16, rgb=None, counters=False, work=None,
                    stream=None):
    dev = scene.device
    rgb = rgb if rgb is not None else torch.zeros(H * W * 3, dtype=torch.float32, device=dev)
    nv = vpls.shape[0] if vpls.dim() == 2 else vpls.numel() // VPL_RECORD_BYTES
    wb = C.c_size_t()
    _check(load_library().vpl_gather_bytes(nv, W, H, C.byref(wb)), "vpl_gather_bytes")
    if work is None or work.numel() < wb.value:
        work = torch.empty(wb.value, dtype=torch.uint8, device=dev)
    ctr = torch.zeros(len(COUNTER_NAMES), dtype=torch.int64, device=dev) if counters else None
    _check(load_library().vpl_gather_indirect(_ptr(scene), _ptr(bvh), _ptr(gbuf), _ptr(vpls), nv, _ptr(tiles),
                                              tiles.numel(), tw, th, _ptr(rgb), _ptr(ctr), _ptr(work), work.numel(),
                                              _stream(stream)), "vpl_gather_indirect")
    return rgb, ctr


def gather_dump(scene, bvh, gbuf, vpls, tiles, W, H, pixels=None, tw=16, th=16, no_cull=False, stream=None):
    """Test hook: the production gather (vpl_gather_dump, counter build) plus its own traced / visible
    bits for `pixels` (pixel indices, or None for counters only); no_cull=True runs it without the
    VPL-cluster cull and candidate lists.  Returns (rgb, counters, traced_bits, vis_bits), the bit
    arrays uint32 [len(pixels), ceil(M/32)] on the host (bit i = VPL i of `vpls`) or None."""
    dev = scene.device
    rgb = torch.zeros(H * W * 3, dtype=torch.float32, device=dev)
    nv = vpls.shape[0] if vpls.dim() == 2 else vpls.numel() // VPL_RECORD_BYTES
    wb = C.c_size_t()
    _check(load_library().vpl_gather_bytes(nv, W, H, C.byref(wb)), "vpl_gather_bytes")
    work = torch.empty(wb.value, dtype=torch.uint8, device=dev)
    ctr = torch.zeros(len(COUNTER_NAMES), dtype=torch.int64, device=dev)
    words = (nv + 31) // 32
    slot = tb = vb = None
    if pixels is not None:
        px = np.asarray(pixels, np.int64)
        slot = torch.full((H * W,), -1, dtype=torch.int32)
        slot[torch.from_numpy(px)] = torch.arange(len(px), dtype=torch.int32)
        slot = slot.to(dev)
        tb = torch.zeros(len(px) * words, dtype=torch.int32, device=dev)
        vb = torch.zeros(len(px) * words, dtype=torch.int32, device=dev)
    _check(load_library().vpl_gather_dump(_ptr(scene), _ptr(bvh), _ptr(gbuf), _ptr(vpls), nv, _ptr(tiles),
                                          tiles.numel(), tw, th, _ptr(rgb), _ptr(ctr), _ptr(work), work.numel(),
                                          _ptr(slot), _ptr(tb), _ptr(vb), 1 if no_cull else 0, _stream(stream)),
           "vpl_gather_dump")
    torch.cuda.synchronize(dev)
    if pixels is None:
        return rgb, ctr, None, None
    n = len(pixels)
    return (rgb, ctr, tb.cpu().numpy().view(np.uint32).reshape(n, words),
            vb.cpu().numpy().view(np.uint32).reshape(n, words))


def render_direct(scene, bvh, gbuf, tiles, W, H, tw=16, th=16, samples=16, seed=0, rgb=None, accumulate=False,
                  stream=None):
    """NEXT f2: direct term L_e of Eq. 1 for the listed tiles (vpl_render_direct)."""
    dev = scene.device
    rgb = rgb if rgb is not None else torch.zeros(H * W * 3, dtype=torch.float32, device=dev)
    _check(load_library().vpl_render_direct(_ptr(scene), _ptr(bvh), _ptr(gbuf), _ptr(tiles), tiles.numel(), tw, th,
                                            int(samples), int(seed), int(bool(accumulate)), _ptr(rgb),
                                            _stream(stream)), "vpl_render_direct")
    return rgb


def generate_rejection(scene, bvh, pilot, budget, seed, stream=None):
    """NEXT f3: keep up to `budget` pilot VPLs by the probe-score rejection rule
    (vpl_generate_rejection).  Returns (vpls uint8 [n, 48], info {accepted,
    mean, scores, n_scanned, probes}).  Synchronises."""
    dev = scene.device
    pilot = pilot.contiguous().view(-1, VPL_RECORD_BYTES)
    n = pilot.shape[0]
    B = min(int(budget), n)
    wb = C.c_size_t()
    _check(load_library().vpl_rejection_bytes(n, C.byref(wb)), "vpl_rejection_bytes")
    work = torch.empty(max(wb.value, 1), dtype=torch.uint8, device=dev)
    out = torch.empty(max(B, 1) * VPL_RECORD_BYTES, dtype=torch.uint8, device=dev)
    scores = torch.empty(max(n, 1), dtype=torch.float32, device=dev)
    mean = torch.zeros(1, dtype=torch.float64, device=dev)
    acc = torch.zeros(1, dtype=torch.int64, device=dev)
    scanned = torch.zeros(1, dtype=torch.int64, device=dev)
    probes = torch.zeros(64, dtype=torch.int32, device=dev)
    _check(load_library().vpl_generate_rejection(_ptr(scene), _ptr(bvh), _ptr(pilot), n, int(budget), int(seed),
                                                 _ptr(out), _ptr(scores), _ptr(mean), _ptr(acc), _ptr(scanned),
                                                 _ptr(probes), _ptr(work), work.numel(), _stream(stream)),
           "vpl_generate_rejection")
    torch.cuda.synchronize(dev)
    a = int(acc.item())
    return out[: a * VPL_RECORD_BYTES].view(-1, VPL_RECORD_BYTES), dict(
        accepted=a, mean=float(mean.item()), scores=scores[:n], n_scanned=int(scanned.item()), probes=probes)


def generate_metropolis(scene, bvh, pilot, chains, per_chain, burn=64, radius=8, seed=0, stream=None):
    """NEXT f4: chains x per_chain VPLs from Metropolis chains over the pilot
    (vpl_generate_metropolis).  Returns (vpls uint8 [N, 48], info {accepted,
    scores, pool}).  Synchronises."""
    dev = scene.device
    pilot = pilot.contiguous().view(-1, VPL_RECORD_BYTES)
    n = pilot.shape[0]
    N = int(chains) * int(per_chain)
    wb = C.c_size_t()
    _check(load_library().vpl_rejection_bytes(n, C.byref(wb)), "vpl_rejection_bytes")
    work = torch.empty(max(wb.value, 1), dtype=torch.uint8, device=dev)
    out = torch.empty(max(N, 1) * VPL_RECORD_BYTES, dtype=torch.uint8, device=dev)
    scores = torch.empty(max(n, 1), dtype=torch.float32, device=dev)
    pool = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    acc = torch.zeros(1, dtype=torch.int64, device=dev)
    _check(load_library().vpl_generate_metropolis(_ptr(scene), _ptr(bvh), _ptr(pilot), n, int(chains), int(per_chain),
                                                  int(burn), int(radius), int(seed), _ptr(out), _ptr(scores),
                                                  _ptr(pool), _ptr(acc), _ptr(work), work.numel(), _stream(stream)),
           "vpl_generate_metropolis")
    torch.cuda.synchronize(dev)
    return out[: N * VPL_RECORD_BYTES].view(-1, VPL_RECORD_BYTES), dict(accepted=int(acc.item()), scores=scores[:n],
                                                                         pool=pool[:n])


IMAGE_ERROR_WORK_BYTES = 8 * 4 * 592


def image_error(img, ref, stream=None) -> dict:
    """NEXT f1: {rmse, rel_rmse, mae, rel_mae} of img against ref (vpl_image_error)."""
    assert img.numel() == ref.numel() and img.dtype == torch.float32 and ref.dtype == torch.float32
    dev = img.device
    out = torch.zeros(4, dtype=torch.float64, device=dev)
    work = torch.empty(IMAGE_ERROR_WORK_BYTES, dtype=torch.uint8, device=dev)
    _check(load_library().vpl_image_error(_ptr(img), _ptr(ref), img.numel(), _ptr(out), _ptr(work), work.numel(),
                                          _stream(stream)), "vpl_image_error")
    sq, r2, ad, ar = out.cpu().tolist()
    n = max(img.numel(), 1)
    return {"rmse": (sq / n) ** 0.5, "rel_rmse": (sq / r2) ** 0.5 if r2 > 0 else float("nan"),
            "mae": ad / n, "rel_mae": ad / ar if ar > 0 else float("nan"), "sums": [sq, r2, ad, ar]}


def visibility_dump(scene, bvh, gbuf, vpls, pixels, stream=None):
    dev = scene.device
    nv = vpls.shape[0]
    words = (nv + 31) // 32
    px = _dev(pixels, torch.int32, dev)
    tb = torch.zeros(px.numel() * words, dtype=torch.int32, device=dev)
    vb = torch.zeros(px.numel() * words, dtype=torch.int32, device=dev)
    _check(load_library().vpl_visibility_dump(_ptr(scene), _ptr(bvh), _ptr(gbuf), _ptr(vpls), nv, _ptr(px),
                                              px.numel(), _ptr(tb), _ptr(vb), _stream(stream)), "vpl_visibility_dump")
    return tb.view(-1, words), vb.view(-1, words)


def closest_hit_batch(scene, bvh, o, d, tmin=0.0, tmax=float("inf"), stream=None):
    dev = scene.device
    o = _dev(o, torch.float32, dev).reshape(-1)
    d = _dev(d, torch.float32, dev).reshape(-1)
    n = o.numel() // 3
    tri = torch.empty(n, dtype=torch.int32, device=dev)
    t = torch.empty(n, dtype=torch.float32, device=dev)
    _check(load_library().vpl_closest_hit_batch(_ptr(scene), _ptr(bvh), _ptr(o), _ptr(d), n, tmin, tmax, _ptr(tri),
                                                _ptr(t), _stream(stream)), "vpl_closest_hit_batch")
    return tri, t


def occluded_batch(scene, bvh, a, b, stream=None):
    dev = scene.device
    a = _dev(a, torch.float32, dev).reshape(-1)
    b = _dev(b, torch.float32, dev).reshape(-1)
    n = a.numel() // 3
    occ = torch.empty(n, dtype=torch.uint8, device=dev)
    _check(load_library().vpl_occluded_batch(_ptr(scene), _ptr(bvh), _ptr(a), _ptr(b), n, _ptr(occ),
                                             _stream(stream)), "vpl_occluded_batch")
    return occ


def philox_batch(ctr_key: np.ndarray, device="cuda", stream=None):
    x = _dev(np.asarray(ctr_key, np.uint32).view(np.int32), torch.int32, device).reshape(-1)
    n = x.numel() // 6
    out = torch.empty(n * 4, dtype=torch.int32, device=device)
    _check(load_library().vpl_philox_batch(_ptr(x), n, _ptr(out), _stream(stream)), "vpl_philox_batch")
    return out.cpu().numpy().view(np.uint32).reshape(n, 4)


# ---------------------------------------------------------------- record decoding (host side, for tests/bench)
VPL_NP = np.dtype([("pos", "<f4", 3), ("tri", "<i4"), ("nrm", "<f4", 3), ("tag_depth", "<i4"),
                   ("flux", "<f4", 3), ("walk", "<i4")])
GPOINT_NP = np.dtype([("pos", "<f4", 3), ("tri", "<i4"), ("nrm", "<f4", 3), ("front", "<i4"),
                      ("alb", "<f4", 3), ("t", "<f4")])


def decode_vpls(v: torch.Tensor) -> np.ndarray:
    return v.contiguous().cpu().numpy().reshape(-1).view(VPL_NP)


def decode_gbuf(g: torch.Tensor) -> np.ndarray:
    return g.contiguous().cpu().numpy().reshape(-1).view(GPOINT_NP)


# ---------------------------------------------------------------- one frame of the whole path
class Renderer:
    """Runs §8(a) rows a1-a8 for one scenegen.Scene on one GPU (or on a tile
    subset for multi-GPU sharding).  Buffers are torch tensors kept across
    frames; every step is a libvplgi call."""

    def __init__(self, scene, device="cuda", tw=16, th=16, tiles=None):
        self.s = scene
        self.device = torch.device(device)
        self.tw, self.th = tw, th
        self.W, self.H = scene.width, scene.height
        self.tiles = tiles if tiles is not None else all_tiles(self.W, self.H, tw, th, self.device)
        self.n = scene.n_tris
        self.max_out = max(scene.M, 1)
        self._bvh = self._bwork = self._gwork = None
        self._vbuf = torch.empty(self.max_out * VPL_RECORD_BYTES, dtype=torch.uint8, device=self.device)
        self.gbuf = torch.zeros(self.W * self.H * GPOINT_BYTES, dtype=torch.uint8, device=self.device)
        self.rgb = torch.zeros(self.W * self.H * 3, dtype=torch.float32, device=self.device)

    def upload(self, verts=None, albedo=None, stream=None):
        v = self.s.verts if verts is None else verts
        a = self.s.albedo if albedo is None else albedo
        self.scene, self.bad, _ = scene_upload(v, a, self.s.lights, self.s.cam, self.W, self.H, self.device, stream)
        return self.scene

    def frame(self, counters=False, stream=None, upload=True, verts=None, albedo=None):
        if upload:
            self.upload(verts, albedo, stream)
        self.bvh, self._bwork = build_bvh(self.scene, self.n, self._bvh, self._bwork, stream)
        self._bvh = self.bvh
        self.labels, self.n_near = classify_near_far(self.scene, self.n, self.s.T, stream=stream)
        self.vpls, self.info, self._gwork = generate_vpls(
            self.scene, self.bvh, self.labels, self.n, self.s.M, self.s.K_near, self.s.max_depth, self.s.rr,
            self.s.seed, max_out=self.max_out, vpls=self._vbuf, work=self._gwork, stream=stream)
        render_gbuffer(self.scene, self.bvh, self.tiles, self.W, self.H, self.tw, self.th, self.gbuf, stream)
        # one persistent gather scratch buffer per renderer (0.4 GB at C4), not one per call
        self._gawork = gather_work(self.vpls, self.W, self.H, self.device, getattr(self, "_gawork", None))
        self.rgb, self.ctr = gather_indirect(self.scene, self.bvh, self.gbuf, self.vpls, self.tiles, self.W, self.H,
                                             self.tw, self.th, self.rgb, counters, work=self._gawork, stream=stream)
        return self.rgb
