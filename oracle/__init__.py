"""ctypes wrapper of the CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product package
(paper_2203_11484_b200).  See oracle.c's header for the arithmetic contract.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
SRC = HERE / "oracle.c"
LIB = HERE / "liboracle.so"
LIB_O0 = HERE / "liboracle_o0.so"   # frozen O0 variant (-DORACLE_O0=1): SPEC S:134-150 MT, no fma
VARIANTS = {"default": (LIB, []), "o0": (LIB_O0, ["-DORACLE_O0=1"])}
_default_variant = "default"


def set_default_variant(v: str) -> None:
    """Variant OracleScene uses when none is given (tests parametrise the pins over both)."""
    global _default_variant
    assert v in VARIANTS, v
    _default_variant = v

CFLAGS = ["-O3", "-march=x86-64-v3", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
          "-fPIC", "-shared", "-std=c11", "-Wall", "-Wno-unused-function"]

VPL_DTYPE = np.dtype([("pos", "<f4", 3), ("nrm", "<f4", 3), ("flux", "<f4", 3),
                      ("tri", "<i4"), ("tag", "<i4"), ("depth", "<i4"), ("walk", "<i4")])
GBUF_DTYPE = np.dtype([("pos", "<f4", 3), ("nrm", "<f4", 3), ("alb", "<f4", 3), ("t", "<f4"),
                       ("tri", "<i4"), ("front", "<i4")])

FLAG_EMPTY_NEAR, FLAG_EMPTY_FAR, FLAG_WALK_BUDGET_UNMET = 1, 2, 4


class OParams(C.Structure):
    _fields_ = [("M", C.c_int64), ("K_near", C.c_int64), ("max_depth", C.c_int64), ("rr", C.c_int64),
                ("n_walks_fixed", C.c_int64), ("seed", C.c_uint64)]


class OInfo(C.Structure):
    _fields_ = [("n_near", C.c_int64), ("n_lit", C.c_int64), ("K", C.c_int64), ("M_far", C.c_int64),
                ("n_walks", C.c_int64), ("flags", C.c_int64), ("n_far_tris", C.c_int64),
                ("n_out", C.c_int64)]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


def build(force: bool = False) -> Path:
    for path, defs in VARIANTS.values():
        if force or not path.exists() or path.stat().st_mtime < SRC.stat().st_mtime:
            tmp = path.with_suffix(f".{os.getpid()}.tmp.so")
            subprocess.check_call(["gcc", *CFLAGS, *defs, "-o", str(tmp), str(SRC), "-lm"])
            os.replace(tmp, path)
    return LIB


_libs = {}


def lib(variant: str | None = None):
    variant = variant or "default"
    if variant not in _libs:
        build()
        L = C.CDLL(str(VARIANTS[variant][0]))
        P, I64, F, U8, U32, U64 = C.c_void_p, C.c_int64, C.c_float, C.c_uint8, C.c_uint32, C.c_uint64
        sig = {
            "oracle_philox4x32_10": (None, [P, P, P]),
            "oracle_draw": (U32, [U64, U32, U32, U32]),
            "oracle_scene_new": (P, [P, P, I64, P, C.c_int, P, C.c_int, C.c_int]),
            "oracle_scene_free": (None, [P]),
            "oracle_scene_bad": (I64, [P]),
            "oracle_scene_consts": (None, [P, P, P, P]),
            "oracle_tri_data": (None, [P, P, P, P, P]),
            "oracle_closest_hit": (I64, [P, P, P, F, F, P]),
            "oracle_occluded": (C.c_int, [P, P, P]),
            "oracle_occluded_batch": (None, [P, P, P, I64, P]),
            "oracle_closest_batch": (None, [P, P, P, I64, F, F, P, P]),
            "oracle_classify": (None, [P, C.c_double, P, P]),
            "oracle_lit": (None, [P, P, P]),
            "oracle_morton3": (U32, [U32, U32, U32]),
            "oracle_near_table": (I64, [P, P, P, P, P]),
            "oracle_stratum": (U64, [U64, I64, I64, U64]),
            "oracle_lookup_g": (I64, [P, I64, U64]),
            "oracle_point_in_tri": (None, [P, I64, F, F, P]),
            "oracle_generate_vpls": (I64, [P, P, P, P, I64, P]),
            "oracle_gbuffer": (None, [P, P, I64, P]),
            "oracle_gather": (None, [P, P, I64, P, I64, P, P, P, P, P]),
            "oracle_pair_visibility": (None, [P, P, P, I64, P]),
            "oracle_direct": (None, [P, P, P, I64, C.c_int32, U64, F, P]),
            "oracle_probe_pixels": (None, [C.c_int, C.c_int, U64, P]),
            "oracle_rejection": (I64, [P, P, I64, P, I64, I64, U64, P, P, P, P]),
            "oracle_metropolis": (I64, [P, P, I64, P, I64, I64, I64, I64, I64, U64, P, P, P, P]),
            "oracle_near_strata": (I64, [P, P, P, I64, I64, I64, P]),
            "oracle_walk_range": (None, [P, P, P, I64, I64, P, P]),
            "oracle_abi": (C.c_int, []),
            "oracle_variant": (C.c_int, []),
            "oracle_threads": (C.c_int, []),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        assert L.oracle_variant() == (variant == "o0")
        _libs[variant] = L
    return _libs[variant]


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def philox(ctr, key):
    c = np.asarray(ctr, np.uint32).copy()
    k = np.asarray(key, np.uint32).copy()
    out = np.zeros(4, np.uint32)
    lib().oracle_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def draw(seed, stream, item, j):
    return int(lib().oracle_draw(seed, stream, item, j))


def morton3(qx, qy, qz):
    return int(lib().oracle_morton3(qx, qy, qz))


def stratum(seed, k, K, F):
    return int(lib().oracle_stratum(seed, k, K, F))


def lookup_g(P: np.ndarray, s: int) -> int:
    P = np.ascontiguousarray(P, np.uint64)
    return int(lib().oracle_lookup_g(_p(P), P.size, s))


def threads() -> int:
    return int(lib().oracle_threads())


class OracleScene:
    """Oracle view of a scenegen.Scene (or raw arrays)."""

    def __init__(self, scene, variant: str | None = None):
        self.variant = variant or _default_variant
        self.L = lib(self.variant)
        self.scene = scene
        self._keep = [np.ascontiguousarray(scene.verts, np.float32),
                      np.ascontiguousarray(scene.albedo, np.float32),
                      np.ascontiguousarray(scene.lights, np.float32).reshape(-1, 16),
                      np.ascontiguousarray(scene.cam, np.float32)]
        V, A, Lt, Cm = self._keep
        self.n = V.shape[0]
        self.h = self.L.oracle_scene_new(_p(V), _p(A), self.n, _p(Lt), Lt.shape[0], _p(Cm),
                                        scene.width, scene.height)
        if not self.h:
            raise ValueError("oracle_scene_new failed")

    def __del__(self):
        if getattr(self, "h", None):
            self.L.oracle_scene_free(self.h)
            self.h = None

    # ---- O1 ----
    @property
    def bad(self) -> int:
        return int(self.L.oracle_scene_bad(self.h))

    def consts(self):
        d, e, b = C.c_double(), C.c_float(), C.c_float()
        self.L.oracle_scene_consts(self.h, C.byref(d), C.byref(e), C.byref(b))
        return d.value, np.float32(e.value), np.float32(b.value)

    def tri_data(self):
        n = self.n
        nrm, cen = np.zeros((n, 3), np.float32), np.zeros((n, 3), np.float32)
        area, aq = np.zeros(n, np.float32), np.zeros(n, np.uint64)
        self.L.oracle_tri_data(self.h, _p(nrm), _p(cen), _p(area), _p(aq))
        return dict(normal=nrm, centroid=cen, area=area, aq=aq)

    # ---- O9 ----
    def closest_hit(self, o, d, tmin=0.0, tmax=np.inf):
        o = np.asarray(o, np.float32); d = np.asarray(d, np.float32)
        t = C.c_float()
        i = self.L.oracle_closest_hit(self.h, _p(o), _p(d), tmin, tmax, C.byref(t))
        return int(i), np.float32(t.value)

    def closest_batch(self, o, d, tmin=0.0, tmax=np.inf):
        o = np.ascontiguousarray(o, np.float32).reshape(-1, 3)
        d = np.ascontiguousarray(d, np.float32).reshape(-1, 3)
        idx, t = np.zeros(len(o), np.int64), np.zeros(len(o), np.float32)
        self.L.oracle_closest_batch(self.h, _p(o), _p(d), len(o), tmin, tmax, _p(idx), _p(t))
        return idx, t

    def occluded(self, a, b) -> bool:
        a = np.asarray(a, np.float32); b = np.asarray(b, np.float32)
        return bool(self.L.oracle_occluded(self.h, _p(a), _p(b)))

    def occluded_batch(self, a, b):
        a = np.ascontiguousarray(a, np.float32).reshape(-1, 3)
        b = np.ascontiguousarray(b, np.float32).reshape(-1, 3)
        out = np.zeros(len(a), np.uint8)
        self.L.oracle_occluded_batch(self.h, _p(a), _p(b), len(a), _p(out))
        return out.astype(bool)

    # ---- O2 ----
    def classify(self, T=None):
        T = self.scene.T if T is None else T
        labels = np.zeros(self.n, np.uint8)
        nn = C.c_int64()
        self.L.oracle_classify(self.h, float(T), _p(labels), C.byref(nn))
        return labels, int(nn.value)

    # ---- O3-O5 ----
    def lit(self, labels):
        labels = np.ascontiguousarray(labels, np.uint8)
        out = np.zeros(self.n, np.uint8)
        self.L.oracle_lit(self.h, _p(labels), _p(out))
        return out

    def near_table(self, lit):
        lit = np.ascontiguousarray(lit, np.uint8)
        order, P = np.zeros(self.n, np.int64), np.zeros(self.n, np.uint64)
        codes = np.zeros(self.n, np.uint32)
        m = self.L.oracle_near_table(self.h, _p(lit), _p(order), _p(P), _p(codes))
        return order[:m], P[:m], codes[:m]

    def point_in_tri(self, t, u1, u2):
        out = np.zeros(3, np.float32)
        self.L.oracle_point_in_tri(self.h, int(t), float(u1), float(u2), _p(out))
        return out

    # ---- O3-O11 ----
    def generate_vpls(self, labels, M=None, K_near=None, max_depth=None, rr=None, seed=None,
                      n_walks_fixed=0, max_out=None):
        s = self.scene
        p = OParams(M=s.M if M is None else M, K_near=s.K_near if K_near is None else K_near,
                    max_depth=s.max_depth if max_depth is None else max_depth,
                    rr=s.rr if rr is None else rr, n_walks_fixed=n_walks_fixed,
                    seed=s.seed if seed is None else seed)
        cap = max_out if max_out is not None else max(p.M, 1) + (n_walks_fixed * max(p.max_depth, 1))
        out = np.zeros(cap, VPL_DTYPE)
        info = OInfo()
        labels = np.ascontiguousarray(labels, np.uint8)
        n = self.L.oracle_generate_vpls(self.h, _p(labels), C.byref(p), _p(out), cap, C.byref(info))
        if n < 0:
            raise RuntimeError("oracle_generate_vpls: output capacity too small")
        return out[:n].copy(), info.as_dict()

    def _params(self, **kw):
        s = self.scene
        return OParams(M=kw.get("M", s.M), K_near=kw.get("K_near", s.K_near),
                       max_depth=kw.get("max_depth", s.max_depth), rr=kw.get("rr", s.rr),
                       n_walks_fixed=kw.get("n_walks_fixed", 0), seed=kw.get("seed", s.seed))

    def near_strata(self, labels, K, k0, k1, **kw):
        """near VPLs of strata k0..k1-1 (K = final near count, info['K'])"""
        p = self._params(**kw)
        out = np.zeros(max(k1 - k0, 0), VPL_DTYPE)
        labels = np.ascontiguousarray(labels, np.uint8)
        self.L.oracle_near_strata(self.h, _p(labels), C.byref(p), K, k0, k1, _p(out))
        return out

    def walk_range(self, labels, w0, w1, **kw):
        """raw deposits of walks w0..w1-1 in (w, d) order (flux not divided by the walk count)"""
        p = self._params(**kw)
        md = max(p.max_depth, 1)
        dep = np.zeros((w1 - w0) * md, VPL_DTYPE)
        cnt = np.zeros(w1 - w0, np.int32)
        labels = np.ascontiguousarray(labels, np.uint8)
        self.L.oracle_walk_range(self.h, _p(labels), C.byref(p), w0, w1, _p(dep), _p(cnt))
        return np.concatenate([dep[i * md:i * md + c] for i, c in enumerate(cnt)]) if len(cnt) else dep[:0]

    # ---- O12 ----
    def gbuffer(self, pixels):
        pixels = np.ascontiguousarray(pixels, np.int32)
        out = np.zeros(len(pixels), GBUF_DTYPE)
        self.L.oracle_gbuffer(self.h, _p(pixels), len(pixels), _p(out))
        return out

    # ---- O13 ----
    def gather(self, gb, vpls, bits=False):
        gb = np.ascontiguousarray(gb, GBUF_DTYPE)
        vpls = np.ascontiguousarray(vpls, VPL_DTYPE)
        n, M = len(gb), len(vpls)
        rgb = np.zeros((n, 3), np.float32)
        rgb64 = np.zeros((n, 3), np.float64)
        traced = C.c_int64()
        words = (M + 31) // 32
        tb = np.zeros((n, words), np.uint32) if bits else None
        vb = np.zeros((n, words), np.uint32) if bits else None
        self.L.oracle_gather(self.h, _p(gb), n, _p(vpls), M, _p(rgb), _p(rgb64), C.byref(traced),
                            _p(tb) if bits else None, _p(vb) if bits else None)
        res = dict(rgb=rgb, rgb64=rgb64, traced=int(traced.value))
        if bits:
            res["traced_bits"], res["vis_bits"] = tb, vb
        return res

    # ---- O14 (direct term, reading R21) ----
    def direct(self, gb, pixels, S, seed=None):
        """Direct radiance at the listed pixels' G-buffer points (gb from
        gbuffer(pixels)): S uniform light samples per light per pixel."""
        gb = np.ascontiguousarray(gb, GBUF_DTYPE)
        pixels = np.ascontiguousarray(pixels, np.int32)
        rgb = np.zeros((len(gb), 3), np.float32)
        seed = self.scene.seed if seed is None else seed
        self.L.oracle_direct(self.h, _p(gb), _p(pixels), len(gb), int(S), int(seed), float(np.float32(1.0 / S)),
                            _p(rgb))
        return rgb

    # ---- O15 (rejection-sampling comparator, reading R23) ----
    def probe_pixels(self, seed=None):
        out = np.zeros(64, np.int32)
        s = self.scene
        self.L.oracle_probe_pixels(s.width, s.height, int(s.seed if seed is None else seed), _p(out))
        return out

    def rejection(self, pilot, budget, seed=None, gb=None):
        """Keep up to `budget` of the pilot VPLs by the probe-score rejection
        rule (O15).  gb: explicit probe G-buffer records (default: the 64 probe
        pixels' G-buffer; probes and acceptance draws use `seed`, default the
        scene seed).  Returns (vpls, info {accepted, mean, scores, n_scanned,
        probes})."""
        pilot = np.ascontiguousarray(pilot, VPL_DTYPE)
        seed = self.scene.seed if seed is None else seed
        px = None
        if gb is None:
            px = self.probe_pixels(seed)
            gb = self.gbuffer(px)
        gb = np.ascontiguousarray(gb, GBUF_DTYPE)
        B = min(int(budget), len(pilot))
        out = np.zeros(max(B, 1), VPL_DTYPE)
        sc = np.zeros(max(len(pilot), 1), np.float32)
        mean = C.c_double()
        scanned = C.c_int64()
        acc = self.L.oracle_rejection(self.h, _p(gb), len(gb), _p(pilot), len(pilot), int(budget), int(seed), _p(out),
                                     _p(sc), C.byref(mean), C.byref(scanned))
        return out[:acc], dict(accepted=int(acc), mean=float(mean.value), scores=sc[:len(pilot)],
                               n_scanned=int(scanned.value), probes=px)

    # ---- O16 (Metropolis comparator, reading R24) ----
    def metropolis(self, pilot, chains, per_chain, burn=64, radius=8, seed=None, gb=None):
        """chains x per_chain VPLs from Metropolis chains over the Morton-ordered
        pilot pool (O16).  Returns (vpls, info {scores, pool, accepted})."""
        pilot = np.ascontiguousarray(pilot, VPL_DTYPE)
        seed = self.scene.seed if seed is None else seed
        if gb is None:
            gb = self.gbuffer(self.probe_pixels(seed))
        gb = np.ascontiguousarray(gb, GBUF_DTYPE)
        n = int(chains) * int(per_chain)
        out = np.zeros(max(n, 1), VPL_DTYPE)
        sc = np.zeros(len(pilot), np.float32)
        pool = np.zeros(len(pilot), np.int64)
        acc = C.c_int64()
        self.L.oracle_metropolis(self.h, _p(gb), len(gb), _p(pilot), len(pilot), int(chains), int(per_chain),
                                int(burn), int(radius), int(seed), _p(out), _p(sc), _p(pool), C.byref(acc))
        return out[:n], dict(scores=sc, pool=pool, accepted=int(acc.value))

    def pair_visibility(self, x, y):
        x = np.ascontiguousarray(x, np.float32).reshape(-1, 3)
        y = np.ascontiguousarray(y, np.float32).reshape(-1, 3)
        out = np.zeros(len(x), np.uint8)
        self.L.oracle_pair_visibility(self.h, _p(x), _p(y), len(x), _p(out))
        return out.astype(bool)
