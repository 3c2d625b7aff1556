// gather.cuh — the warp-cooperative shadow-ray engine of the a8 gather
// (Eq. 1; DESIGN.md §3 O13 and §5).
//
// A warp owns 32 x kSeg receivers x_j (kSeg = VPL_RECV per lane: one, or the
// two pixels (c, r) and (c, r + 4) of an 8 x 8 block) and walks a chunk of the
// gather's Morton-ordered VPL copy (render.cu) one VPL at a time.  For each
// VPL every lane computes the Eq. 1 cosine terms of its receivers (exact fp32,
// O13), and the shadow segments x_j -> y that need a visibility test are
// resolved together:
//   1. occluder cache: exact MT tests of each receiver's segment against the
//      receiver's two latest occluders, skipped by receivers whose last traced
//      segment was visible;
//   2. one beam {y + s*D : D in Dbox, s in [s_lo, s_hi]} over all pending
//      segments of the warp: a per-run candidate-triangle list (one beam
//      traversal per run of 16 VPLs, then a flat test of the list per VPL) or,
//      when the list is unavailable, a traversal of the 16-wide BVH (lane c of
//      each half-warp tests child c against the beam, two nodes per step, hit
//      inner children on a warp-uniform shared-memory stack); hit triangles are
//      tested by every pending segment with the exact MT of O9;
//   3. loose beams (a D component changes sign, or the spread of D is more
//      than 0.3 of the shortest segment) fall back to per-ray packet traversal
//      of the 4-wide BVH, one packet per receiver slot.
// Every segment's answer equals the exact any-hit of O9: the beams and the
// boxes are conservative (boxes padded at build time) and extra MT tests cannot
// change an any-hit result.
#pragma once
#include "common.cuh"

namespace vplgi {

#ifndef VPL_RECV
#define VPL_RECV 2          // receivers per lane: 8 x 4k pixel blocks share each beam (C4: 1 -> 2: 970 -> 790 ms)
#endif
#ifndef VPL_SMEM_ADDR
#define VPL_SMEM_ADDR 1     // traversal stack accessed through a 32-bit shared-window address held in a register
#endif
#ifndef VPL_CACHE_STREAK
#define VPL_CACHE_STREAK 1  // skip the cache for receivers whose last traced segment was visible (C4: -45% cache MT, -2%)
#endif
#ifndef VPL_CACHE_OWN2
#define VPL_CACHE_OWN2 1    // test the receiver's second most recent occluder
#endif
#ifndef VPL_CANDS
#define VPL_CANDS 1         // per-run candidate-triangle lists
#endif
#ifndef VPL_CAND_CAP
#define VPL_CAND_CAP 128    // list capacity (entries at the top of the warp's stack array); C4: 64 / 128 / 192 / 256 measured, 128 best
#endif
#ifndef VPL_CAND_GROUP
#define VPL_CAND_GROUP 16     // a list covers the next VPL_CAND_GROUP VPLs of the cluster from the first that needs it
                              // (C4: 8 / 12 / 16 / 24 / 32 measured, 16 best)
#endif
#ifndef VPL_CAND_STRADDLE
#define VPL_CAND_STRADDLE 1   // 1: also build lists for beams with straddling axes (extent test; C4 -3%)
#endif
#ifndef VPL_FAST_SEG
#define VPL_FAST_SEG 1   // segment setup by one rsqrt instead of IEEE sqrt + division (C4 -2.8%; reading R28)
#endif
#ifndef VPL_SCAP
#define VPL_SCAP 0.5f   // beam s-range cap at each end, in units of eps / |D|max (O9 tests t in (eps, L - eps))
#endif
constexpr int kSeg = VPL_RECV;
static_assert(kSeg >= 1 && kSeg <= 4, "one to four receivers per lane");
constexpr int kCandCap = VPL_CAND_CAP;
static_assert(kCandCap + 64 <= kWarpStack, "candidate list must leave room for the traversal stack");

// Beam: per axis a, a segment point y + s*D can lie in the slab [lo, hi] only
// for s in [s0, s1] with (D_a > 0)  s0 = (lo - yhi)/Dmax, s1 = (hi - ylo)/Dmin
//                        (D_a < 0)  s0 = (hi - ylo)/Dmin, s1 = (lo - yhi)/Dmax
// (s > 0; y and D range independently over their boxes, a superset of the
// actual segments).  Stored as s0 = N*a0 - b0, s1 = F*a1 - b1 with N/F the
// box face picked by the sign of D_a; evaluated with one FFMA each.  The
// rounding (position error ~ulp(coord)) is absorbed by the box padding.
// beam bounds only (conservative by the box padding, never an O9 operand): one MUFU op each, with
// flush-to-zero (a sub-normal component of D is ~0 against the padding; the plain .approx forms
// expand to ~8 range-scaling instructions)
__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
// L1 prefetch of a triangle's three float4 (48 B, 16-byte aligned: at most two 32-byte sectors apart):
// the lane that finds a box hit issues it, so the serial MT loop that follows finds the data in L1
#ifndef VPL_TRI_PREFETCH
#define VPL_TRI_PREFETCH 0   // measured: C4 753 -> 760 ms, C3 247 -> 251 ms (more L1 requests than the latency they hide)
#endif
__device__ __forceinline__ void prefetch_tri(const float4* tr) {
#if VPL_TRI_PREFETCH
    asm volatile("prefetch.global.L1 [%0];" ::"l"(tr));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(tr + 2));
#endif
}
__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

#ifndef VPL_PLANE_SMEM
#define VPL_PLANE_SMEM 0   // measured: spills 292 -> 268 B but C4 +0.5-2%: off
#endif
struct Beam {
    float a0[3], b0[3], a1[3], b1[3];
    float s_lo, s_hi;
    unsigned pos;   // bit a: D_a > 0
#if !VPL_PLANE_SMEM
    float y[3], dc[3], de[3];   // per-VPL beams: the VPL y, centre / half extent of the D box (plane_cull)
#endif
};
// (VPL_PLANE_SMEM: y, dc, de are uniform and only read at the head of a filter batch, so they live in
// shared memory — 12 floats per warp — instead of 9 registers across the MT loops)
__device__ __forceinline__ float* plane_terms() {
    __shared__ __align__(16) float s_plane[2][12];   // [warp of the CTA (k_visdump runs two)][y dc de, padded]
    return s_plane[(threadIdx.x >> 5) & 1];
}

// Plane-side cull of a candidate triangle before its exact MT tests.  f(p) = n.p - o is the signed
// distance from the triangle's plane (unit normal, BvhView::planes).  For the VPL, a = f(y); for the
// receivers of the pending segments, x = y + D with D in the beam's D box, f(x) in [b_lo, b_hi] =
// a + n.Dc -+ |n|.De.  Both ranges are widened by mu (the scene's box padding, ~100x the fp32 rounding
// of f).  A segment x -> y can only be hit (O9: t in (eps, L - eps)) if it crosses the plane there:
//   * a and every b on the same side: no crossing;
//   * a > 0, some b < 0: the crossing is at t* = L|b| / (|b| + a) <= Lmax|b_lo| / a, below eps/2 when
//     b_lo >= -s a with s = (eps/2) / Lmax (= Beam::s_lo): MT's t (error ~1e-7 |x - v0| / cos, and the
//     condition forces cos >= 2 mu / eps) stays below eps — receivers lying on the triangle's own plane;
//   * every b > 0, a < 0: likewise L - t* <= Lmax|a| / b_lo <= eps/2 — the VPL's own surface;
// and the mirrored cases.  Such a triangle cannot produce an O9 hit for any pending segment, so
// skipping its MT tests leaves every visibility bit unchanged.
#ifndef VPL_PLANE_CULL
#define VPL_PLANE_CULL 1
#endif
#ifndef VPL_PLANE_CULL_FILTER
#define VPL_PLANE_CULL_FILTER 1   // per-VPL cull of list entries before their MT tests
#endif
#ifndef VPL_PLANE_CULL_TRAV
#define VPL_PLANE_CULL_TRAV 0     // per-VPL cull of triangle children in the beam traversal (measured: C4 +26 ms, off)
#endif
__device__ __forceinline__ bool plane_cull(const Beam& B, float mu, float4 pl) {
#if VPL_PLANE_SMEM
    const float4* sp = (const float4*)plane_terms();
    const float4 Y = sp[0], DC = sp[1], DE = sp[2];
    const float a = fmaf(pl.x, Y.x, fmaf(pl.y, Y.y, fmaf(pl.z, Y.z, -pl.w)));
    const float c = fmaf(pl.x, DC.x, fmaf(pl.y, DC.y, pl.z * DC.z));
    const float e = fmaf(fabsf(pl.x), DE.x, fmaf(fabsf(pl.y), DE.y, fmaf(fabsf(pl.z), DE.z, mu + mu)));
#else
    const float a = fmaf(pl.x, B.y[0], fmaf(pl.y, B.y[1], fmaf(pl.z, B.y[2], -pl.w)));
    const float c = fmaf(pl.x, B.dc[0], fmaf(pl.y, B.dc[1], pl.z * B.dc[2]));
    const float e = fmaf(fabsf(pl.x), B.de[0], fmaf(fabsf(pl.y), B.de[1], fmaf(fabsf(pl.z), B.de[2], mu + mu)));
#endif
    const float a_lo = a - mu, a_hi = a + mu;
    const float b_lo = (a + c) - e, b_hi = (a + c) + e;
    const float s = B.s_lo;
    const bool pos = (fmaxf(a_lo, b_lo) > 0.0f) & (fmaf(s, a_lo, b_lo) >= 0.0f) & (fmaf(s, b_lo, a_lo) >= 0.0f);
    const bool neg = (fminf(a_hi, b_hi) < 0.0f) & (fmaf(s, a_hi, b_hi) <= 0.0f) & (fmaf(s, b_hi, a_hi) <= 0.0f);
    return pos | neg;
}
// the same cull for a run beam: y ranges over the run's position box (centre yc, half extent ye),
// x over the participating receivers' box (xc, xe); s = (eps/2) / Lmax of the run beam
#ifndef VPL_PLANE_CULL_RUN
#define VPL_PLANE_CULL_RUN 0   // measured: shorter lists, but the test inside every build step costs more (C4 +47 ms): off
#endif
__device__ __forceinline__ bool plane_cull_run(const float* yc, const float* ye, const float* xc, const float* xe,
                                               float s, float mu, float4 pl) {
    const float ax = fabsf(pl.x), ay = fabsf(pl.y), az = fabsf(pl.z);
    const float a = fmaf(pl.x, yc[0], fmaf(pl.y, yc[1], fmaf(pl.z, yc[2], -pl.w)));
    const float b = fmaf(pl.x, xc[0], fmaf(pl.y, xc[1], fmaf(pl.z, xc[2], -pl.w)));
    const float ea = fmaf(ax, ye[0], fmaf(ay, ye[1], fmaf(az, ye[2], mu)));
    const float eb = fmaf(ax, xe[0], fmaf(ay, xe[1], fmaf(az, xe[2], mu)));
    const float a_lo = a - ea, a_hi = a + ea, b_lo = b - eb, b_hi = b + eb;
    const bool pos = (fmaxf(a_lo, b_lo) > 0.0f) & (fmaf(s, a_lo, b_lo) >= 0.0f) & (fmaf(s, b_lo, a_lo) >= 0.0f);
    const bool neg = (fminf(a_hi, b_hi) < 0.0f) & (fmaf(s, a_hi, b_hi) <= 0.0f) & (fmaf(s, b_hi, a_hi) <= 0.0f);
    return pos | neg;
}

__device__ __forceinline__ bool beam_from_bounds(const float* Dn, const float* Dm, const float* yl, const float* yh,
                                                 float lmin, float lmax, float spread_tol, float eps, Beam& B);

__device__ __forceinline__ bool beam_box(const Beam& B, float4 lo, float4 hi) {
    const bool px = B.pos & 1u, py = B.pos & 2u, pz = B.pos & 4u;
    float s0x = fmaf(px ? lo.x : hi.x, B.a0[0], -B.b0[0]), s1x = fmaf(px ? hi.x : lo.x, B.a1[0], -B.b1[0]);
    float s0y = fmaf(py ? lo.y : hi.y, B.a0[1], -B.b0[1]), s1y = fmaf(py ? hi.y : lo.y, B.a1[1], -B.b1[1]);
    float s0z = fmaf(pz ? lo.z : hi.z, B.a0[2], -B.b0[2]), s1z = fmaf(pz ? hi.z : lo.z, B.a1[2], -B.b1[2]);
    float sn = fmax3(s0x, s0y, fmaxf(s0z, B.s_lo));
    float sf = fmin3(s1x, s1y, fminf(s1z, B.s_hi));
    return sn <= sf;
}

// One lane's shadow segments: segment k runs from receiver o[k] with direction
// d[k] = (y - o[k])/|y - o[k]|, t in (eps, |y - o[k]| - eps)  (O9).
struct Segs {
    f3 o[kSeg], d[kSeg];
    float tmax[kSeg];
    unsigned pend;   // bit k: segment k still unresolved
    unsigned occ;    // bit k: segment k occluded
};

// exact MT (O9) of the segments in `mask` against one triangle (the any-hit form of readings
// R25/R26: division-free, fused products in a fixed order — identical operations to mt_any)
// (k0, k1): the segment slots evaluated (all of them, or the one slot of a receiver's own cache test)
template <bool kCount, int k0 = 0, int k1 = kSeg>
__device__ __forceinline__ unsigned mt_segs(const Segs& S, unsigned mask, float tmin, float4 a, float4 b, float4 c,
                                            TravStats* st) {
    const f3 v0 = xyz(a), e1 = xyz(b), e2 = xyz(c);
    unsigned hit = 0;
#pragma unroll
    for (int k = k0; k < k1; ++k) {
        if (kCount && (mask & (1u << k))) st->tris += 1;
        const f3 s = S.o[k] - v0;
        const f3 q = cross_fma(s, e1);
        const float tq = dot_fma(e2, q);
        const f3 d = S.d[k];
        const f3 pv = cross_fma(d, e2);
        const float det = dot_fma(e1, pv);
        // sign-normalised by det (exact negations)
        const unsigned sg = __float_as_uint(det) & 0x80000000u;
        const float adet = fabsf(det);
        const float u = __uint_as_float(__float_as_uint(dot_fma(s, pv)) ^ sg);
        const float v = __uint_as_float(__float_as_uint(dot_fma(d, q)) ^ sg);
        const float t = __uint_as_float(__float_as_uint(tq) ^ sg);
        // (det = +-0 or NaN: t > tmin*|det| and t < tmax*|det| cannot both hold.  O9's u <= |det|
        // is implied: v >= 0 makes RN(u + v) >= u, so RN(u + v) <= |det| gives u <= |det|; a NaN
        // u or v fails the other tests)
        if ((u >= 0.0f) & (v >= 0.0f) & ((u + v) <= adet) & (t > tmin * adet) & (t < S.tmax[k] * adet))
            hit |= 1u << k;
    }
    return hit & mask;   // no branch around the test: segments not in the mask are dropped here
}

// the occluder that resolved segments `h` goes into their receivers' caches
__device__ __forceinline__ void cache_found(OccluderCache* cache, unsigned h, int tri) {
#pragma unroll
    for (int k = 0; k < kSeg; ++k)
        if (h & (1u << k)) cache[k].found(tri);
}

template <bool kCount, int k0 = 0, int k1 = kSeg>
__device__ __forceinline__ void test_tri(const BvhView& bv, Segs& S, unsigned mask, float tmin, int tri,
                                         OccluderCache* cache, TravStats* st) {
    if (mask) {
        const float4* tr = bv.tris + 3 * tri;
        const unsigned h = mt_segs<kCount, k0, k1>(S, mask, tmin, __ldg(tr), __ldg(tr + 1), __ldg(tr + 2), st);
        if (h) {
            S.occ |= h;
            S.pend &= ~h;
            cache_found(cache, h, tri);
        }
    }
}

// Beam of the pending segments of one VPL y (warp reductions of D = x - y over the pending
// segments).  Returns false if the beam is loose.
__device__ __forceinline__ bool beam_from_bounds(const float* Dn, const float* Dm, const float* yl, const float* yh,
                                                 float lmin, float lmax, float spread_tol, float eps, Beam& B);
__device__ __forceinline__ bool make_beam(const Segs& S, f3 y, float eps, Beam& B) {
    const float inf = __int_as_float(0x7f800000);
    float dn[3] = {inf, inf, inf}, dm[3] = {-inf, -inf, -inf};
    float l2n = inf, l2m = 0.0f;
#pragma unroll
    for (int k = 0; k < kSeg; ++k) {
        if (S.pend & (1u << k)) {
            const f3 D = S.o[k] - y;
            dn[0] = fminf(dn[0], D.x); dm[0] = fmaxf(dm[0], D.x);
            dn[1] = fminf(dn[1], D.y); dm[1] = fmaxf(dm[1], D.y);
            dn[2] = fminf(dn[2], D.z); dm[2] = fmaxf(dm[2], D.z);
            const float l2 = dot(D, D);
            l2n = fminf(l2n, l2); l2m = fmaxf(l2m, l2);
        }
    }
    float Dn[3], Dm[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {   // sm_100a float warp reductions (CREDUX, result in a uniform register)
        Dn[a] = warp_min_f32(dn[a]);
        Dm[a] = warp_max_f32(dm[a]);
    }
    const float lmin = sqrt_approx(warp_min_f32(l2n));
    const float lmax = sqrt_approx(warp_max_f32(l2m));
    const float yv[3] = {y.x, y.y, y.z};
#if VPL_PLANE_SMEM
    if (VPL_PLANE_CULL) {
        float* sp = plane_terms();
        __syncwarp();   // the previous beam's readers are done
        if ((threadIdx.x & 31) < 3) {
            const int a = threadIdx.x & 31;
            const float dn = a == 0 ? Dn[0] : a == 1 ? Dn[1] : Dn[2], dm = a == 0 ? Dm[0] : a == 1 ? Dm[1] : Dm[2];
            sp[a] = a == 0 ? yv[0] : a == 1 ? yv[1] : yv[2];
            sp[4 + a] = 0.5f * (dn + dm);
            sp[8 + a] = 0.5f * (dm - dn) + 2e-7f * fmaxf(fabsf(dn), fabsf(dm));   // |D - Dc| <= De incl. rounding
        }
        __syncwarp();
    }
#else
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        B.y[a] = yv[a];
        B.dc[a] = 0.5f * (Dn[a] + Dm[a]);
        B.de[a] = 0.5f * (Dm[a] - Dn[a]) + 2e-7f * fmaxf(fabsf(Dn[a]), fabsf(Dm[a]));   // |D - Dc| <= De incl. rounding
    }
#endif
    return beam_from_bounds(Dn, Dm, yv, yv, lmin, lmax, kConeSpread, eps, B);
}

// Beam {y + s*D : y in [yl, yh], D in [Dn, Dm], s in [s_lo, s_hi]} from uniform bounds; lmin / lmax
// bound the segment lengths from below / above.  Returns false if the beam is loose.
//
// A "straddling" axis (D changes sign on it: the VPL and the receivers overlap along it) has no
// s-interval; it is encoded in the same two-FFMA slab form as an extent test of the segment points'
// range [L, U] = [yl + Dn, yh + Dm] on that axis (s in [0, 1]):  with N = lo, F = hi and a power of
// two G = 2^21 / 2^e (2^e >= max(|L|, |U|, 1), so L*G and U*G are exact and |.| < 2^21),
//   s0 = lo*G - (U*G + 2)  <= -2 + rounding < 0   whenever lo <= U,
//   s1 = hi*G - (L*G - 2)  >=  2 - rounding > 1   whenever hi >= L,
// i.e. neutral for every box that meets [L, U] (conservative), and s0 > s_hi (or s1 < s_lo) once the
// box misses it by more than 3 / G.
#ifndef VPL_STRADDLE_BEAM
#define VPL_STRADDLE_BEAM 1   // per-VPL beams with straddling axes instead of per-ray packets
#endif
__device__ __forceinline__ void straddle_axis(float L, float U, float& a0, float& b0, float& a1, float& b1) {
    const float m = fmaxf(fmaxf(fabsf(L), fabsf(U)), 1.0f);
    const int e = ((__float_as_int(m) >> 23) & 0xFF) - 126;          // m < 2^e
    const float G = __int_as_float((127 + 21 - e) << 23);              // 2^(21 - e)
    a0 = G; b0 = U * G + 2.0f;
    a1 = G; b1 = L * G - 2.0f;
}
__device__ __forceinline__ bool beam_from_bounds(const float* Dn, const float* Dm, const float* yl, const float* yh,
                                                 float lmin, float lmax, float spread_tol, float eps, Beam& B) {
    const float spread = fmax3(Dm[0] - Dn[0], Dm[1] - Dn[1], Dm[2] - Dn[2]);
    bool tight = spread < spread_tol * lmin;
    B.pos = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const bool p = Dn[a] > 0.0f, n = Dm[a] < 0.0f;
        if (!VPL_STRADDLE_BEAM) tight &= p | n;
        if (p || !n) B.pos |= 1u << a;   // straddling: N = lo, F = hi
        // approximate reciprocals: a0 and b0 = y*a0 share the same a0, so s is scaled by
        // (1 + 2^-22) at most — a position error far below the box padding
        const float rmax = rcp_approx(Dm[a]), rmin = rcp_approx(Dn[a]);
        B.a0[a] = p ? rmax : rmin;
        B.b0[a] = (p ? yh[a] : yl[a]) * B.a0[a];
        B.a1[a] = p ? rmin : rmax;
        B.b1[a] = (p ? yl[a] : yh[a]) * B.a1[a];
        if (VPL_STRADDLE_BEAM && !p && !n)
            straddle_axis(yl[a] + Dn[a], yh[a] + Dm[a], B.a0[a], B.b0[a], B.a1[a], B.b1[a]);
    }
    // segment (x_j, y_k) tests t in (eps, L - eps): s = 1 - t/L in (eps/L, 1 - eps/L) within
    // [eps/Lmax, 1 - eps/Lmax]; half the cap is cut (the rest is slack for MT's rounding of t)
    B.s_lo = (VPL_SCAP * eps) * rcp_approx(lmax);   // relative error ~1e-6: far inside the factor
    B.s_hi = 1.0f - B.s_lo;
    return tight;
}

// Beam of a whole VPL cluster: every segment from a participating receiver x_j to any point of the
// cluster's position box [ylo, yhi] (a superset of the segments to the cluster's VPLs).  An axis on
// which D changes sign ("straddling": the cluster and the receivers overlap along it) gives no
// s-interval; its slab factor is made neutral (a0 = 0, b0 = +inf -> s0 = -inf; likewise s1 = +inf)
// and replaced by the extent test lo <= U, hi >= L with [L, U] = [yl + Dn, yh + Dm] the range of the
// segment points on that axis (s in [0, 1]).  Returns false only if every axis straddles.
struct ClusterBeam {
    Beam B;
    float L[3], U[3];
};
// xl / xh: the box of the participating receivers (warp reductions); D = x - y over the two boxes is
// [xl - yh, xh - yl] (fp32 subtraction is monotonic in each operand, so every lane's rounded D is inside).
__device__ __forceinline__ bool make_cluster_beam(const float* xl, const float* xh, float4 ylo, float4 yhi, float eps,
                                                  ClusterBeam& C) {
    const float inf = __int_as_float(0x7f800000);
    const float yl[3] = {ylo.x, ylo.y, ylo.z}, yh[3] = {yhi.x, yhi.y, yhi.z};
    float Dn[3], Dm[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) { Dn[a] = xl[a] - yh[a]; Dm[a] = xh[a] - yl[a]; }
    float l2n = 0.0f, l2m = 0.0f;
#pragma unroll
    for (int a = 0; a < 3; ++a) {   // |D| over the box: per axis the nearer / farther face
        const float n2 = Dn[a] * Dn[a], m2 = Dm[a] * Dm[a];
        l2n += Dn[a] > 0.0f ? n2 : (Dm[a] < 0.0f ? m2 : 0.0f);
        l2m += fmaxf(n2, m2);
    }
    beam_from_bounds(Dn, Dm, yl, yh, sqrt_approx(l2n), sqrt_approx(l2m), inf, eps, C.B);
    int straddle = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const bool sa = !(Dn[a] > 0.0f) && !(Dm[a] < 0.0f);
        C.L[a] = sa && !VPL_STRADDLE_BEAM ? yl[a] + Dn[a] : -inf;
        C.U[a] = sa && !VPL_STRADDLE_BEAM ? yh[a] + Dm[a] : inf;
        if (sa) ++straddle;
        if (sa && !VPL_STRADDLE_BEAM) {   // (VPL_STRADDLE_BEAM: beam_from_bounds encoded the extent test)
            C.B.pos |= 1u << a;   // N = lo, F = hi
            C.B.a0[a] = 0.0f; C.B.b0[a] = inf;
            C.B.a1[a] = 0.0f; C.B.b1[a] = -inf;
        }
    }
    return VPL_CAND_STRADDLE ? straddle < 3 : straddle == 0;
}
__device__ __forceinline__ bool cluster_beam_box(const ClusterBeam& C, float4 lo, float4 hi) {
    if (VPL_STRADDLE_BEAM) return beam_box(C.B, lo, hi);
    const bool ext = (lo.x <= C.U[0]) & (lo.y <= C.U[1]) & (lo.z <= C.U[2]) & (hi.x >= C.L[0]) &
                     (hi.y >= C.L[1]) & (hi.z >= C.L[2]);
    return ext & beam_box(C.B, lo, hi);
}

// beam traversal (two nodes per step); returns when every pending segment is resolved or the tree
// is exhausted
template <bool kCount>
__device__ __forceinline__ void beam_traverse(const BvhView& bv, Segs& S, float tmin, const Beam& B,
                                              OccluderCache* cache, int* __restrict__ sstack, TravStats* st) {
    const int lane = threadIdx.x & 31;
    const int half = lane >> 4;
    const unsigned below = (1u << lane) - 1u;
    const unsigned hmask = half ? 0xFFFF0000u : 0x0000FFFFu;
    const unsigned dir_neg = B.pos;
    if (bv.root < 0) {  // single-triangle scene
        test_tri<kCount>(bv, S, S.pend, tmin, 0, cache, st);
        return;
    }
    // the stack holds inner nodes only
    if (lane == 0) sstack[0] = bv.root;
    __syncwarp();
    int sp = 1;
#if VPL_SMEM_ADDR
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(sstack);   // 32-bit shared-window address
#endif
    // each step pops the top two (lanes 0-15 take the top one)
    while (sp > 0) {
        const int idx = sp - 1 - half;
#if VPL_SMEM_ADDR
        int node = -1;
        if (idx >= 0) asm volatile("ld.shared.s32 %0, [%1];" : "=r"(node) : "r"(sbase + 4u * (unsigned)idx));
#else
        const int node = idx >= 0 ? sstack[idx] : -1;
#endif
        if (kCount && lane == 0) st->wsteps += 1;
        sp = max(sp - 2, 0);
        // no branch: an empty half-step loads the root's children (cached) and masks the result
        const int nsafe = node >= 0 ? node : 0;
        VPL_DCHECK(nsafe < (bv.n > 1 ? bv.n - 1 : 1));
        const float4* nd = (const float4*)((const char*)bv.wide + ((size_t)nsafe << 9) + ((lane & (kWide - 1)) << 5));
        const float4 lo = __ldg(nd), hi = __ldg(nd + 1);
        int ref = node >= 0 ? __float_as_int(lo.w) : INT_MIN;
        const int axis = __float_as_int(hi.w);
        const bool hit = (ref != INT_MIN) & beam_box(B, lo, hi);
        if (kCount) {   // beam tests of real children only (empty slots are not algorithmic work)
            const unsigned real = __ballot_sync(0xFFFFFFFFu, ref != INT_MIN);
            if (lane == 0) st->cones += __popc(real);
        }
        const unsigned Bi = __ballot_sync(0xFFFFFFFFu, hit && ref >= 0);
        bool leaf = hit && ref < 0;
        if (VPL_PLANE_CULL && VPL_PLANE_CULL_TRAV && bv.planes && leaf) {
            const bool cull = plane_cull(B, bv.box_pad, __ldg(bv.planes + (~ref >> 3)));
            if (kCount && cull) st->pculled += 1;
            leaf = !cull;
        }
        if (leaf) prefetch_tri(bv.tris + 3 * (~ref >> 3));
        unsigned Bl = __ballot_sync(0xFFFFFFFFu, leaf);
        if (Bi) {
            const int nB = __popc(Bi >> 16), nA = __popc(Bi & 0xFFFFu);
            const int rank = __popc(Bi & below & hmask);
            const int nh = half ? nB : nA;
            const bool rev = (dir_neg >> axis) & 1u;   // segments run x -> y along -axis: visit descending
            const int pos = (half ? 0 : nB) + (rev ? rank : nh - 1 - rank);   // first to visit ends on top
#if VPL_SMEM_ADDR
            if (hit && ref >= 0)
                asm volatile("st.shared.s32 [%0], %1;" ::"r"(sbase + 4u * (unsigned)(sp + pos)), "r"(ref) : "memory");
#else
            if (hit && ref >= 0) sstack[sp + pos] = ref;
#endif
            sp += nA + nB;
            VPL_DCHECK(sp <= kWarpStack - kCandCap);   // a live candidate list occupies the top kCandCap
        }
        __syncwarp();
        while (Bl) {   // hit triangle children
            const int k = __ffs(Bl) - 1;
            Bl &= Bl - 1u;
            const int tri = ~__shfl_sync(0xFFFFFFFFu, ref, k) >> 3;
            VPL_DCHECK(tri >= 0 && tri < bv.n);
            const float4* tr = bv.tris + 3 * tri;
            const unsigned h = mt_segs<kCount>(S, S.pend, tmin, __ldg(tr), __ldg(tr + 1), __ldg(tr + 2), st);
            S.occ |= h;
            S.pend &= ~h;
            if (h) cache_found(cache, h, tri);
            if (!__any_sync(0xFFFFFFFFu, S.pend != 0)) return;
        }
    }
}

// Candidate list of a run of VPLs: one beam traversal of the 16-wide BVH with
// the run beam (make_cluster_beam: the participating receivers' box [xl, xh]
// to the run's position box) that records every triangle child whose box the
// beam reaches — no MT tests, no early exit, children pushed in lane order.
// Any triangle that can block a segment of the run is in the list (the same
// conservative beam / padded box argument as beam_traverse), so each VPL of
// the run then tests only the list (filter_cands).  The list holds 16-wide
// child slots (node * 16 + child) at the top of the warp's stack array;
// returns its length, or -1 if every axis straddles, the list overflows
// kCandCap or the stack meets the list.
#ifndef VPL_CAND_NOINLINE
#define VPL_CAND_NOINLINE 1   // keep the (rare) list build out of the hot loop's register allocation
#endif
template <bool kCount>
#if VPL_CAND_NOINLINE
__device__ __noinline__
#else
__device__ __forceinline__
#endif
int build_cands(const BvhView& bv, const float* xl, const float* xh, const vpl_record* __restrict__ vg, int ng,
                float eps, int* __restrict__ sstack, TravStats* st) {
    const int lane = threadIdx.x & 31;
    if (bv.root < 0) return -1;
    const float inf = __int_as_float(0x7f800000);
    // position box of the run vg[0..ng) (lane l loads VPL l)
    float4 ylo = make_float4(inf, inf, inf, 0.0f), yhi = make_float4(-inf, -inf, -inf, 0.0f);
    if (lane < ng) { const float4 p = __ldg((const float4*)(vg + lane)); ylo = p; yhi = p; }
    ylo.x = warp_min_f32(ylo.x); ylo.y = warp_min_f32(ylo.y); ylo.z = warp_min_f32(ylo.z);
    yhi.x = warp_max_f32(yhi.x); yhi.y = warp_max_f32(yhi.y); yhi.z = warp_max_f32(yhi.z);
    ClusterBeam CB;
    if (!make_cluster_beam(xl, xh, ylo, yhi, eps, CB)) return -1;
    // centre / half extent of the run box and the receivers' box (half extents rounded up)
    const float yc[3] = {0.5f * (ylo.x + yhi.x), 0.5f * (ylo.y + yhi.y), 0.5f * (ylo.z + yhi.z)};
    const float xc[3] = {0.5f * (xl[0] + xh[0]), 0.5f * (xl[1] + xh[1]), 0.5f * (xl[2] + xh[2])};
    const float ye[3] = {fmaxf(yhi.x - yc[0], yc[0] - ylo.x) * 1.000001f, fmaxf(yhi.y - yc[1], yc[1] - ylo.y) * 1.000001f,
                         fmaxf(yhi.z - yc[2], yc[2] - ylo.z) * 1.000001f};
    const float xe[3] = {fmaxf(xh[0] - xc[0], xc[0] - xl[0]) * 1.000001f, fmaxf(xh[1] - xc[1], xc[1] - xl[1]) * 1.000001f,
                         fmaxf(xh[2] - xc[2], xc[2] - xl[2]) * 1.000001f};
    const int half = lane >> 4;
    const unsigned below = (1u << lane) - 1u;
    if (lane == 0) sstack[0] = bv.root;
    __syncwarp();
    int sp = 1, n = 0;
    while (sp > 0) {
        const int idx = sp - 1 - half;
        const int node = idx >= 0 ? sstack[idx] : -1;
        if (kCount && lane == 0) { st->wsteps += 1; st->lsteps += 1; }
        sp = max(sp - 2, 0);
        const int nsafe = node >= 0 ? node : 0;
        const int slot = (nsafe << 4) + (lane & (kWide - 1));
        const float4* nd = (const float4*)((const char*)bv.wide + ((size_t)slot << 5));
        const float4 lo = __ldg(nd), hi = __ldg(nd + 1);
        const int ref = node >= 0 ? __float_as_int(lo.w) : INT_MIN;
        const bool hit = (ref != INT_MIN) & cluster_beam_box(CB, lo, hi);
        if (kCount) {
            const unsigned real = __ballot_sync(0xFFFFFFFFu, ref != INT_MIN);
            if (lane == 0) st->cones += __popc(real);
        }
        const unsigned Bi = __ballot_sync(0xFFFFFFFFu, hit && ref >= 0);
        bool leaf = hit && ref < 0;
        if (VPL_PLANE_CULL && VPL_PLANE_CULL_RUN && bv.planes && leaf)
            leaf = !plane_cull_run(yc, ye, xc, xe, CB.B.s_lo, bv.box_pad, __ldg(bv.planes + (~ref >> 3)));
        const unsigned Bl = __ballot_sync(0xFFFFFFFFu, leaf);
        __syncwarp();
        if (Bl) {
            const int nl = __popc(Bl);
            if (n + nl > kCandCap) return -1;
            if (leaf) sstack[kWarpStack - 1 - (n + __popc(Bl & below))] = slot;
            n += nl;
        }
        if (Bi) {
            const int ni = __popc(Bi);
            if (sp + ni > kWarpStack - kCandCap) return -1;
            if (hit && ref >= 0) sstack[sp + __popc(Bi & below)] = ref;   // collection order does not matter
            sp += ni;
        }
        __syncwarp();
    }
    return n;
}

// The pending segments of one VPL against its run's candidate list: lane c
// tests candidate c of each batch of 32 against the VPL's own beam; hit
// triangles get the exact MT of O9 from every pending segment, highest lane first.
template <bool kCount>
__device__ __forceinline__ void filter_cands(const BvhView& bv, Segs& S, float tmin, const Beam& B,
                                             const int* __restrict__ sstack, int ncand, OccluderCache* cache,
                                             TravStats* st) {
    const int lane = threadIdx.x & 31;
    for (int base = 0; base < ncand; base += 32) {
        const int i = base + lane;
        const bool ok = i < ncand;
        const int slot = ok ? sstack[kWarpStack - 1 - i] : 0;   // slot 0: a real child, masked below
        const float4* nd = (const float4*)((const char*)bv.wide + ((size_t)slot << 5));
        const float4 lo = __ldg(nd), hi = __ldg(nd + 1);
        bool hit = ok & beam_box(B, lo, hi);
        if (kCount && lane == 0) { st->fsteps += 1; st->cones += min(32, ncand - base); }
        const int tri = ok ? ~__float_as_int(lo.w) >> 3 : 0;
        if (VPL_PLANE_CULL && VPL_PLANE_CULL_FILTER && bv.planes) {
            const bool cull = plane_cull(B, bv.box_pad, __ldg(bv.planes + tri));
            if (kCount && hit && cull) st->pculled += 1;
            hit &= !cull;
        }
        unsigned Bl = __ballot_sync(0xFFFFFFFFu, hit);
        const int toff = 3 * tri;   // float4 offset of the candidate's triangle
        if (hit) prefetch_tri(bv.tris + toff);
        while (Bl) {
            const int k = 31 - __clz(Bl);                      // highest first: one FLO
            Bl &= ~(1u << k);
            const int to = __shfl_sync(0xFFFFFFFFu, toff, k);
            VPL_DCHECK(to >= 0 && to < 3 * bv.n);
            const float4* tr = bv.tris + to;
            const unsigned h = mt_segs<kCount>(S, S.pend, tmin, __ldg(tr), __ldg(tr + 1), __ldg(tr + 2), st);
            if (kCount) {   // warp-level MT tests of the filter, and those that found an occluder
                const bool any = __any_sync(0xFFFFFFFFu, h != 0);
                if (lane == 0) { st->fmt += 1; st->fmt_hit += any; }
            }
            S.occ |= h;
            S.pend &= ~h;
            if (h) cache_found(cache, h, to / 3);
            if (!__any_sync(0xFFFFFFFFu, S.pend != 0)) return;
        }
    }
}

// Per-ray packet of one receiver slot (loose beams, ~1% of the packets): kept out of line so that its
// code is not duplicated per slot inside the hot loop (instruction-cache footprint).  Returns the
// occluding triangle of this lane's segment, or -1.
#ifndef VPL_RAY_NOINLINE
#define VPL_RAY_NOINLINE 0   // measured: C3 -1.6%, C4 +1.8%
#endif
template <bool kCount>
#if VPL_RAY_NOINLINE
__device__ __noinline__
#else
__device__ __forceinline__
#endif
int ray_packet(const BvhView& bv, f3 o, f3 d, float eps, float tmax, bool live, int* __restrict__ sstack,
               TravStats* st) {
    Ray r;
    r.o = o; r.d = d; r.tmin = eps; r.tmax = tmax;
    const unsigned lm = __ballot_sync(0xFFFFFFFFu, live);
    const int leader = __ffs(lm) - 1;
    const unsigned neg = (d.x < 0.0f ? 1u : 0u) | (d.y < 0.0f ? 2u : 0u) | (d.z < 0.0f ? 4u : 0u);
    const unsigned dn = __shfl_sync(0xFFFFFFFFu, neg, leader);
    OccluderCache c;
    const bool occ = warp_traverse_ray<kCount>(bv, r, live, false, c, dn, sstack, st);
    return occ && live ? c.own0 : -1;
}

#ifndef VPL_LIST_FIRST
#define VPL_LIST_FIRST 1   // 1: the run list is looked up before the VPL's beam is made (an empty list needs no beam; a list
                           // also serves loose beams); 0: beam first, lists only for tight beams
#endif
// Resolve the pending segments of one VPL y: the run's candidate list or a beam traversal, else
// (loose beam) one per-ray packet per receiver slot.  part: bit k set if receiver k may trace the
// current VPL cluster (render.cu's conservative cluster cull); xl / xh of the run beam are the box of
// those receivers.
template <bool kCount>
__device__ __forceinline__ void resolve(const BvhView& bv, Segs& S, float eps, f3 y, OccluderCache* cache,
                                        int* __restrict__ sstack, TravStats* st, int& cand, int& cand_end, int cend,
                                        unsigned part, const f3* xr, const vpl_record* __restrict__ vpls, int i) {
    const int lane = threadIdx.x & 31;
    if (!__any_sync(0xFFFFFFFFu, S.pend != 0)) return;
    if (kCount && lane == 0) st->wrays += 1;
    Beam B;
    // the run list covers the participating receivers only (the cluster cull is conservative, so a
    // pending segment always belongs to one; checked anyway)
    const bool covered = !__any_sync(0xFFFFFFFFu, (S.pend & ~part) != 0);
#if !VPL_LIST_FIRST
    bool tight = make_beam(S, y, eps, B);
    if (VPL_CANDS && tight && i >= cand_end) {
#else
    bool tight = false;
    if (VPL_CANDS && i >= cand_end) {
#endif
        const float inf = __int_as_float(0x7f800000);
        float l[3] = {inf, inf, inf}, h[3] = {-inf, -inf, -inf};
#pragma unroll
        for (int k = 0; k < kSeg; ++k)
            if (part & (1u << k)) {
                l[0] = fminf(l[0], xr[k].x); l[1] = fminf(l[1], xr[k].y); l[2] = fminf(l[2], xr[k].z);
                h[0] = fmaxf(h[0], xr[k].x); h[1] = fmaxf(h[1], xr[k].y); h[2] = fmaxf(h[2], xr[k].z);
            }
        const float xl[3] = {warp_min_f32(l[0]), warp_min_f32(l[1]), warp_min_f32(l[2])};
        const float xh[3] = {warp_max_f32(h[0]), warp_max_f32(h[1]), warp_max_f32(h[2])};
        cand_end = min(i + VPL_CAND_GROUP, cend);
        cand = build_cands<kCount>(bv, xl, xh, vpls + i, cand_end - i, eps, sstack, st);
        if (kCount && lane == 0) { if (cand >= 0) { st->lists += 1; st->entries += cand; } else st->lfail += 1; }
    }
    const bool listed = VPL_CANDS && covered && cand >= 0;
#if VPL_LIST_FIRST
    if (listed && cand == 0) {   // nothing can block a segment of this run: every pending segment is visible
        if (kCount && lane == 0) st->cpk += 1;
        S.pend = 0;
        return;
    }
    // (a list serves loose beams too: it holds every possible occluder of the run's segments)
    tight = make_beam(S, y, eps, B) || listed;
#endif
    if (tight) {
        if (kCount && lane == 0) st->cpk += 1;
        if (listed)
            filter_cands<kCount>(bv, S, eps, B, sstack, cand, cache, st);
        else
            beam_traverse<kCount>(bv, S, eps, B, cache, sstack, st);
    } else {
        // loose: per-ray packet traversal of the 4-wide BVH, one packet per receiver slot
#pragma unroll
        for (int k = 0; k < kSeg; ++k) {
            const bool live = (S.pend >> k) & 1u;
            const unsigned lm = __ballot_sync(0xFFFFFFFFu, live);
            if (!lm) continue;                                          // uniform
            if (kCount && lane == 0) st->rpk += 1;
            const int tri = ray_packet<kCount>(bv, S.o[k], S.d[k], eps, S.tmax[k], live, sstack, st);
            if (tri >= 0) { S.occ |= 1u << k; cache[k].found(tri); }
        }
    }
    S.pend = 0;
}

// receiver k's segment against its own recent occluders (only slot k's MT is evaluated)
template <bool kCount, int k>
__device__ __forceinline__ void cache_tests(const BvhView& bv, Segs& S, float eps, OccluderCache* cache,
                                            TravStats* st) {
    const unsigned bit = 1u << k;
#if VPL_CACHE_STREAK
    const unsigned m = cache[k].vis_streak ? 0u : (S.pend & bit);
#else
    const unsigned m = S.pend & bit;
#endif
    if (m && cache[k].own0 >= 0) test_tri<kCount, k, k + 1>(bv, S, m, eps, cache[k].own0, cache, st);
    if (VPL_CACHE_OWN2 && (S.pend & m) && cache[k].own1 >= 0)
        test_tri<kCount, k, k + 1>(bv, S, S.pend & m, eps, cache[k].own1, cache, st);
}

// One VPL (position y, triangle yt; uniform) for one lane's receivers: Eq. 1 terms (O13, exact fp32
// order), segment setup (O9), occluder caches, resolution — in two functions.  `shade` (inlined in the
// kernel's VPL loop) evaluates the two cosine tests; only if some receiver of the warp traces the VPL it
// calls `shade_heavy`: segment setup, cache tests, lists, filter, traversals, MT.  The state only the
// heavy part touches (occluder caches, candidate-list cursor, the weights) is grouped in a HeavyState.
// (VPL_HEAVY_NOINLINE = 1 compiles shade_heavy out of line, with a register allocation of its own and
// the HeavyState in local memory: measured, slower — see the knob.)
#ifndef VPL_HEAVY_NOINLINE
#define VPL_HEAVY_NOINLINE 0   // measured at 1: ptxas then keeps every value that lives across the call in local memory
                               // (17 reloads per VPL in the light loop instead of 11) and the call itself costs: C4 652 ->
                               // 870 ms, C3 220 -> 286 ms.  0: inlined (the HeavyState is then scalarised into registers).
#endif
struct HeavyState {
    OccluderCache cache[kSeg];
    float w[kSeg];        // in: cx * ci of the traced receivers; out: w = cx*ci / (r2 * max(r2, b2))
    int cand, cand_end;   // the run's candidate list (length or -1) and the VPL index its run ends at
    float eps, b2;
};
struct RecvPos { f3 x[kSeg]; };

template <bool kCount>
#if VPL_HEAVY_NOINLINE
__device__ __noinline__
#else
__device__ __forceinline__
#endif
unsigned shade_heavy(const BvhView& bv, const vpl_record* __restrict__ vpls, int i, f3 y, RecvPos X, unsigned traced,
                     int cend, unsigned part, HeavyState* __restrict__ hs, int* __restrict__ sstack, TravStats* st) {
    const float eps = hs->eps, b2 = hs->b2;
    const f3* xr = X.x;
    OccluderCache cache[kSeg];
    float w[kSeg];
#pragma unroll
    for (int k = 0; k < kSeg; ++k) { cache[k] = hs->cache[k]; w[k] = hs->w[k]; }
    int cand = hs->cand, cand_end = hs->cand_end;
    // Eq. 1 weight and segment setup of the traced receivers
    Segs S;
    S.pend = 0; S.occ = 0;
#pragma unroll
    for (int k = 0; k < kSeg; ++k) {
        S.o[k] = xr[k];
        S.d[k] = mk3(0.0f, 0.0f, 0.0f);
        S.tmax[k] = 0.0f;
        if (traced & (1u << k)) {
            const f3 d = y - xr[k];
            const float r2 = dot(d, d);
            w[k] = w[k] * rcp_approx(r2 * fmaxf(r2, b2));   // (cx * ci) / ...; r2 * max(r2, b2) >= b2^2: normal range
#if VPL_FAST_SEG
            // one MUFU: 1/dist and dist within ~2 ulp of O9's IEEE sqrt / division (visibility then
            // differs from the oracle only for grazing hits, inside BJ:5's 1e-4 budget; reading R28)
            float inv;
            asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(r2));
            const float dist = r2 * inv;
#else
            const float dist = sqrtf(r2);   // = sqrtf(dot(d, d)) of O9's segment setup
            const float inv = 1.0f / dist;  // R25: dir = d * (1/dist)
#endif
            S.d[k] = mk3(d.x * inv, d.y * inv, d.z * inv);
            S.tmax[k] = dist - eps;
            if (S.tmax[k] > eps) S.pend |= 1u << k;
        }
    }
    // occluder caches: exact MT of each receiver's segment against its recent occluders; a receiver
    // whose last traced segment was visible skips its cache (visibility is coherent along the
    // spatially ordered VPLs)
    const uint32_t t0 = kCount ? st->tris : 0;
    cache_tests<kCount, 0>(bv, S, eps, cache, st);
    if (kSeg > 1) cache_tests<kCount, (kSeg > 1 ? 1 : 0)>(bv, S, eps, cache, st);
    if (kSeg > 2) cache_tests<kCount, (kSeg > 2 ? 2 : 0)>(bv, S, eps, cache, st);
    if (kSeg > 3) cache_tests<kCount, (kSeg > 3 ? 3 : 0)>(bv, S, eps, cache, st);
    if (kCount) { st->chits += __popc(S.occ); st->ctests += st->tris - t0; }
    resolve<kCount>(bv, S, eps, y, cache, sstack, st, cand, cand_end, cend, part, xr, vpls, i);
    const unsigned vis = traced & ~S.occ;
#if VPL_CACHE_STREAK
#pragma unroll
    for (int k = 0; k < kSeg; ++k)
        if (traced & (1u << k)) cache[k].vis_streak = (vis >> k) & 1u;
#endif
#pragma unroll
    for (int k = 0; k < kSeg; ++k) { hs->cache[k] = cache[k]; hs->w[k] = w[k]; }
    hs->cand = cand; hs->cand_end = cand_end;
    return traced | vis << 16;
}

// act: bit k = receiver k is a front-face hit; nb: the VPL's normal record.  Returns traced | vis << 16
// (bit k per receiver); the weights of the visible receivers are in hs->w.
template <bool kCount>
__device__ __forceinline__ unsigned shade(const BvhView& bv, const vpl_record* __restrict__ vpls, int i, f3 y, int yt,
                                          float4 nb, const f3* xr, const f3* nr, const int* tri_x, unsigned act,
                                          HeavyState* hs, int* __restrict__ sstack, TravStats* st, int cend,
                                          unsigned part) {
    // the cosine tests only (most VPLs are traced by no receiver of the warp: nothing else is computed
    // or stored for them)
    unsigned traced = 0;
    float wp[kSeg];
#pragma unroll
    for (int k = 0; k < kSeg; ++k) {
        const f3 d = y - xr[k];
        const float cx = dot_fma(nr[k], d);          // R26: the cosine terms as fused dots
        const float ci = -dot_fma(xyz(nb), d);
        wp[k] = cx * ci;
        if (((act >> k) & 1u) && yt != tri_x[k] && cx > 0.0f && ci > 0.0f) traced |= 1u << k;
    }
    if (!__any_sync(0xFFFFFFFFu, traced != 0)) return 0;
    RecvPos X;
#pragma unroll
    for (int k = 0; k < kSeg; ++k) { X.x[k] = xr[k]; hs->w[k] = wp[k]; }
    return shade_heavy<kCount>(bv, vpls, i, y, X, traced, cend, part, hs, sstack, st);
}

}  // namespace vplgi
