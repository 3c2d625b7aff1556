// gather.cuh — the warp-cooperative shadow-ray engine of the a8 gather
// (Eq. 1; DESIGN.md §3 O13 and §5).
//
// A warp owns 32 receivers x_j (one per lane) and walks a chunk of the
// gather's Morton-ordered VPL copy (render.cu), one VPL at a time — or, with
// VPL_GROUP > 1, in groups of nearby consecutive VPLs (measured slower at C4,
// off).  For each VPL every lane computes the Eq. 1 cosine terms of its
// receiver (exact fp32, O13), and the shadow segments x_j -> y that need a
// visibility test are resolved together:
//   1. occluder cache: exact MT tests against the lane's two latest occluders
//      (and, with VPL_CACHE_WARP, the warp's latest one), skipped by lanes
//      whose last traced segment was visible;
//   2. beam traversal of the 16-wide BVH (leaves = single triangles): all
//      remaining segments lie in the beam {y + s*D : y in Ybox, D in Dbox,
//      s in [s_lo, s_hi]}; lane c of each half-warp tests child c of a node
//      against it (interval arithmetic, two nodes per step, branch-free node
//      loads), hit inner children go on a warp-uniform shared-memory stack,
//      hit triangles are tested at once by every lane with a pending segment
//      with the exact MT of O9;
//   3. loose beams (a D component changes sign, or the spread of D is more
//      than 0.3 of the shortest segment) fall back to the per-ray packet
//      traversal of the 4-wide BVH (with groups: first one beam per VPL).
// Every lane's answer equals the exact any-hit of O9 for each of its
// segments: the beam and the boxes are conservative (boxes padded at build
// time), and extra MT tests cannot change an any-hit result.
#pragma once
#include "common.cuh"

namespace vplgi {

#ifndef VPL_GROUP
#define VPL_GROUP 1
#endif
#ifndef VPL_SMEM_ADDR
#define VPL_SMEM_ADDR 1     // traversal stack accessed through a 32-bit shared-window address held in a register
#endif
#ifndef VPL_NO_ORDER
#define VPL_NO_ORDER 0      // 1: push hit children in lane order (no near-to-far ordering)
#endif
#ifndef VPL_CACHE_STREAK
#define VPL_CACHE_STREAK 1  // skip the cache for lanes whose last traced segment was visible (C4: -45% cache MT, -2% time)
#endif
#ifndef VPL_CACHE_OWN2
#define VPL_CACHE_OWN2 1    // test the lane's second most recent occluder
#endif
#ifndef VPL_CACHE_WARP
#define VPL_CACHE_WARP 0    // 1: also test the warp's most recent occluder (v20: +0.8% at C4, off)
#endif
#ifndef VPL_GROUP_TOL
#define VPL_GROUP_TOL 0.05f
#endif
#ifndef VPL_CANDS
#define VPL_CANDS 1         // per-cluster candidate-triangle lists (one beam traversal per 32-VPL cluster)
#endif
#ifndef VPL_CAND_CAP
#define VPL_CAND_CAP 128    // list capacity (entries at the top of the warp's stack array); C4: 64 / 128 / 192 / 256 measured, 128 best
#endif
#ifndef VPL_CAND_GROUP
#define VPL_CAND_GROUP 16     // a list covers the next VPL_CAND_GROUP VPLs of the cluster from the first that needs it
                              // (C4: 8 / 12 / 16 / 24 / 32 measured, 16 best)
#endif
#ifndef VPL_CAND_TOL_PCT
#define VPL_CAND_TOL_PCT 0    // > 0: adaptive runs (box extent < VPL_CAND_TOL_PCT % of the distance), <= VPL_CAND_GROUP long
#endif
#ifndef VPL_CAND_MINRUN
#define VPL_CAND_MINRUN 2     // shorter adaptive runs get no list (per-VPL traversal)
#endif
#ifndef VPL_FAST_SEG
#define VPL_FAST_SEG 1   // segment setup by one rsqrt instead of IEEE sqrt + division (C4 -2.8%; reading R28)
#endif
#ifndef VPL_SCAP
#define VPL_SCAP 0.5f   // beam s-range cap at each end, in units of eps / |D|max (O9 tests t in (eps, L - eps))
#endif
#ifndef VPL_CAND_HYBRID
#define VPL_CAND_HYBRID 0     // 1: a list that would overflow keeps its unexpanded subtrees as entries (C4 +15%, off)
#endif
#ifndef VPL_CAND_ORDER
#define VPL_CAND_ORDER 0      // 1: list builds push children near-to-far like beam_traverse
#endif
#ifndef VPL_CAND_STRADDLE
#define VPL_CAND_STRADDLE 1   // 1: also build lists for beams with straddling axes (extent test; C4 -3%)
#endif
constexpr int kCandCap = VPL_CAND_CAP;
static_assert(kCandCap + 64 <= kWarpStack, "candidate list must leave room for the traversal stack");
constexpr int kGroup = VPL_GROUP;          // max VPLs per group
constexpr float kGroupTol = VPL_GROUP_TOL; // group iff the VPL box extent < tol * distance to the warp's receivers

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
__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

struct Beam {
    float a0[3], b0[3], a1[3], b1[3];
    float s_lo, s_hi;
    unsigned pos;   // bit a: D_a > 0
};

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

// One lane's shadow segments of a group: origin x (the receiver), direction
// d_k = (y_k - x)/|y_k - x|, t in (eps, |y_k - x| - eps)  (O9).
struct Segs {
    f3 d[kGroup];
    float tmax[kGroup];
    unsigned pend;   // bit k: segment k still unresolved
    unsigned occ;    // bit k: segment k occluded
};

// exact MT (O9) of the pending segments of one lane against one triangle;
// the origin-only terms s = x - v0, q = s x e1, e2.q are shared (identical
// operations to mt_any, so identical bits)
template <bool kCount>
__device__ __forceinline__ unsigned mt_segs(f3 o, const Segs& S, unsigned mask, float tmin, float4 a, float4 b,
                                            float4 c, TravStats* st) {
    const f3 v0 = xyz(a), e1 = xyz(b), e2 = xyz(c);
    const f3 s = o - v0;
    unsigned hit = 0;
    const f3 q = cross_fma(s, e1);
    const float tq = dot_fma(e2, q);
#pragma unroll
    for (int k = 0; k < kGroup; ++k) {
        if (kGroup == 1 || (mask & (1u << k))) {   // one segment: no branch, the mask is applied below
            if (kCount && (mask & (1u << k))) st->tris += 1;
            const f3 d = S.d[k];
            const f3 pv = cross_fma(d, e2);
            const float det = dot_fma(e1, pv);
            // O9 any hit, division-free (reading R25): sign-normalised by det (exact negations)
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
            hit &= mask;
        }
    }
    return hit;
}

template <bool kCount>
__device__ __forceinline__ void test_tri(const BvhView& bv, f3 x, Segs& S, float tmin, int tri, OccluderCache& cache,
                                         TravStats* st) {
    const unsigned m = S.pend;
    if (m) {
        const float4* tr = bv.tris + 3 * tri;
        unsigned h = mt_segs<kCount>(x, S, m, tmin, __ldg(tr), __ldg(tr + 1), __ldg(tr + 2), st);
        if (h) {
            S.occ |= h;
            S.pend &= ~h;
            cache.found(tri);
        }
    }
}

// Build the beam of the segments in `want` (bit k per lane; the group's
// VPL positions yk are uniform).  Returns false if the beam is loose.
__device__ __forceinline__ bool make_beam(f3 x, const f3* yk, unsigned want, unsigned kset, float eps, Beam& B) {
    const float inf = __int_as_float(0x7f800000);
    float dn[3] = {inf, inf, inf}, dm[3] = {-inf, -inf, -inf};
    float yl[3] = {inf, inf, inf}, yh[3] = {-inf, -inf, -inf};
    float l2n = inf, l2m = 0.0f;
#pragma unroll
    for (int k = 0; k < kGroup; ++k) {
        if (kset & (1u << k)) {   // uniform: VPL k takes part in the beam
            yl[0] = fminf(yl[0], yk[k].x); yh[0] = fmaxf(yh[0], yk[k].x);
            yl[1] = fminf(yl[1], yk[k].y); yh[1] = fmaxf(yh[1], yk[k].y);
            yl[2] = fminf(yl[2], yk[k].z); yh[2] = fmaxf(yh[2], yk[k].z);
        }
        if (want & (1u << k)) {
            f3 D = x - yk[k];
            dn[0] = fminf(dn[0], D.x); dm[0] = fmaxf(dm[0], D.x);
            dn[1] = fminf(dn[1], D.y); dm[1] = fmaxf(dm[1], D.y);
            dn[2] = fminf(dn[2], D.z); dm[2] = fmaxf(dm[2], D.z);
            float l2 = dot(D, D);
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
    return beam_from_bounds(Dn, Dm, yl, yh, lmin, lmax, kConeSpread, eps, B);
}

// Beam {y + s*D : y in [yl, yh], D in [Dn, Dm], s in [s_lo, s_hi]} from uniform bounds; lmin / lmax
// bound the segment lengths from below / above.  Returns false if the beam is loose.
__device__ __forceinline__ bool beam_from_bounds(const float* Dn, const float* Dm, const float* yl, const float* yh,
                                                 float lmin, float lmax, float spread_tol, float eps, Beam& B) {
    const float spread = fmax3(Dm[0] - Dn[0], Dm[1] - Dn[1], Dm[2] - Dn[2]);
    bool tight = spread < spread_tol * lmin;
    B.pos = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const bool p = Dn[a] > 0.0f, n = Dm[a] < 0.0f;
        tight &= p | n;
        if (p) B.pos |= 1u << a;
        // approximate reciprocals: a0 and b0 = y*a0 share the same a0, so s is scaled by
        // (1 + 2^-22) at most — a position error far below the box padding
        const float rmax = rcp_approx(Dm[a]), rmin = rcp_approx(Dn[a]);
        B.a0[a] = p ? rmax : rmin;
        B.b0[a] = (p ? yh[a] : yl[a]) * B.a0[a];
        B.a1[a] = p ? rmin : rmax;
        B.b1[a] = (p ? yl[a] : yh[a]) * B.a1[a];
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
        C.L[a] = sa ? yl[a] + Dn[a] : -inf;
        C.U[a] = sa ? yh[a] + Dm[a] : inf;
        if (sa) {
            ++straddle;
            C.B.pos |= 1u << a;   // N = lo, F = hi
            C.B.a0[a] = 0.0f; C.B.b0[a] = inf;
            C.B.a1[a] = 0.0f; C.B.b1[a] = -inf;
        }
    }
    return VPL_CAND_STRADDLE ? straddle < 3 : straddle == 0;
}
__device__ __forceinline__ bool cluster_beam_box(const ClusterBeam& C, float4 lo, float4 hi) {
    const bool ext = (lo.x <= C.U[0]) & (lo.y <= C.U[1]) & (lo.z <= C.U[2]) & (hi.x >= C.L[0]) &
                     (hi.y >= C.L[1]) & (hi.z >= C.L[2]);
    return ext & beam_box(C.B, lo, hi);
}

// beam traversal (two nodes per step); returns when every lane's S.pend is 0 or the tree is exhausted
template <bool kCount>
__device__ __forceinline__ void beam_traverse(const BvhView& bv, f3 x, Segs& S, float tmin, const Beam& B,
                                              unsigned dir_neg, OccluderCache& cache, int* __restrict__ sstack,
                                              TravStats* st, int sp0 = 0) {
    const int lane = threadIdx.x & 31;
    const int half = lane >> 4;
    const unsigned below = (1u << lane) - 1u;
    const unsigned hmask = half ? 0xFFFF0000u : 0x0000FFFFu;
    if (bv.root < 0) {  // single-triangle scene
        test_tri<kCount>(bv, x, S, tmin, 0, cache, st);
        return;
    }
    // the stack holds inner nodes only; sp0 > 0: the caller pre-filled it (a hybrid list's subtrees)
    int sp = sp0;
    if (sp0 == 0) {
        if (lane == 0) sstack[0] = bv.root;
        __syncwarp();
        sp = 1;
    }
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
        unsigned Bl = __ballot_sync(0xFFFFFFFFu, hit && ref < 0);
        if (Bi) {
            const int nB = __popc(Bi >> 16), nA = __popc(Bi & 0xFFFFu);
            const int rank = __popc(Bi & below & hmask);
#if VPL_NO_ORDER
            const int pos = (half ? 0 : nB) + rank;
#else
            const int nh = half ? nB : nA;
            const bool rev = (dir_neg >> axis) & 1u;   // segments run x -> y along -axis: visit descending
            const int pos = (half ? 0 : nB) + (rev ? rank : nh - 1 - rank);   // first to visit ends on top
#endif
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
            {   // no branch around the test: lanes with nothing pending are masked inside mt_segs
                const float4* tr = bv.tris + 3 * tri;
                const unsigned h = mt_segs<kCount>(x, S, S.pend, tmin, __ldg(tr), __ldg(tr + 1), __ldg(tr + 2), st);
                S.occ |= h;
                S.pend &= ~h;
                if (h) cache.found(tri);
            }
            if (!__any_sync(0xFFFFFFFFu, S.pend != 0)) return;
        }
    }
}

// Candidate list of a VPL cluster: one beam traversal of the 16-wide BVH with
// the cluster beam (make_cluster_beam) that records every triangle child whose
// box the beam reaches — no MT tests, no early exit.  Any triangle that can
// block a segment of the cluster is in the list (the same conservative beam /
// padded box argument as beam_traverse), so each VPL of the cluster then tests
// only the list (filter_cands) instead of traversing the tree.  The list holds
// 16-wide child slots (node * 16 + child) at the top of the warp's stack
// array, in the order the traversal met them; returns its length, or -1 if
// the beam is loose, the list overflows kCandCap or the stack meets the list.
template <bool kCount>
#ifndef VPL_CAND_NOINLINE
#define VPL_CAND_NOINLINE 1   // keep the (rare) list build out of the hot loop's register allocation
#endif
#if VPL_CAND_NOINLINE
__device__ __noinline__
#else
__device__ __forceinline__
#endif
int build_cands(const BvhView& bv, f3 x, bool part, const vpl_record* __restrict__ vg, int ng, float eps,
                                        int* __restrict__ sstack, TravStats* st, int& run) {
    const int lane = threadIdx.x & 31;
    run = ng;
    if (bv.root < 0) return -1;
    const float inf = __int_as_float(0x7f800000);
    const float xl[3] = {warp_min_f32(part ? x.x : inf), warp_min_f32(part ? x.y : inf), warp_min_f32(part ? x.z : inf)};
    const float xh[3] = {warp_max_f32(part ? x.x : -inf), warp_max_f32(part ? x.y : -inf),
                         warp_max_f32(part ? x.z : -inf)};
    // position box of the run vg[0..run) (lane l loads VPL l)
    float4 ylo = make_float4(inf, inf, inf, 0.0f), yhi = make_float4(-inf, -inf, -inf, 0.0f);
    if (lane < ng) { const float4 p = __ldg((const float4*)(vg + lane)); ylo = p; yhi = p; }
#if VPL_CAND_TOL_PCT > 0
    {   // adaptive run: the longest prefix whose box stays within VPL_CAND_TOL_PCT % of the distance from its first
        // VPL to the receivers (inclusive prefix min / max over the lanes)
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const float a0 = __shfl_up_sync(0xFFFFFFFFu, ylo.x, o), a1 = __shfl_up_sync(0xFFFFFFFFu, ylo.y, o);
            const float a2 = __shfl_up_sync(0xFFFFFFFFu, ylo.z, o), b0 = __shfl_up_sync(0xFFFFFFFFu, yhi.x, o);
            const float b1 = __shfl_up_sync(0xFFFFFFFFu, yhi.y, o), b2 = __shfl_up_sync(0xFFFFFFFFu, yhi.z, o);
            if (lane >= o) {
                ylo.x = fminf(ylo.x, a0); ylo.y = fminf(ylo.y, a1); ylo.z = fminf(ylo.z, a2);
                yhi.x = fmaxf(yhi.x, b0); yhi.y = fmaxf(yhi.y, b1); yhi.z = fmaxf(yhi.z, b2);
            }
        }
        const float y0x = __shfl_sync(0xFFFFFFFFu, ylo.x, 0), y0y = __shfl_sync(0xFFFFFFFFu, ylo.y, 0),
                    y0z = __shfl_sync(0xFFFFFFFFu, ylo.z, 0);
        const float cx = 0.5f * (xl[0] + xh[0]) - y0x, cy = 0.5f * (xl[1] + xh[1]) - y0y,
                    cz = 0.5f * (xl[2] + xh[2]) - y0z;
        constexpr float kTol = VPL_CAND_TOL_PCT * 0.01f;
        const float lim2 = (kTol * kTol) * ((cx * cx + cy * cy) + cz * cz);
        const float ext = fmax3(yhi.x - ylo.x, yhi.y - ylo.y, yhi.z - ylo.z);
        const unsigned bad = __ballot_sync(0xFFFFFFFFu, lane < ng && !(ext * ext < lim2));
        run = bad ? min(ng, __ffs(bad) - 1) : ng;
        if (run < VPL_CAND_MINRUN) { run = 1; return -1; }
        const int l = run - 1;
        ylo.x = __shfl_sync(0xFFFFFFFFu, ylo.x, l); ylo.y = __shfl_sync(0xFFFFFFFFu, ylo.y, l);
        ylo.z = __shfl_sync(0xFFFFFFFFu, ylo.z, l); yhi.x = __shfl_sync(0xFFFFFFFFu, yhi.x, l);
        yhi.y = __shfl_sync(0xFFFFFFFFu, yhi.y, l); yhi.z = __shfl_sync(0xFFFFFFFFu, yhi.z, l);
    }
#else
    ylo.x = warp_min_f32(ylo.x); ylo.y = warp_min_f32(ylo.y); ylo.z = warp_min_f32(ylo.z);
    yhi.x = warp_max_f32(yhi.x); yhi.y = warp_max_f32(yhi.y); yhi.z = warp_max_f32(yhi.z);
#endif
    ClusterBeam CB;
    if (!make_cluster_beam(xl, xh, ylo, yhi, eps, CB)) return -1;
    const int half = lane >> 4;
    const unsigned below = (1u << lane) - 1u;
#if VPL_CAND_ORDER
    const unsigned hmask = half ? 0xFFFF0000u : 0x0000FFFFu;
    const unsigned dir_neg = CB.B.pos;
#endif
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
#if VPL_CAND_ORDER
        const int axis = __float_as_int(hi.w);
#endif
        const bool hit = (ref != INT_MIN) & cluster_beam_box(CB, lo, hi);
        if (kCount) {
            const unsigned real = __ballot_sync(0xFFFFFFFFu, ref != INT_MIN);
            if (lane == 0) st->cones += __popc(real);
        }
        const unsigned Bi = __ballot_sync(0xFFFFFFFFu, hit && ref >= 0);
        const unsigned Bl = __ballot_sync(0xFFFFFFFFu, hit && ref < 0);
        const int nl = __popc(Bl), ni = __popc(Bi);
#if VPL_CAND_HYBRID
        // invariant n + sp <= kCandCap: if this step's results would break it, the two nodes just
        // popped and every node still on the stack go into the list unexpanded (node | 0x80000000):
        // each VPL then tests the expanded part flat and traverses those subtrees with its own beam
        if (n + nl + sp + ni > kCandCap) {
            __syncwarp();
            const unsigned Bp = __ballot_sync(0xFFFFFFFFu, (lane & (kWide - 1)) == 0 && node >= 0);
            if ((lane & (kWide - 1)) == 0 && node >= 0)
                sstack[kWarpStack - 1 - (n + __popc(Bp & below))] = node | (int)0x80000000u;
            n += __popc(Bp);
            for (int k = lane; k < sp; k += 32) sstack[kWarpStack - 1 - (n + k)] = sstack[k] | (int)0x80000000u;
            n += sp;
            __syncwarp();
            if (kCount && lane == 0) st->lfail += 1;   // counted as a partial list
            return n;
        }
#endif
        __syncwarp();
        if (Bl) {
#if !VPL_CAND_HYBRID
            if (n + nl > kCandCap) {
#ifdef VPL_CAND_DIAG
                if (kCount && lane == 0) st->boxes += 1u << 20;   // diagnostic builds: overflow count in box_tests
#endif
                return -1;
            }
#endif
            if (hit && ref < 0) sstack[kWarpStack - 1 - (n + __popc(Bl & below))] = slot;
            n += nl;
        }
        if (Bi) {
            const int nB = __popc(Bi >> 16), nA = __popc(Bi & 0xFFFFu);
#if !VPL_CAND_HYBRID
            if (sp + nA + nB > kWarpStack - kCandCap) {
#ifdef VPL_CAND_DIAG
                if (kCount && lane == 0) st->boxes += 1u << 20;
#endif
                return -1;
            }
#endif
#if VPL_CAND_ORDER
            const int rank = __popc(Bi & below & hmask);
            const int nh = half ? nB : nA;
            const bool rev = (dir_neg >> axis) & 1u;
            const int pos = (half ? 0 : nB) + (rev ? rank : nh - 1 - rank);
#else
            const int pos = __popc(Bi & below);   // collection order does not matter: push in lane order
#endif
            if (hit && ref >= 0) sstack[sp + pos] = ref;
            sp += nA + nB;
        }
        __syncwarp();
    }
    return n;
}

// Frustum of one VPL's pending segments (apex y, the VPL): with m the dominant axis of the first
// pending segment's direction d_j = (y - x_j)/L_j and a, b the other two, every pending d_j has the
// same sign of d_m (a tight beam never changes sign) and slopes p_j = d_a/d_m, q_j = d_b/d_m; every
// point of segment j is P = y - s L_j d_j, s in [0, 1], so with sigma = -sign(d_m),
// A = sigma (P - y)_a, B = sigma (P - y)_b, U = sigma (P - y)_m it satisfies U >= 0,
// pmin U <= A <= pmax U, qmin U <= B <= qmax U (slopes
// widened by 2^-18 relative).  A triangle whose three vertices all violate one of these by more than
// the margin (the box padding, times the plane normal's L1 norm) cannot be crossed by any pending
// segment: the same conservative argument as the padded boxes (MT's rounding stays far inside it).
#ifndef VPL_FRUSTUM
#define VPL_FRUSTUM 0   // 1: frustum pre-test before MT in the filter (C4: filter MT -19%, time +8%; off)
#endif
struct Frustum {
    int a, b, m;
    float sg, yA, yB, yU;           // sigma and the apex in the (A, B, U) frame
    float pmin, pmax, qmin, qmax;
    float mp, mq, mu;               // margins
    __device__ __forceinline__ void make(const Segs& S, f3 y, float pad) {
        const float inf = __int_as_float(0x7f800000);
        const bool live = S.pend != 0;
        const unsigned act = __ballot_sync(0xFFFFFFFFu, live);
        const int l0 = __ffs(act) - 1;
        const f3 d = S.d[0];
        const float ax = fabsf(d.x), ay = fabsf(d.y), az = fabsf(d.z);
        const int mm = (ax >= ay && ax >= az) ? 0 : (ay >= az ? 1 : 2);
        m = __shfl_sync(0xFFFFFFFFu, mm, l0);
        a = m == 0 ? 1 : 0;
        b = m == 2 ? 1 : 2;
        const float dv[3] = {d.x, d.y, d.z};
        const float dm = dv[m], da = dv[a], db = dv[b];
        const float r = __fdividef(1.0f, dm);
        const float p = live ? da * r : 0.0f, q = live ? db * r : 0.0f;
        sg = __shfl_sync(0xFFFFFFFFu, dm, l0) < 0.0f ? 1.0f : -1.0f;   // P - y = -s L d_j: U = sigma (P - y)_m >= 0
        const float p0 = warp_min_f32(live ? p : inf), p1 = warp_max_f32(live ? p : -inf);
        const float q0 = warp_min_f32(live ? q : inf), q1 = warp_max_f32(live ? q : -inf);
        const float w = 0x1p-18f;
        pmin = p0 - w * (fabsf(p0) + 1.0f); pmax = p1 + w * (fabsf(p1) + 1.0f);
        qmin = q0 - w * (fabsf(q0) + 1.0f); qmax = q1 + w * (fabsf(q1) + 1.0f);
        const float yv[3] = {y.x, y.y, y.z};
        yA = sg * yv[a]; yB = sg * yv[b]; yU = sg * yv[m];
        mp = pad * (1.0f + fmaxf(fabsf(pmin), fabsf(pmax)));
        mq = pad * (1.0f + fmaxf(fabsf(qmin), fabsf(qmax)));
        mu = pad;
    }
    // v0 = a.xyz, v1 = v0 + e1, v2 = v0 + e2 (the leaf-ordered triangle record)
    __device__ __forceinline__ bool culls(float4 t0, float4 t1, float4 t2) const {
        const float v0[3] = {t0.x, t0.y, t0.z};
        const float e1[3] = {t1.x, t1.y, t1.z}, e2[3] = {t2.x, t2.y, t2.z};
        float A[3], B[3], U[3];
        const float s = sg;
        A[0] = s * v0[a] - yA; A[1] = s * (v0[a] + e1[a]) - yA; A[2] = s * (v0[a] + e2[a]) - yA;
        B[0] = s * v0[b] - yB; B[1] = s * (v0[b] + e1[b]) - yB; B[2] = s * (v0[b] + e2[b]) - yB;
        U[0] = s * v0[m] - yU; U[1] = s * (v0[m] + e1[m]) - yU; U[2] = s * (v0[m] + e2[m]) - yU;
        // each plane: cull iff min over the vertices of its outside distance > margin
        const float f1 = fmin3(fmaf(-pmax, U[0], A[0]), fmaf(-pmax, U[1], A[1]), fmaf(-pmax, U[2], A[2]));
        const float f2 = fmin3(fmaf(pmin, U[0], -A[0]), fmaf(pmin, U[1], -A[1]), fmaf(pmin, U[2], -A[2]));
        const float f3v = fmin3(fmaf(-qmax, U[0], B[0]), fmaf(-qmax, U[1], B[1]), fmaf(-qmax, U[2], B[2]));
        const float f4 = fmin3(fmaf(qmin, U[0], -B[0]), fmaf(qmin, U[1], -B[1]), fmaf(qmin, U[2], -B[2]));
        const float f5 = -fmax3(U[0], U[1], U[2]);
        return (f1 > mp) | (f2 > mp) | (f3v > mq) | (f4 > mq) | (f5 > mu);
    }
};

// The pending segments of one VPL against its cluster's candidate list: lane c
// tests candidate c of each batch of 32 against the VPL's own beam; hit
// triangles get the exact MT of O9 from every lane with a pending segment.
template <bool kCount>
__device__ __forceinline__ void filter_cands(const BvhView& bv, f3 x, Segs& S, float tmin, const Beam& B,
                                             int* __restrict__ sstack, int ncand, OccluderCache& cache,
                                             TravStats* st, f3 y) {
    const int lane = threadIdx.x & 31;
#if VPL_CAND_HYBRID
    const unsigned below = (1u << lane) - 1u;
#endif
#if VPL_FRUSTUM
    Frustum F;
    F.make(S, y, fmaxf(bv.box_pad, tmin));
#endif
#if VPL_CAND_HYBRID
    int sp = 0;   // subtrees of a hybrid list, traversed after the flat part
#endif
    for (int base = 0; base < ncand; base += 32) {
        const int i = base + lane;
        const bool ok = i < ncand;
        const int e = ok ? sstack[kWarpStack - 1 - i] : 0;     // child slot, or node | 0x80000000
        const bool sub = e < 0;
        const int slot = sub ? 0 : e;                          // slot 0: a real child, masked below
        const float4* nd = (const float4*)((const char*)bv.wide + ((size_t)slot << 5));
        const float4 lo = __ldg(nd), hi = __ldg(nd + 1);
        bool hit = ok & !sub & beam_box(B, lo, hi);
        if (kCount && lane == 0) { st->fsteps += 1; st->cones += min(32, ncand - base); }
#if VPL_FRUSTUM
        if (__any_sync(0xFFFFFFFFu, hit)) {   // frustum pre-test of the box hits (lane-parallel)
            const int to0 = 3 * (~__float_as_int(lo.w) >> 3);
            const float4* tr = bv.tris + (hit ? to0 : 0);
            const float4 a = __ldg(tr), b = __ldg(tr + 1), c = __ldg(tr + 2);
            if (kCount && hit) st->ftests += 1;
            hit &= !F.culls(a, b, c);
        }
#endif
#if VPL_CAND_HYBRID
        const unsigned Bs = __ballot_sync(0xFFFFFFFFu, ok && sub);
        if (Bs) {
            if (ok && sub) sstack[sp + __popc(Bs & below)] = e & 0x7FFFFFFF;
            sp += __popc(Bs);
            __syncwarp();
        }
#endif
        unsigned Bl = __ballot_sync(0xFFFFFFFFu, hit);
        const int toff = 3 * (~__float_as_int(lo.w) >> 3);   // float4 offset of the candidate's triangle
        while (Bl) {
            const int k = 31 - __clz(Bl);                      // highest first: one FLO
            Bl &= ~(1u << k);
            const int to = __shfl_sync(0xFFFFFFFFu, toff, k);
            VPL_DCHECK(to >= 0 && to < 3 * bv.n);
            const float4* tr = bv.tris + to;
            const unsigned h = mt_segs<kCount>(x, S, S.pend, tmin, __ldg(tr), __ldg(tr + 1), __ldg(tr + 2), st);
            if (kCount) {   // warp-level MT tests of the filter, and those that found an occluder
                const bool any = __any_sync(0xFFFFFFFFu, h != 0);
                if (lane == 0) { st->fmt += 1; st->fmt_hit += any; }
            }
            S.occ |= h;
            S.pend &= ~h;
            if (h) cache.found(to / 3);
            if (!__any_sync(0xFFFFFFFFu, S.pend != 0)) return;
        }
    }
#if VPL_CAND_HYBRID
    if (sp > 0) beam_traverse<kCount>(bv, x, S, tmin, B, B.pos, cache, sstack, st, sp);
#endif
}

// Resolve the pending segments of a group: beam over the group, else one beam
// per VPL, else per-ray packets.  yk: the group's VPL positions (uniform).
template <bool kCount>
__device__ __forceinline__ void resolve_group(const BvhView& bv, f3 x, Segs& S, float eps, const f3* yk, int g,
                                              OccluderCache& cache, int* __restrict__ sstack, TravStats* st,
                                              int& cand, int& cand_end, int cend, bool part,
                                              const vpl_record* __restrict__ vpls, int i) {
    const int lane = threadIdx.x & 31;
    unsigned kany = 0;   // VPLs with a pending segment in some lane (uniform)
#pragma unroll
    for (int k = 0; k < kGroup; ++k)
        if (__any_sync(0xFFFFFFFFu, (S.pend >> k) & 1u)) kany |= 1u << k;
    if (!kany) return;
    const unsigned had = S.occ;
    if (kCount && lane == 0) st->wrays += 1;
    Beam B;
    if (make_beam(x, yk, S.pend, kany, eps, B)) {
        if (kCount && lane == 0) st->cpk += 1;
        if (VPL_CANDS && kGroup == 1 && i >= cand_end) {
            int run;
            cand = build_cands<kCount>(bv, x, part, vpls + i, min(VPL_CAND_GROUP, cend - i), eps, sstack, st, run);
            cand_end = i + run;
            if (kCount && lane == 0) { if (cand >= 0) { st->lists += 1; st->entries += cand; } else st->lfail += 1; }
        }
        // the list covers the participating receivers only (the cluster cull is conservative, so a lane
        // with a pending segment always participates; checked anyway)
        if (VPL_CANDS && kGroup == 1 && cand >= 0 && !__any_sync(0xFFFFFFFFu, S.pend && !part))
            filter_cands<kCount>(bv, x, S, eps, B, sstack, cand, cache, st, yk[0]);
        else
            beam_traverse<kCount>(bv, x, S, eps, B, B.pos, cache, sstack, st);
    } else {
        // loose: one beam per VPL of the group, loose single beams go per ray
        const bool several = kGroup > 1 && __popc(kany) > 1;   // compile-time false for single-VPL groups
        const unsigned all = S.pend;
#pragma unroll
        for (int k = 0; k < kGroup; ++k) {
            if (!(kany & (1u << k))) continue;                      // uniform
            S.pend = all & (1u << k);
            if (several && make_beam(x, yk, S.pend, 1u << k, eps, B)) {
                if (kCount && lane == 0) st->cpk += 1;
                beam_traverse<kCount>(bv, x, S, eps, B, B.pos, cache, sstack, st);
            } else {
                if (kCount && lane == 0) st->rpk += 1;
                // per-ray packet traversal of the 4-wide BVH for segment k
                Ray r;
                r.o = x; r.d = S.d[k]; r.tmin = eps; r.tmax = S.tmax[k];
                const bool live = S.pend != 0;
                const int leader = __ffs(__ballot_sync(0xFFFFFFFFu, live)) - 1;
                const unsigned neg = (r.d.x < 0.0f ? 1u : 0u) | (r.d.y < 0.0f ? 2u : 0u) | (r.d.z < 0.0f ? 4u : 0u);
                const unsigned dn = __shfl_sync(0xFFFFFFFFu, neg, leader);
                if (warp_traverse_ray<kCount>(bv, r, live, false, cache, dn, sstack, st) && live) S.occ |= 1u << k;
            }
        }
    }
    S.pend = 0;
#if VPL_CACHE_WARP
    // share the newest occluder found in this resolution with the whole warp
    const unsigned fresh = __ballot_sync(0xFFFFFFFFu, (S.occ & ~had) != 0);
    if (fresh) cache.warp = __shfl_sync(0xFFFFFFFFu, cache.own0, __ffs(fresh) - 1);
#else
    (void)had;
#endif
}

// The VPL group starting at i (uniform): the longest run of <= kGroup VPLs in
// [i, iend) whose position box stays within kGroupTol x the distance from
// the first VPL to the warp's reference receiver xr.
__device__ __forceinline__ int group_at(const vpl_record* __restrict__ vpls, int i, int iend, f3 xr, f3* yk,
                                        int* yt) {
    const float4* p = (const float4*)(vpls + i);
    float4 a = __ldg(p);
    yk[0] = xyz(a);
    yt[0] = __float_as_int(a.w);   // the VPL's triangle (record field tri)
    f3 lo = yk[0], hi = yk[0];
    f3 dr = yk[0] - xr;
    const float lim = kGroupTol * sqrtf(dot(dr, dr));
    int g = 1;
#pragma unroll
    for (int k = 1; k < kGroup; ++k) {
        if (g == k && i + k < iend) {
            float4 b = __ldg(p + 3 * k);
            f3 y = xyz(b);
            f3 l2 = mk3(fminf(lo.x, y.x), fminf(lo.y, y.y), fminf(lo.z, y.z));
            f3 h2 = mk3(fmaxf(hi.x, y.x), fmaxf(hi.y, y.y), fmaxf(hi.z, y.z));
            if (fmax3(h2.x - l2.x, h2.y - l2.y, h2.z - l2.z) < lim) {
                yk[k] = y; yt[k] = __float_as_int(b.w); lo = l2; hi = h2; g = k + 1;
            }
        }
    }
    return g;
}

// One group for one lane: Eq. 1 terms (O13, exact fp32 order), segment
// setup (O9), cache, traversal.  Returns traced | vis << 16: the traced mask and vis = traced and
// unoccluded; w[k] = cx*ci / (r2 * max(r2, b2)) for the visible ones.
template <bool kCount>
__device__ __forceinline__ unsigned shade_group(const BvhView& bv, const vpl_record* __restrict__ vpls, int i, int g,
                                                const f3* yk, const int* yt, f3 x, f3 nx, int tri_x, bool active,
                                                float eps,
                                                float b2, OccluderCache& cache, int* __restrict__ sstack,
                                                TravStats* st, float* w, int& cand, int& cand_end, int cend,
                                                bool part) {
    Segs S;
    S.pend = 0; S.occ = 0;
    unsigned traced = 0;
#pragma unroll
    for (int k = 0; k < kGroup; ++k) {
        w[k] = 0.0f;
        S.d[k] = mk3(0.0f, 0.0f, 0.0f);
        S.tmax[k] = 0.0f;
        if (k < g) {
            const float4 nb = __ldg((const float4*)(vpls + i + k) + 1);
            const int tri_i = yt[k];
            const f3 d = yk[k] - x;
            const float r2 = dot(d, d);
            const float cx = dot_fma(nx, d);          // R26: the cosine terms as fused dots
            const float ci = -dot_fma(xyz(nb), d);
            if (active && tri_i != tri_x && cx > 0.0f && ci > 0.0f) {
                traced |= 1u << k;
                w[k] = (cx * ci) * rcp_approx(r2 * fmaxf(r2, b2));   // r2 * max(r2, b2) >= b2^2: normal range
#if VPL_FAST_SEG
                // one MUFU: 1/dist and dist within ~2 ulp of O9's IEEE sqrt / division (visibility then
                // differs from the oracle only for grazing hits, inside BJ:5's 1e-4 budget)
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
    }
    if (!__any_sync(0xFFFFFFFFu, traced != 0)) return 0;
    // occluder cache: exact MT against recent occluders
    const uint32_t t0 = kCount ? st->tris : 0;
#if VPL_CACHE_STREAK
    // a lane whose last traced segment was visible skips the cache (visibility is coherent
    // along the spatially ordered VPLs)
    const unsigned cpend = cache.vis_streak ? 0u : S.pend;
    const unsigned keep_pend = S.pend & ~cpend;
    S.pend = cpend;
#endif
    if (S.pend && cache.own0 >= 0) test_tri<kCount>(bv, x, S, eps, cache.own0, cache, st);
    if (VPL_CACHE_OWN2 && S.pend && cache.own1 >= 0) test_tri<kCount>(bv, x, S, eps, cache.own1, cache, st);
    if (VPL_CACHE_WARP && S.pend && cache.warp >= 0 && cache.warp != cache.own0 && cache.warp != cache.own1)
        test_tri<kCount>(bv, x, S, eps, cache.warp, cache, st);
#if VPL_CACHE_STREAK
    S.pend |= keep_pend;
#endif
    if (kCount) { st->chits += __popc(S.occ); st->ctests += st->tris - t0; }
    resolve_group<kCount>(bv, x, S, eps, yk, g, cache, sstack, st, cand, cand_end, cend, part, vpls, i);
    const unsigned vis = traced & ~S.occ;
#if VPL_CACHE_STREAK
    if (traced) cache.vis_streak = (vis == traced);
#endif
    return traced | vis << 16;
}

}  // namespace vplgi
