// common.cuh — device-side layouts, exact fp32 helpers, Philox and BVH
// traversal shared by the kernels of libvplgi.so (sm_100a).
//
// Every translation unit is compiled with -fmad=false: a*b+c stays an FMUL
// followed by an FADD, so the bit-exact steps (DESIGN.md §3 O1-O12) match the
// IEEE definition written in DESIGN.md.  Where a result only has to be
// conservative (the BVH slab test) the code calls fmaf() explicitly.
#pragma once
#include <cstdint>
#include <cstddef>
#include <climits>
#include <cstdio>
#include <cuda_runtime.h>

#include "../../include/vplgi.h"

namespace vplgi {

// ------------------------------------------------------------------ errors
void set_error(const char* fmt, ...);
int32_t check_cuda(cudaError_t e, const char* what);
int32_t check_launch(const char* what);  // also counts the launch (vpl_launch_count)
int32_t check_arch();

#define VPL_TRY(expr)                      \
    do {                                   \
        int32_t _st = (expr);              \
        if (_st != VPL_OK) return _st;     \
    } while (0)
#define VPL_CUDA(call) VPL_TRY(::vplgi::check_cuda((call), #call))
#define VPL_LAUNCHED(name) VPL_TRY(::vplgi::check_launch(name))

// Device-side bounds checks (stack depth, node / triangle / block indices),
// compiled in with -DVPL_DEBUG=1 (tools/debug_checks.py builds that variant
// and runs the parity tests on it); a failed check prints and traps, which
// the next call reports as VPL_ECUDA.
#ifndef VPL_DEBUG
#define VPL_DEBUG 0
#endif
#if VPL_DEBUG
#define VPL_DCHECK(c)                                                                   \
    do {                                                                                \
        if (!(c)) {                                                                     \
            printf("VPL_DCHECK %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c, \
                   (int)blockIdx.x, (int)threadIdx.x);                                  \
            __trap();                                                                   \
        }                                                                               \
    } while (0)
#else
#define VPL_DCHECK(c) \
    do {              \
    } while (0)
#endif

// ------------------------------------------------------------------ layouts
constexpr int kMaxLights = VPL_MAX_LIGHTS;
constexpr size_t kAlign = 256;
__host__ __device__ inline size_t align_up(size_t x) { return (x + kAlign - 1) & ~(kAlign - 1); }

// Scene blob = SceneHdr followed by SoA arrays (offsets from the blob start).
struct SceneHdr {
    int64_t n;
    int32_t nL, W, H, pad0;
    float cam[14];                  // pos fwd up right tan_x tan_y
    float lights[16 * kMaxLights];  // vpl_light rows
    uint32_t bbox_enc[6];           // order-preserving encodings (lo x y z, hi x y z) for atomics
    float bbox_lo[3], bbox_hi[3];
    double diag;
    float eps, b2, box_pad, pad1;
    unsigned long long bad;         // lowest degenerate triangle (ULLONG_MAX = none)
    int64_t off_verts, off_nrm, off_alb, off_cen, off_aq;
};

struct SceneView {
    const SceneHdr* hdr;
    const float* verts;     // [9N]
    const float4* nrm;      // [N] xyz = unit normal, w = area
    const float4* alb;      // [N] rgb albedo
    const float4* cen;      // [N] centroid
    const uint64_t* aq;     // [N] 40-bit fixed-point area
};

inline size_t scene_layout(int64_t n, SceneHdr* h) {
    size_t off = align_up(sizeof(SceneHdr));
    size_t o_v = off; off = align_up(off + sizeof(float) * 9 * (size_t)n);
    size_t o_n = off; off = align_up(off + sizeof(float4) * (size_t)n);
    size_t o_a = off; off = align_up(off + sizeof(float4) * (size_t)n);
    size_t o_c = off; off = align_up(off + sizeof(float4) * (size_t)n);
    size_t o_q = off; off = align_up(off + sizeof(uint64_t) * (size_t)n);
    if (h) { h->off_verts = o_v; h->off_nrm = o_n; h->off_alb = o_a; h->off_cen = o_c; h->off_aq = o_q; }
    return off;
}

// Host-side view: offsets are read from a host copy of the header.
inline SceneView scene_view(const void* blob, int64_t n) {
    SceneHdr h;
    scene_layout(n, &h);
    const char* b = (const char*)blob;
    SceneView v;
    v.hdr = (const SceneHdr*)b;
    v.verts = (const float*)(b + h.off_verts);
    v.nrm = (const float4*)(b + h.off_nrm);
    v.alb = (const float4*)(b + h.off_alb);
    v.cen = (const float4*)(b + h.off_cen);
    v.aq = (const uint64_t*)(b + h.off_aq);
    return v;
}

// BVH blob = BvhHdr, internal nodes (4 float4 each), leaf-ordered triangles
// (3 float4 each: v0 | orig index bits, e1, e2), leaf-ordered triangle planes
// (1 float4 each: unit normal of e1 x e2 and offset n.v0, rounded from float64).
// Two wide node formats built from the binary PLOC tree:
//  * 4-wide (per-ray packet traversal): SoA child boxes as centre / half
//    extent c.x[4] e.x[4] c.y[4] e.y[4] c.z[4] e.z[4], refs[4], meta (axis,
//    valid-slot mask) — 8 float4;
//  * 16-wide (cone traversal, one child per lane): child c = 2 float4
//    (lo.xyz | ref bits, hi.xyz | split-axis bits), empty slots ref INT_MIN.
// Children are sorted by centre along the node's largest axis.
constexpr int kWide4 = 4;
constexpr int kWide4F4 = 8;
constexpr int kWide = 16;
constexpr int kWideF4 = 2 * kWide;  // float4s per 16-wide node (512 B)

struct BvhHdr {
    int64_t n;
    int32_t root;       // 0 (internal) or ~0 (single leaf)
    int32_t pad;
    int64_t off_nodes, off_tris, off_wide, off_wide4, off_planes;
};
struct BvhView {
    const float4* nodes;   // binary nodes (per-thread traversals)
    const float4* tris;
    const float4* wide;    // 16-wide nodes (cone traversal)
    const float4* wide4;   // 4-wide nodes (per-ray packet traversal)
    const float4* planes;  // leaf-ordered triangle planes (unit normal, offset): the gather's plane-side cull
    int32_t root;
    int32_t n;             // triangles (bounds checks under VPL_DEBUG)
    float box_pad;         // the scene's box padding (SceneHdr::box_pad), set by callers that need it
};
inline size_t bvh_layout(int64_t n, BvhHdr* h) {
    size_t off = align_up(sizeof(BvhHdr));
    size_t ni = (size_t)(n > 1 ? n - 1 : 1);
    size_t o_n = off; off = align_up(off + sizeof(float4) * 4 * ni);
    size_t o_t = off; off = align_up(off + sizeof(float4) * 3 * (size_t)n);
    size_t o_w = off; off = align_up(off + sizeof(float4) * kWideF4 * ni);
    size_t o_w4 = off; off = align_up(off + sizeof(float4) * kWide4F4 * ni);
    size_t o_pl = off; off = align_up(off + sizeof(float4) * (size_t)n);
    if (h) {
        h->n = n; h->root = n > 1 ? 0 : ~0;
        h->off_nodes = o_n; h->off_tris = o_t; h->off_wide = o_w; h->off_wide4 = o_w4; h->off_planes = o_pl;
    }
    return off;
}
inline BvhView bvh_view(const void* blob, int64_t n) {
    BvhHdr h;
    bvh_layout(n, &h);
    BvhView v;
    v.nodes = (const float4*)((const char*)blob + h.off_nodes);
    v.tris = (const float4*)((const char*)blob + h.off_tris);
    v.wide = (const float4*)((const char*)blob + h.off_wide);
    v.wide4 = (const float4*)((const char*)blob + h.off_wide4);
    v.planes = (const float4*)((const char*)blob + h.off_planes);
    v.root = h.root;
    v.n = (int32_t)n;
    v.box_pad = 0.0f;
    return v;
}

// stream-ordered host copy of the scene header (n, offsets, constants)
inline int32_t read_scene_hdr(const void* d_scene, cudaStream_t s, SceneHdr* out) {
    VPL_CUDA(cudaMemcpyAsync(out, d_scene, sizeof(SceneHdr), cudaMemcpyDeviceToHost, s));
    VPL_CUDA(cudaStreamSynchronize(s));
    return VPL_OK;
}

// bump allocator over a caller work buffer (base may be null for sizing)
struct Bump {
    char* base;
    size_t off = 0;
    template <class T>
    T* take(size_t count) {
        T* p = base ? (T*)(base + off) : nullptr;
        off = align_up(off + sizeof(T) * count);
        return p;
    }
};

// ------------------------------------------------------------------ fp32 vector math (exact op order, O0)
struct f3 { float x, y, z; };
__device__ __forceinline__ f3 mk3(float x, float y, float z) { return f3{x, y, z}; }
__device__ __forceinline__ f3 ld3(const float* p) { return f3{p[0], p[1], p[2]}; }
__device__ __forceinline__ f3 xyz(float4 a) { return f3{a.x, a.y, a.z}; }
__device__ __forceinline__ f3 operator+(f3 a, f3 b) { return f3{a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ f3 operator-(f3 a, f3 b) { return f3{a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ f3 operator*(float s, f3 a) { return f3{s * a.x, s * a.y, s * a.z}; }
__device__ __forceinline__ float dot(f3 a, f3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
__device__ __forceinline__ f3 cross(f3 a, f3 b) {
    return f3{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}

// ------------------------------------------------------------------ lights
// A light row (vpl_light, 16 floats) with area == 0 is an isotropic point light at `corner` whose
// `radiance` field holds its power Phi (reading R27; e_u = e_v = 0).
__device__ __forceinline__ bool light_is_point(const float* L) { return L[12] == 0.0f; }
// Eq. 2's point-light geometry term without D (R1): cos(omega) / (4 pi r^2) with
// cos(omega) = cp / r, cp = n.d for the unnormalised d = light - x: cp / ((r2 sqrt(r2)) 4 pi), exact fp32
__device__ __forceinline__ float point_g(float cp, float r2) {
    constexpr float kFourPi = (float)(4.0 * 3.14159265358979323846);
    return cp / ((r2 * sqrtf(r2)) * kFourPi);
}

// ------------------------------------------------------------------ Philox4x32-10
struct Philox {
    // counter = (j >> 2, item, stream, 0), key = (seed lo, seed hi); draw j = lane j & 3
    uint32_t item, stream, k0, k1;
    uint32_t j = 0;
    uint32_t blk_id = 0xFFFFFFFFu;
    uint32_t blk[4];
    __device__ Philox(uint64_t seed, uint32_t stream_, uint32_t item_)
        : item(item_), stream(stream_), k0((uint32_t)seed), k1((uint32_t)(seed >> 32)) {}
    __device__ static void block(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1,
                                 uint32_t out[4]) {
#pragma unroll
        for (int r = 0; r < 10; ++r) {
            if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
            uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
            uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
            uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
            c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        }
        out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
    }
    __device__ uint32_t at(uint32_t jj) {
        uint32_t b = jj >> 2;
        if (b != blk_id) { block(b, item, stream, 0u, k0, k1, blk); blk_id = b; }
        return blk[jj & 3u];
    }
    __device__ uint32_t next() { return at(j++); }
};
__device__ __forceinline__ float u01(uint32_t x) { return (float)(x >> 8) * 0x1p-24f; }

// ------------------------------------------------------------------ ray / box / triangle
struct Ray {
    f3 o, d;           // origin, direction (not necessarily unit)
    f3 idir, ood;      // 1/d (zero components nudged) and o * idir, for the slab test only
    float tmin, tmax;
};
__device__ __forceinline__ float nudge(float x) { return fabsf(x) < 1e-30f ? copysignf(1e-30f, x) : x; }
__device__ __forceinline__ Ray make_ray(f3 o, f3 d, float tmin, float tmax) {
    Ray r;
    r.o = o; r.d = d; r.tmin = tmin; r.tmax = tmax;
    r.idir = mk3(1.0f / nudge(d.x), 1.0f / nudge(d.y), 1.0f / nudge(d.z));
    r.ood = mk3(o.x * r.idir.x, o.y * r.idir.y, o.z * r.idir.z);
    return r;
}

__device__ __forceinline__ float fmin3(float a, float b, float c) {
    float r;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

// Conservative slab test (boxes are padded at build time).
__device__ __forceinline__ bool slab(const Ray& r, float lox, float hix, float loy, float hiy, float loz,
                                     float hiz, float tlimit, float& tnear) {
    float tx0 = fmaf(lox, r.idir.x, -r.ood.x), tx1 = fmaf(hix, r.idir.x, -r.ood.x);
    float ty0 = fmaf(loy, r.idir.y, -r.ood.y), ty1 = fmaf(hiy, r.idir.y, -r.ood.y);
    float tz0 = fmaf(loz, r.idir.z, -r.ood.z), tz1 = fmaf(hiz, r.idir.z, -r.ood.z);
    float tn = fmax3(fminf(tx0, tx1), fminf(ty0, ty1), fmaxf(fminf(tz0, tz1), r.tmin));
    float tf = fmin3(fmaxf(tx0, tx1), fmaxf(ty0, ty1), fminf(fmaxf(tz0, tz1), tlimit));
    tnear = tn;
    return tn <= tf;
}

// Moller-Trumbore exactly as DESIGN.md §3 O9 (no FMA: -fmad=false TU).
__device__ __forceinline__ bool mt_hit(f3 o, f3 d, float4 a, float4 b, float4 c, float tmin, float tmax, float& t) {
    f3 v0 = xyz(a), e1 = xyz(b), e2 = xyz(c);
    f3 pv = cross(d, e2);
    float det = dot(e1, pv);
    float inv = 1.0f / det;
    f3 s = o - v0;
    float u = dot(s, pv) * inv;
    f3 q = cross(s, e1);
    float v = dot(d, q) * inv;
    t = dot(e2, q) * inv;
    return (det != 0.0f) & (u >= 0.0f) & (u <= 1.0f) & (v >= 0.0f) & ((u + v) <= 1.0f) & (t > tmin) & (t < tmax);
}

// O9 any hit (the V of Eq. 1), division-free (reading R25): the closest-hit
// predicate above with u, v, t scaled by |det| — a_u, a_v, a_t sign-normalised
// by det (exact negations), compared with |det|, tmin*|det|, tmax*|det|.
// The any-hit products are fused multiply-adds in a fixed order (reading R26):
// cross(a,b).x = fma(a.y, b.z, -(a.z*b.y)) (cyclic), dot(a,b) = fma(a.z, b.z,
// fma(a.y, b.y, a.x*b.x)) — one IEEE rounding per fma, identical in the oracle.
__device__ __forceinline__ float dot_fma(f3 a, f3 b) { return __fmaf_rn(a.z, b.z, __fmaf_rn(a.y, b.y, a.x * b.x)); }
__device__ __forceinline__ f3 cross_fma(f3 a, f3 b) {
    return f3{__fmaf_rn(a.y, b.z, -(a.z * b.y)), __fmaf_rn(a.z, b.x, -(a.x * b.z)), __fmaf_rn(a.x, b.y, -(a.y * b.x))};
}

__device__ __forceinline__ bool mt_any(f3 o, f3 d, float4 a, float4 b, float4 c, float tmin, float tmax) {
    f3 v0 = xyz(a), e1 = xyz(b), e2 = xyz(c);
    f3 pv = cross_fma(d, e2);
    float det = dot_fma(e1, pv);
    const unsigned sg = __float_as_uint(det) & 0x80000000u;
    const float adet = fabsf(det);
    f3 s = o - v0;
    float u = __uint_as_float(__float_as_uint(dot_fma(s, pv)) ^ sg);
    f3 q = cross_fma(s, e1);
    float v = __uint_as_float(__float_as_uint(dot_fma(d, q)) ^ sg);
    float t = __uint_as_float(__float_as_uint(dot_fma(e2, q)) ^ sg);
    // u <= |det| is implied by v >= 0 and RN(u + v) <= |det| (see mt_segs)
    return (u >= 0.0f) & (v >= 0.0f) & ((u + v) <= adet) & (t > tmin * adet) & (t < tmax * adet);
}

struct TravStats {
    uint32_t boxes = 0, tris = 0;
    uint32_t wrays = 0, wsteps = 0;  // warp-level packets / iterations (counted on lane 0)
    uint32_t cones = 0, cpk = 0, rpk = 0, chits = 0;  // cone tests, cone / per-ray packets, cache hits
    uint32_t ctests = 0;                              // MT tests in the occluder cache
    uint32_t lists = 0, entries = 0, lfail = 0;       // cluster candidate lists built / their entries / unusable
    uint32_t fsteps = 0;                              // candidate-filter iterations (32 candidates each)
    uint32_t lsteps = 0;                              // traversal steps spent building candidate lists
    uint32_t pculled = 0;                             // box-hit triangles dropped by the plane-side cull (lane-level)
    uint32_t fmt = 0, fmt_hit = 0;                    // filter MT tests (warp-level) / those with a hit
};

// leaf refs: ~((first << 3) | (count - 1)), count in [1, 8]
__device__ __forceinline__ void leaf_range(int node, int& first, int& count) {
    int p = ~node;
    first = p >> 3;
    count = (p & 7) + 1;
}

constexpr int kStack = 128;  // > max tree depth, checked at build time (vpl_build_bvh)
#ifndef VPL_WARP_STACK
#define VPL_WARP_STACK 512
#endif
constexpr int kWarpStack = VPL_WARP_STACK;  // >= 2 * kWide * wide levels, checked at build time (vpl_build_bvh)

// Any hit in (tmin, tmax), one ray per thread.
template <bool kCount>
__device__ __forceinline__ bool bvh_any_hit(const BvhView& bv, const Ray& r, TravStats* st) {
    int stack[kStack];
    int sp = 0;
    int node = bv.root;
    while (true) {
        if (node >= 0) {
            const float4* nd = bv.nodes + 4 * node;
            float4 n0 = __ldg(nd + 0), n1 = __ldg(nd + 1), n2 = __ldg(nd + 2), n3 = __ldg(nd + 3);
            float t0, t1;
            bool h0 = slab(r, n0.x, n0.y, n0.z, n0.w, n2.x, n2.y, r.tmax, t0);
            bool h1 = slab(r, n1.x, n1.y, n1.z, n1.w, n2.z, n2.w, r.tmax, t1);
            if (kCount) st->boxes += 2;
            int c0 = __float_as_int(n3.x), c1 = __float_as_int(n3.y);
            if (h0 && h1) {
                bool first0 = t0 <= t1;
                VPL_DCHECK(sp < kStack);
                stack[sp++] = first0 ? c1 : c0;
                node = first0 ? c0 : c1;
                continue;
            }
            if (h0) { node = c0; continue; }
            if (h1) { node = c1; continue; }
        } else {
            int first, count;
            leaf_range(node, first, count);
            for (int k = 0; k < count; ++k) {
                const float4* tr = bv.tris + 3 * (first + k);
                if (kCount) st->tris += 1;
                if (mt_any(r.o, r.d, __ldg(tr), __ldg(tr + 1), __ldg(tr + 2), r.tmin, r.tmax)) return true;
            }
        }
        if (sp == 0) return false;
        node = stack[--sp];
    }
}

// Closest hit in (tmin, tmax): lexicographic min of (t, original index) (O9, R15).
__device__ __forceinline__ int bvh_closest(const BvhView& bv, const Ray& r, float& t_best) {
    int stack[kStack];
    int sp = 0;
    int node = bv.root;
    int best = -1;
    float tb = r.tmax;
    while (true) {
        if (node >= 0) {
            const float4* nd = bv.nodes + 4 * node;
            float4 n0 = __ldg(nd + 0), n1 = __ldg(nd + 1), n2 = __ldg(nd + 2), n3 = __ldg(nd + 3);
            float t0, t1;
            // ties at t == t_best must still be explored (lowest index wins): tnear <= tb
            bool h0 = slab(r, n0.x, n0.y, n0.z, n0.w, n2.x, n2.y, tb, t0);
            bool h1 = slab(r, n1.x, n1.y, n1.z, n1.w, n2.z, n2.w, tb, t1);
            int c0 = __float_as_int(n3.x), c1 = __float_as_int(n3.y);
            if (h0 && h1) {
                bool first0 = t0 <= t1;
                VPL_DCHECK(sp < kStack);
                stack[sp++] = first0 ? c1 : c0;
                node = first0 ? c0 : c1;
                continue;
            }
            if (h0) { node = c0; continue; }
            if (h1) { node = c1; continue; }
        } else {
            int first, count;
            leaf_range(node, first, count);
            for (int k = 0; k < count; ++k) {
                const float4* tr = bv.tris + 3 * (first + k);
                float4 a = __ldg(tr);
                float t;
                // hit test against the ORIGINAL (tmin, tmax); order against the best so far
                if (mt_hit(r.o, r.d, a, __ldg(tr + 1), __ldg(tr + 2), r.tmin, r.tmax, t)) {
                    int orig = __float_as_int(a.w);
                    if (t < tb || (t == tb && orig < best)) { tb = t; best = orig; }
                }
            }
        }
        if (sp == 0) break;
        node = stack[--sp];
    }
    t_best = tb;
    return best;
}

// unoccluded(a, b) with the eps-shrunk segment (O9) — segment setup shared by
// the per-thread and the warp-cooperative traversals.  seg_ray() leaves the
// slab-test fields (idir, ood) unset: the warp traversal derives them only on
// its per-ray path (with_slab()).
__device__ __forceinline__ bool seg_ray(f3 a, f3 b, float eps, Ray& r) {
    f3 d = b - a;
    float dist = sqrtf(dot(d, d));
    r.o = a;
    const float inv = 1.0f / dist;   // R25: dir = d * (1/dist)
    r.d = mk3(d.x * inv, d.y * inv, d.z * inv);
    r.tmin = eps;
    r.tmax = dist - eps;
    return r.tmax > r.tmin;
}
__device__ __forceinline__ void with_slab(Ray& r) {
    r.idir = mk3(1.0f / nudge(r.d.x), 1.0f / nudge(r.d.y), 1.0f / nudge(r.d.z));
    r.ood = mk3(r.o.x * r.idir.x, r.o.y * r.idir.y, r.o.z * r.idir.z);
}
__device__ __forceinline__ bool segment_ray(f3 a, f3 b, float eps, Ray& r) {
    if (!seg_ray(a, b, eps, r)) return false;
    with_slab(r);
    return true;
}

template <bool kCount>
__device__ __forceinline__ bool segment_occluded(const BvhView& bv, f3 a, f3 b, float eps, TravStats* st) {
    Ray r;
    if (!segment_ray(a, b, eps, r)) return false;
    return bvh_any_hit<kCount>(bv, r, st);
}

struct OccluderCache {
    int own0 = -1, own1 = -1;  // this lane's two most recent occluders (leaf-order triangle index)
    int warp = -1;             // the warp's most recent occluder (uniform)
    bool vis_streak = false;   // last traced segment of this lane was visible (VPL_CACHE_STREAK)
    __device__ __forceinline__ void found(int tri) {
        if (tri != own0) { own1 = own0; own0 = tri; }
    }
};

// warp-wide float min / max (redux.sync .f32, sm_100a): all 32 lanes take part
__device__ __forceinline__ float warp_min_f32(float v) {
    float r;
    asm volatile("redux.sync.min.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
    return r;
}
__device__ __forceinline__ float warp_max_f32(float v) {
    float r;
    asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
    return r;
}

__device__ __forceinline__ int fkey(float f) {   // order-preserving float -> int
    int i = __float_as_int(f);
    return i ^ ((i >> 31) & 0x7FFFFFFF);
}
__device__ __forceinline__ float fkey_inv(int k) { return __int_as_float(k ^ ((k >> 31) & 0x7FFFFFFF)); }

#ifndef VPL_CONE_SPREAD
#define VPL_CONE_SPREAD 0.3f   // 0.3-1.0 measured equal at C4, 1.3% faster than 0.1
#endif
constexpr float kConeSpread = VPL_CONE_SPREAD;  // beam traversal iff max_a (Dmax_a - Dmin_a) < kConeSpread * |D|_min

// Per-ray packet traversal of the 4-wide BVH: every live lane tests its own
// ray against the 4 children; a child is entered if any lane's ray enters it.

// Packet slab test on a wide-node child in centre / half-extent form:
// t = (c - o) * idir -+ e * |idir| per axis — 12 FMA-pipe ops and 5 ALU ops,
// independent of the ray's direction signs (no per-axis min/max).
__device__ __forceinline__ bool slab_ce(const Ray& r, f3 aidir, float cx, float ex, float cy, float ey, float cz,
                                        float ez) {
    float ux = fmaf(cx, r.idir.x, -r.ood.x), vx = ex * aidir.x;
    float uy = fmaf(cy, r.idir.y, -r.ood.y), vy = ey * aidir.y;
    float uz = fmaf(cz, r.idir.z, -r.ood.z), vz = ez * aidir.z;
    float tn = fmax3(ux - vx, uy - vy, fmaxf(uz - vz, r.tmin));
    float tf = fmin3(ux + vx, uy + vy, fminf(uz + vz, r.tmax));
    return tn <= tf;
}


template <bool kCount>
__device__ __forceinline__ bool warp_traverse_ray(const BvhView& bv, Ray r, bool live, bool occl,
                                              OccluderCache& cache, unsigned dir_neg, int* __restrict__ sstack,
                                              TravStats* st) {
    with_slab(r);
    const f3 aidir = mk3(fabsf(r.idir.x), fabsf(r.idir.y), fabsf(r.idir.z));
    int sp = 0;
    int node = bv.root;
    while (true) {
        const bool go = live && !occl;
        if (kCount && (threadIdx.x & 31) == 0) st->wsteps += 1;
        if (node >= 0) {
            const float4* nd = bv.wide4 + kWide4F4 * node;
            float4 cx = __ldg(nd + 0), ex = __ldg(nd + 1), cy = __ldg(nd + 2), ey = __ldg(nd + 3);
            float4 cz = __ldg(nd + 4), ez = __ldg(nd + 5), rf = __ldg(nd + 6), mt = __ldg(nd + 7);
            bool h0 = slab_ce(r, aidir, cx.x, ex.x, cy.x, ey.x, cz.x, ez.x) & go;
            bool h1 = slab_ce(r, aidir, cx.y, ex.y, cy.y, ey.y, cz.y, ez.y) & go;
            bool h2 = slab_ce(r, aidir, cx.z, ex.z, cy.z, ey.z, cz.z, ez.z) & go;
            bool h3 = slab_ce(r, aidir, cx.w, ex.w, cy.w, ey.w, cz.w, ez.w) & go;
            if (kCount && go) st->boxes += 4;
            unsigned lm = (h0 ? 1u : 0u) | (h1 ? 2u : 0u) | (h2 ? 4u : 0u) | (h3 ? 8u : 0u);
            unsigned m = __reduce_or_sync(0xFFFFFFFFu, lm) & (unsigned)__float_as_int(mt.y);  // valid-slot mask
            if (m) {
                int r0 = __float_as_int(rf.x), r1 = __float_as_int(rf.y), r2 = __float_as_int(rf.z),
                    r3 = __float_as_int(rf.w);
                // visit order: stored order (ascending centre along axis), reversed for a -axis packet
                if ((dir_neg >> __float_as_int(mt.x)) & 1u) {
                    m = __brev(m) >> 28;
                    int t0 = r0, t1 = r1;
                    r0 = r3; r1 = r2; r2 = t1; r3 = t0;
                }
                int first = (m & 1u) ? r0 : (m & 2u) ? r1 : (m & 4u) ? r2 : r3;
                unsigned rest = m & (m - 1u);
                // push the later hits, farthest first, so the next in order is on top
                VPL_DCHECK(sp + 3 <= kWarpStack);
                if (rest & 8u) sstack[sp++] = r3;
                if (rest & 4u) sstack[sp++] = r2;
                if (rest & 2u) sstack[sp++] = r1;
                node = first;
                continue;
            }
        } else {
            int first, count;
            leaf_range(node, first, count);
            VPL_DCHECK(first >= 0 && count >= 1 && first + count <= bv.n);
            for (int k = 0; k < count; ++k) {
                const float4* tr = bv.tris + 3 * (first + k);
                float4 a = __ldg(tr), b = __ldg(tr + 1), c = __ldg(tr + 2);
                bool hit = mt_any(r.o, r.d, a, b, c, r.tmin, r.tmax) & go & !occl;
                if (kCount && go && !occl) st->tris += 1;
                if (hit) { occl = true; cache.found(first + k); }
            }
            if (!__any_sync(0xFFFFFFFFu, live && !occl)) break;
        }
        if (sp == 0) break;
        node = sstack[--sp];
    }
    return occl;
}

// O12 — G-buffer record of pixel `pix`: centre-sample pinhole ray,
// closest hit in (0, inf), x = cam + t*dir, front face iff n.dir < 0
__device__ __forceinline__ vpl_gpoint primary_hit(const SceneView& sv, const BvhView& bv, int32_t pix) {
    const SceneHdr* h = sv.hdr;
    const float* c = h->cam;
    int px = pix % h->W, py = pix / h->W;
    f3 pos = ld3(c), fwd = ld3(c + 3), up = ld3(c + 6), right = ld3(c + 9);
    float sx = ((2.0f * ((float)px + 0.5f)) / (float)h->W - 1.0f) * c[12];
    float sy = (1.0f - (2.0f * ((float)py + 0.5f)) / (float)h->H) * c[13];
    f3 d = (fwd + sx * right) + sy * up;
    float len = sqrtf(dot(d, d));
    f3 dir = mk3(d.x / len, d.y / len, d.z / len);
    Ray r = make_ray(pos, dir, 0.0f, __int_as_float(0x7f800000));
    float t;
    int hit = bvh_closest(bv, r, t);
    vpl_gpoint o;
    if (hit < 0) {
        o.pos[0] = o.pos[1] = o.pos[2] = 0.0f;
        o.nrm[0] = o.nrm[1] = o.nrm[2] = 0.0f;
        o.alb[0] = o.alb[1] = o.alb[2] = 0.0f;
        o.tri = -1; o.front = 0; o.t = 0.0f;
    } else {
        f3 x = pos + t * dir;
        float4 n = sv.nrm[hit];
        float4 a = sv.alb[hit];
        o.pos[0] = x.x; o.pos[1] = x.y; o.pos[2] = x.z;
        o.nrm[0] = n.x; o.nrm[1] = n.y; o.nrm[2] = n.z;
        o.alb[0] = a.x; o.alb[1] = a.y; o.alb[2] = a.z;
        o.tri = hit; o.t = t;
        o.front = dot(xyz(n), dir) < 0.0f;
    }
    return o;
}

// tile -> pixel mapping: warp w of a call covers an 8 x bh block (bh = 4, or 8 for the gather with two
// receivers per lane: lane l holds (l % 8, l / 8 + 4k), k = 0, 1)
struct TileMap {
    const int32_t* tiles;
    int32_t n_tiles, tw, th, W, H, tiles_x, blocks_per_tile, bx_per_tile;
    int32_t bh = 4;
    __host__ __device__ int64_t n_warps() const { return (int64_t)n_tiles * blocks_per_tile; }
    // returns the pixel of (warp g, lane, receiver k) or -1 when outside the image
    __device__ __forceinline__ int32_t pixel(int64_t g, int lane, int k = 0) const {
        int32_t ti = (int32_t)(g / blocks_per_tile), sub = (int32_t)(g % blocks_per_tile);
        int32_t t = tiles[ti];
        int32_t tx = t % tiles_x, ty = t / tiles_x;
        int32_t x = tx * tw + (sub % bx_per_tile) * 8 + (lane & 7);
        int32_t yt = (sub / bx_per_tile) * bh + (lane >> 3) + 4 * k;   // row inside the tile
        int32_t y = ty * th + yt;
        return (x < W && y < H && yt < th) ? y * W + x : -1;
    }
};

}  // namespace vplgi
