// bvh.cu — a2 build_bvh: PLOC (parallel locally-ordered clustering, Meister &
// Bittner 2018) over Morton-sorted triangles, then a bottom-up SAH pass that
// collapses small subtrees into leaves of <= 4 triangles, a depth-first
// triangle ordering so every leaf is a contiguous range, and emission of
// 64-byte binary nodes (two child boxes + two child refs).  The paper has no
// acceleration structure; this one only has to make the exact MT visibility
// and closest-hit queries (DESIGN.md §3 O9) fast.  Boxes are padded by
// SceneHdr::box_pad so the slab test is conservative w.r.t. the exact MT test.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <climits>

#include "common.cuh"

namespace vplgi {

#ifndef VPL_PLOC_RADIUS
#define VPL_PLOC_RADIUS 128  // PLOC search radius: vs 64, C4 gather -4.8%, C5 -10%, C3 +2% (+1.2 ms build)
#endif
constexpr int kPlocRadius = VPL_PLOC_RADIUS;
constexpr int kPlocBlock = 256;
constexpr int kPlocBatch = 4;   // PLOC iterations per host round trip
constexpr int kMaxLeaf = 4;
constexpr float kCostTri = 1.0f;   // one exact MT test  (~35 thread-ops)
constexpr float kCostNode = 1.0f;  // one node visit = two slab tests (~34 thread-ops)

__device__ __forceinline__ uint64_t spread21(uint32_t x) {
    uint64_t v = x & 0x1FFFFFu;
    v = (v | (v << 32)) & 0x1F00000000FFFFull;
    v = (v | (v << 16)) & 0x1F0000FF0000FFull;
    v = (v | (v << 8)) & 0x100F00F00F00F00Full;
    v = (v | (v << 4)) & 0x10C30C30C30C30C3ull;
    v = (v | (v << 2)) & 0x1249249249249249ull;
    return v;
}

__global__ void k_morton63(const SceneHdr* __restrict__ h, const float4* __restrict__ cen, int64_t n,
                           uint64_t* __restrict__ keys, uint32_t* __restrict__ idx) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    float4 c = cen[i];
    float q[3] = {c.x, c.y, c.z};
    uint32_t qi[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        float ext = h->bbox_hi[a] - h->bbox_lo[a];
        float s = ext > 0.0f ? 2097152.0f / ext : 0.0f;
        float f = fmaxf((q[a] - h->bbox_lo[a]) * s, 0.0f);
        qi[a] = min((uint32_t)f, 2097151u);
    }
    keys[i] = spread21(qi[0]) | (spread21(qi[1]) << 1) | (spread21(qi[2]) << 2);
    idx[i] = (uint32_t)i;
}

// cluster = (lo.xyz | ref bits, hi.xyz | 0); ref >= 0 internal node, ~p leaf at Morton position p
__global__ void k_leaf_clusters(const SceneHdr* __restrict__ h, const float* __restrict__ verts,
                                const uint32_t* __restrict__ sidx, int64_t n, float4* __restrict__ cl,
                                float4* __restrict__ lbox) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    float pad = h->box_pad;
    const float* v = verts + 9 * (int64_t)sidx[p];
    float lo[3], hi[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        lo[a] = fminf(fminf(v[a], v[3 + a]), v[6 + a]) - pad;
        hi[a] = fmaxf(fmaxf(v[a], v[3 + a]), v[6 + a]) + pad;
    }
    float4 L = make_float4(lo[0], lo[1], lo[2], __int_as_float(~(int)p));
    float4 H = make_float4(hi[0], hi[1], hi[2], 0.0f);
    cl[2 * p] = L; cl[2 * p + 1] = H;
    lbox[2 * p] = L; lbox[2 * p + 1] = H;
}

__device__ __forceinline__ float half_area(float4 lo, float4 hi) {
    float dx = hi.x - lo.x, dy = hi.y - lo.y, dz = hi.z - lo.z;
    return dx * dy + dy * dz + dz * dx;
}
__device__ __forceinline__ float merged_area(float4 alo, float4 ahi, float4 blo, float4 bhi) {
    float dx = fmaxf(ahi.x, bhi.x) - fminf(alo.x, blo.x);
    float dy = fmaxf(ahi.y, bhi.y) - fminf(alo.y, blo.y);
    float dz = fmaxf(ahi.z, bhi.z) - fminf(alo.z, blo.z);
    return dx * dy + dy * dz + dz * dx;
}

// nearest neighbour within +-r in Morton order by merged surface area (ties -> lower index)
// PLOC iterations run in batches without a host round trip: the cluster count
// C and the next free node id live in device memory (double-buffered by
// iteration parity), grids are sized by the last count the host saw (C only
// shrinks), and threads beyond the current C do nothing (flags write 0, so
// the scan over the host bound is exact).
__global__ void __launch_bounds__(kPlocBlock) k_ploc_nn(const float4* __restrict__ cl, const int* __restrict__ dC,
                                                        int* __restrict__ nn) {
    __shared__ float4 slo[kPlocBlock + 2 * kPlocRadius], shi[kPlocBlock + 2 * kPlocRadius];
    const int C = *dC;
    int b0 = blockIdx.x * kPlocBlock;
    if (b0 >= C) return;
    for (int k = threadIdx.x; k < kPlocBlock + 2 * kPlocRadius; k += blockDim.x) {
        int j = b0 - kPlocRadius + k;
        if (j >= 0 && j < C) { slo[k] = cl[2 * j]; shi[k] = cl[2 * j + 1]; }
    }
    __syncthreads();
    int i = b0 + threadIdx.x;
    if (i >= C) return;
    int li = threadIdx.x + kPlocRadius;
    float4 alo = slo[li], ahi = shi[li];
    float best = __int_as_float(0x7f800000);
    int bj = -1;
    int j0 = max(0, i - kPlocRadius), j1 = min(C - 1, i + kPlocRadius);
    for (int j = j0; j <= j1; ++j) {
        if (j == i) continue;
        int lj = j - b0 + kPlocRadius;
        float d = merged_area(alo, ahi, slo[lj], shi[lj]);
        if (d < best) { best = d; bj = j; }   // ascending j: ties keep the lower index
    }
    nn[i] = bj;
}

// flags: bit 32.. = merge (this cluster absorbs nn[i]), bit 0 = keep
__global__ void k_ploc_flags(const int* __restrict__ nn, const int* __restrict__ dC, int Cub,
                             unsigned long long* __restrict__ flags) {
    const int C = *dC;
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= Cub) return;
    if (i >= C) { flags[i] = 0ull; return; }
    int j = nn[i];
    bool mutual = j >= 0 && nn[j] == i;
    unsigned long long merge = (mutual && i < j) ? 1ull : 0ull;
    unsigned long long keep = (mutual && i > j) ? 0ull : 1ull;
    flags[i] = (merge << 32) | keep;
}

__global__ void k_ploc_merge(const float4* __restrict__ cl, const int* __restrict__ nn, const int* __restrict__ dC,
                             const unsigned long long* __restrict__ flags, const unsigned long long* __restrict__ off,
                             const int* __restrict__ dNext, float4* __restrict__ out, int2* __restrict__ child,
                             float4* __restrict__ nbox, int* __restrict__ parent_int, int* __restrict__ parent_leaf,
                             int* __restrict__ dCout, int* __restrict__ dNextOut, int* __restrict__ totals) {
    const int C = *dC, next_id = *dNext;
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= C) return;
    unsigned long long f = flags[i], o = off[i];
    int keep = (int)(f & 1ull), merge = (int)(f >> 32);
    int ko = (int)(o & 0xFFFFFFFFull), mo = (int)(o >> 32);
    if (i == C - 1) {
        totals[0] = ko + keep; totals[1] = mo + merge;
        *dCout = ko + keep;
        *dNextOut = next_id - (mo + merge);
    }
    if (!keep) return;
    float4 alo = cl[2 * i], ahi = cl[2 * i + 1];
    if (!merge) {
        out[2 * ko] = alo; out[2 * ko + 1] = ahi;
        return;
    }
    int j = nn[i];
    float4 blo = cl[2 * j], bhi = cl[2 * j + 1];
    int id = next_id - mo;
    int ra = __float_as_int(alo.w), rb = __float_as_int(blo.w);
    child[id] = make_int2(ra, rb);
    if (ra >= 0) parent_int[ra] = id; else parent_leaf[~ra] = id;
    if (rb >= 0) parent_int[rb] = id; else parent_leaf[~rb] = id;
    float4 L = make_float4(fminf(alo.x, blo.x), fminf(alo.y, blo.y), fminf(alo.z, blo.z), __int_as_float(id));
    float4 H = make_float4(fmaxf(ahi.x, bhi.x), fmaxf(ahi.y, bhi.y), fmaxf(ahi.z, bhi.z), 0.0f);
    nbox[2 * id] = L; nbox[2 * id + 1] = H;
    out[2 * ko] = L; out[2 * ko + 1] = H;
}

// bottom-up: triangle counts and SAH cost; collapse subtrees of <= kMaxLeaf triangles when cheaper
__global__ void k_sah_collapse(int64_t n, const int2* __restrict__ child, const float4* __restrict__ nbox,
                               const float4* __restrict__ lbox, const int* __restrict__ parent_int,
                               const int* __restrict__ parent_leaf, int* __restrict__ flags, int* __restrict__ cnt,
                               float* __restrict__ cost, uint8_t* __restrict__ collapsed, int* __restrict__ icount) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    int node = parent_leaf[p];
    while (node >= 0) {
        __threadfence();
        if (atomicAdd(&flags[node], 1) == 0) return;
        __threadfence();
        int2 c = child[node];
        int cn[2], ci[2];
        float cc[2], ca[2];
        int refs[2] = {c.x, c.y};
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            int r = refs[k];
            if (r >= 0) {
                cn[k] = __ldcg(cnt + r);
                cc[k] = __ldcg(cost + r);
                ci[k] = __ldcg(icount + r);
                ca[k] = half_area(nbox[2 * r], nbox[2 * r + 1]);
            } else {
                cn[k] = 1;
                ci[k] = 0;
                cc[k] = kCostTri;
                ca[k] = half_area(lbox[2 * (~r)], lbox[2 * (~r) + 1]);
            }
        }
        int total = cn[0] + cn[1];
        float an = half_area(nbox[2 * node], nbox[2 * node + 1]);
        float c_int = kCostNode + (an > 0.0f ? (ca[0] * cc[0] + ca[1] * cc[1]) / an : cc[0] + cc[1]);
        float c_leaf = kCostTri * (float)total;
        bool col = total <= kMaxLeaf && c_leaf <= c_int && node != 0;
        __stcg(cnt + node, total);
        __stcg(cost + node, col ? c_leaf : c_int);
        __stcg(icount + node, col ? 0 : 1 + ci[0] + ci[1]);
        collapsed[node] = col;
        node = parent_int[node];
    }
}

// 16-wide collapse by dynamic programming (VPL_WIDE_DP).  The beam traversal
// pays one half-step per visited 16-wide node whatever its fill, and every
// triangle is its own child slot, so the expected traversal cost is
// sum over wide nodes w of A(w) (surface area ~ visit probability) plus a term
// that does not depend on the collapse.  Bottom up over the binary tree:
//   g(n, i) = least cost of covering n's subtree with <= i child slots,
//             a slot being a triangle (cost 0) or a wide node m (cost f(m));
//   f(n)    = A(n) + min_j g(L, j) + g(R, 16 - j)     (n as a wide node);
//   g(n, 1) = f(n) (inner) or 0 (leaf);  g(n, i) = min(g(n, i-1), min_j g(L, j) + g(R, i - j)).
// choice[n][i] = 0 when g(n, i) = g(n, i - 1), else the split j; choice[n][0] = the split of f(n).
__global__ void k_wide_dp(int64_t n, const int2* __restrict__ child, const float4* __restrict__ nbox,
                          const int* __restrict__ parent_int, const int* __restrict__ parent_leaf,
                          int* __restrict__ flags, float* __restrict__ g, uint8_t* __restrict__ choice) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    int node = parent_leaf[p];
    while (node >= 0) {
        __threadfence();
        if (atomicAdd(&flags[node], 1) == 0) return;
        __threadfence();
        const int2 c = child[node];
        float gl[kWide + 1], gr[kWide + 1];
#pragma unroll
        for (int i = 1; i <= kWide; ++i) {
            gl[i] = c.x >= 0 ? __ldcg(g + (int64_t)c.x * kWide + (i - 1)) : 0.0f;
            gr[i] = c.y >= 0 ? __ldcg(g + (int64_t)c.y * kWide + (i - 1)) : 0.0f;
        }
        uint8_t ch[kWide + 1];
        float best16 = 3.0e38f;
        int j16 = 1;
        for (int j = 1; j < kWide; ++j) {
            const float v = gl[j] + gr[kWide - j];
            if (v < best16) { best16 = v; j16 = j; }
        }
        const float f = half_area(nbox[2 * node], nbox[2 * node + 1]) + best16;
        ch[0] = (uint8_t)j16;
        float prev = f;
        __stcg(g + (int64_t)node * kWide + 0, f);
        ch[1] = 0;
        for (int i = 2; i <= kWide; ++i) {
            float bi = 3.0e38f;
            int ji = 1;
            for (int j = 1; j < i; ++j) {
                const float v = gl[j] + gr[i - j];
                if (v < bi) { bi = v; ji = j; }
            }
            if (prev <= bi) { ch[i] = 0; } else { ch[i] = (uint8_t)ji; prev = bi; }
            __stcg(g + (int64_t)node * kWide + (i - 1), prev);
        }
        for (int i = 0; i <= kWide; ++i) choice[(int64_t)node * (kWide + 1) + i] = ch[i];
        node = parent_int[node];
    }
}

// slots of wide node b from the DP choices: (node, i) pairs on a small stack
__global__ void k_wide_expand_dp(const int* __restrict__ F, int nF, const int2* __restrict__ child,
                                 const uint8_t* __restrict__ choice, int* __restrict__ exp, int* __restrict__ nint) {
    int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= nF) return;
    const int b = F[f];
    int st_n[2 * kWide], st_i[2 * kWide];
    int sp = 0, cntc = 0, ni = 0;
    const int2 cb = child[b];
    const int j0 = choice[(int64_t)b * (kWide + 1) + 0];
    st_n[sp] = cb.y; st_i[sp++] = kWide - j0;
    st_n[sp] = cb.x; st_i[sp++] = j0;
    while (sp > 0) {
        const int nd = st_n[--sp];
        int i = st_i[sp];
        if (nd < 0 || i == 1) {             // a triangle, or an inner node that becomes a wide node
            exp[f * kWide + cntc++] = nd;
            ni += nd >= 0;
            continue;
        }
        const uint8_t* cn = choice + (int64_t)nd * (kWide + 1);
        while (i > 1 && cn[i] == 0) --i;    // fewer slots cover it at the same cost
        if (i == 1) { exp[f * kWide + cntc++] = nd; ++ni; continue; }
        const int j = cn[i];
        const int2 cc = child[nd];
        st_n[sp] = cc.y; st_i[sp++] = i - j;
        st_n[sp] = cc.x; st_i[sp++] = j;
    }
    for (int k = cntc; k < kWide; ++k) exp[f * kWide + k] = INT_MIN;
    nint[f] = ni;
}

// depth-first triangle offset of every node (leaves: index ~p -> slot n-1+p)
__global__ void k_dfs_offsets(int64_t n, const int2* __restrict__ child, const int* __restrict__ parent_int,
                              const int* __restrict__ parent_leaf, const int* __restrict__ cnt, int* __restrict__ off,
                              int* __restrict__ max_depth, const int* __restrict__ icount,
                              const uint8_t* __restrict__ collapsed, int* __restrict__ pre, uint8_t* __restrict__ hidden) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= 2 * n - 1) return;
    int self = k < n - 1 ? (int)k : ~(int)(k - (n - 1));
    int node = self;
    int par = node >= 0 ? parent_int[node] : parent_leaf[~node];
    int o = 0, depth = 0, pr = 0;
    bool hid = false;
    while (par >= 0) {
        int2 c = child[par];
        if (c.y == node) {
            o += c.x >= 0 ? cnt[c.x] : 1;
            pr += c.x >= 0 ? icount[c.x] : 0;
        }
        pr += 1;
        hid |= collapsed[par] != 0;
        node = par;
        par = parent_int[node];
        ++depth;
    }
    off[k] = o;
    if (self < 0) atomicMax(max_depth, depth);
    else { pre[self] = pr; hidden[self] = hid; }
}

__device__ __forceinline__ int leaf_ref(int first, int count) { return ~((first << 3) | (count - 1)); }

__global__ void k_emit_nodes(int64_t n, const int2* __restrict__ child, const float4* __restrict__ nbox,
                             const float4* __restrict__ lbox, const int* __restrict__ cnt, const int* __restrict__ off,
                             const uint8_t* __restrict__ collapsed, const int* __restrict__ pre,
                             const uint8_t* __restrict__ hidden, float4* __restrict__ nodes) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n - 1 || collapsed[i] || hidden[i]) return;
    int2 c = child[i];
    int refs[2] = {c.x, c.y};
    float4 lo[2], hi[2];
    int out[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        int r = refs[k];
        if (r >= 0) {
            lo[k] = nbox[2 * r]; hi[k] = nbox[2 * r + 1];
            out[k] = collapsed[r] ? leaf_ref(off[r], cnt[r]) : pre[r];
        } else {
            lo[k] = lbox[2 * (~r)]; hi[k] = lbox[2 * (~r) + 1];
            out[k] = leaf_ref(off[(n - 1) + (~r)], 1);
        }
    }
    // order children along the axis of largest centre separation (child 0 = lower centre) and
    // store that axis in n3.z: packet traversal visits child 0 first iff the packet travels +axis
    float dc[3] = {(lo[1].x + hi[1].x) - (lo[0].x + hi[0].x), (lo[1].y + hi[1].y) - (lo[0].y + hi[0].y),
                   (lo[1].z + hi[1].z) - (lo[0].z + hi[0].z)};
    int axis = 0;
    if (fabsf(dc[1]) > fabsf(dc[axis])) axis = 1;
    if (fabsf(dc[2]) > fabsf(dc[axis])) axis = 2;
    if (dc[axis] < 0.0f) {
        float4 tl = lo[0], th = hi[0];
        lo[0] = lo[1]; hi[0] = hi[1]; lo[1] = tl; hi[1] = th;
        int to = out[0]; out[0] = out[1]; out[1] = to;
    }
    int64_t s = pre[i];  // depth-first preorder slot (root = 0, first child adjacent)
    nodes[4 * s + 0] = make_float4(lo[0].x, hi[0].x, lo[0].y, hi[0].y);
    nodes[4 * s + 1] = make_float4(lo[1].x, hi[1].x, lo[1].y, hi[1].y);
    nodes[4 * s + 2] = make_float4(lo[0].z, hi[0].z, lo[1].z, hi[1].z);
    nodes[4 * s + 3] = make_float4(__int_as_float(out[0]), __int_as_float(out[1]), __int_as_float(axis), 0.0f);
}


// ---------------------------------------------------------------- kWide-wide collapse (BFS levels)
__device__ __forceinline__ bool is_inner(int r, const uint8_t* __restrict__ collapsed) { return r >= 0 && !collapsed[r]; }
// The 16-wide (cone) tree opens the SAH leaves too: its leaves are single
// triangles, each with its own box tested against the packet cone in
// parallel with its siblings, so the per-lane exact MT tests only run on
// triangles the cone can reach.  (The 4-wide per-ray tree keeps the SAH leaves.)
template <int kW>
__device__ __forceinline__ bool is_inner_w(int r, const uint8_t* __restrict__ collapsed) {
    return kW == kWide ? r >= 0 : is_inner(r, collapsed);
}

__device__ __forceinline__ void ref_box(int r, const float4* __restrict__ nbox, const float4* __restrict__ lbox,
                                        float4& lo, float4& hi) {
    if (r >= 0) { lo = nbox[2 * r]; hi = nbox[2 * r + 1]; }
    else { lo = lbox[2 * (~r)]; hi = lbox[2 * (~r) + 1]; }
}

// greedy: open the inner child of largest surface area until kWide children
#ifndef VPL_WIDE_DP
#define VPL_WIDE_DP 0     // 1: the 16-wide collapse by dynamic programming (least total wide-node area)
#endif
#ifndef VPL_WIDE_SMALL
#define VPL_WIDE_SMALL 2   // absorb inner children of <= 2 triangles first (C4: -0.7%)
#endif
#ifndef VPL_WIDE_OPEN
#define VPL_WIDE_OPEN 0   // 16-wide collapse opens the inner child of 0: largest area, 1: most triangles, 2: area x triangles
#endif
template <int kW>
__global__ void k_wide_expand(const int* __restrict__ F, int nF, const int2* __restrict__ child,
                              const float4* __restrict__ nbox, const uint8_t* __restrict__ collapsed,
                              const int* __restrict__ cnt, int* __restrict__ exp, int* __restrict__ nint) {
    int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= nF) return;
    int b = F[f];
    int ref[kW];
    int2 c = child[b];
    ref[0] = c.x; ref[1] = c.y;
    int cntc = 2;
    while (cntc < kW) {
        int best = -1;
        float ba = -1.0f;
        for (int k = 0; k < cntc; ++k)
            if (is_inner_w<kW>(ref[k], collapsed)) {
                float a = half_area(nbox[2 * ref[k]], nbox[2 * ref[k] + 1]);
                if (kW == kWide && VPL_WIDE_OPEN == 1) a = (float)cnt[ref[k]];
                if (kW == kWide && VPL_WIDE_OPEN == 2) a *= (float)cnt[ref[k]];
                // absorb small subtrees first: an inner child of <= VPL_WIDE_SMALL triangles is opened
                // before any large one, so it never becomes a nearly empty wide node of its own
                if (kW == kWide && VPL_WIDE_SMALL > 0 && cnt[ref[k]] <= VPL_WIDE_SMALL) a = 3.0e38f;
                if (a > ba) { ba = a; best = k; }
            }
        if (best < 0) break;
        int2 cc = child[ref[best]];
        ref[best] = cc.x;
        ref[cntc++] = cc.y;
    }
    int ni = 0;
    for (int k = 0; k < kW; ++k) {
        int r = k < cntc ? ref[k] : INT_MIN;
        exp[f * kW + k] = r;
        ni += (k < cntc && is_inner_w<kW>(r, collapsed)) ? 1 : 0;
    }
    nint[f] = ni;
}

__global__ void k_wide_write(const int* __restrict__ F, int nF, const int* __restrict__ exp,
                             const int* __restrict__ nint, const int* __restrict__ noff, int base_cur, int base_next,
                             const float4* __restrict__ nbox, const float4* __restrict__ lbox,
                             const uint8_t* __restrict__ collapsed, const int* __restrict__ cnt,
                             const int* __restrict__ toff, int64_t n, int* __restrict__ Fnext, float4* __restrict__ wide,
                             int* __restrict__ total) {
    int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= nF) return;
    if (f == nF - 1) *total = noff[f] + nint[f];
    int b = F[f];
    float4 L = nbox[2 * b], H = nbox[2 * b + 1];
    float ex = H.x - L.x, ey = H.y - L.y, ez = H.z - L.z;
    int axis = (ex >= ey && ex >= ez) ? 0 : (ey >= ez ? 1 : 2);
    int ref[kWide];
    float key[kWide];
    int cntc = 0;
    for (int k = 0; k < kWide; ++k) {
        int r = exp[f * kWide + k];
        if (r == INT_MIN) continue;
        float4 lo, hi;
        ref_box(r, nbox, lbox, lo, hi);
        ref[cntc] = r;
        key[cntc] = axis == 0 ? lo.x + hi.x : axis == 1 ? lo.y + hi.y : lo.z + hi.z;
        ++cntc;
    }
    // insertion sort by centre along axis (stable)
    for (int i = 1; i < cntc; ++i)
        for (int j = i; j > 0 && key[j] < key[j - 1]; --j) {
            float tk = key[j]; key[j] = key[j - 1]; key[j - 1] = tk;
            int tr = ref[j]; ref[j] = ref[j - 1]; ref[j - 1] = tr;
        }
    float4* w = wide + (int64_t)kWideF4 * (base_cur + f);
    int j = 0;
    for (int k = 0; k < kWide; ++k) {
        if (k >= cntc) {
            w[2 * k] = make_float4(0.0f, 0.0f, 0.0f, __int_as_float(INT_MIN));
            w[2 * k + 1] = make_float4(0.0f, 0.0f, 0.0f, __int_as_float(axis));
            continue;
        }
        int r = ref[k];
        float4 lo, hi;
        ref_box(r, nbox, lbox, lo, hi);
        int out;
        if (is_inner_w<kWide>(r, collapsed)) {
            int slot = noff[f] + j++;
            Fnext[slot] = r;
            out = base_next + slot;
        } else {
            out = leaf_ref(toff[(n - 1) + (~r)], 1);
        }
        w[2 * k] = make_float4(lo.x, lo.y, lo.z, __int_as_float(out));
        w[2 * k + 1] = make_float4(hi.x, hi.y, hi.z, __int_as_float(axis));
    }
}

__global__ void k_wide4_write(const int* __restrict__ F, int nF, const int* __restrict__ exp,
                             const int* __restrict__ nint, const int* __restrict__ noff, int base_cur, int base_next,
                             const float4* __restrict__ nbox, const float4* __restrict__ lbox,
                             const uint8_t* __restrict__ collapsed, const int* __restrict__ cnt,
                             const int* __restrict__ toff, int64_t n, int* __restrict__ Fnext, float4* __restrict__ wide,
                             int* __restrict__ total) {
    int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= nF) return;
    if (f == nF - 1) *total = noff[f] + nint[f];
    int b = F[f];
    float4 L = nbox[2 * b], H = nbox[2 * b + 1];
    float ex = H.x - L.x, ey = H.y - L.y, ez = H.z - L.z;
    int axis = (ex >= ey && ex >= ez) ? 0 : (ey >= ez ? 1 : 2);
    int ref[kWide4];
    float key[kWide4];
    float4 lo[kWide4], hi[kWide4];
    int cntc = 0;
    for (int k = 0; k < kWide4; ++k) {
        int r = exp[f * kWide4 + k];
        if (r == INT_MIN) continue;
        ref[cntc] = r;
        ref_box(r, nbox, lbox, lo[cntc], hi[cntc]);
        key[cntc] = axis == 0 ? lo[cntc].x + hi[cntc].x : axis == 1 ? lo[cntc].y + hi[cntc].y : lo[cntc].z + hi[cntc].z;
        ++cntc;
    }
    // insertion sort by centre along axis (stable)
    for (int i = 1; i < cntc; ++i)
        for (int j = i; j > 0 && key[j] < key[j - 1]; --j) {
            float tk = key[j]; key[j] = key[j - 1]; key[j - 1] = tk;
            int tr = ref[j]; ref[j] = ref[j - 1]; ref[j - 1] = tr;
            float4 tl = lo[j]; lo[j] = lo[j - 1]; lo[j - 1] = tl;
            float4 th = hi[j]; hi[j] = hi[j - 1]; hi[j - 1] = th;
        }
    float q[6][kWide4];
    int out[kWide4];
    int j = 0;
    // centre / half-extent form (packet slab test on the FMA pipe); the half extent is
    // widened by 2^-20 * max|coord| so rounding of c and e keeps the box conservative.
    // Empty slots are masked by the child count stored in the meta word.
    for (int k = 0; k < kWide4; ++k) {
        if (k >= cntc) {
            for (int a = 0; a < 6; ++a) q[a][k] = 0.0f;
            out[k] = INT_MIN;
            continue;
        }
        int r = ref[k];
        float l3[3] = {lo[k].x, lo[k].y, lo[k].z}, h3[3] = {hi[k].x, hi[k].y, hi[k].z};
        for (int a = 0; a < 3; ++a) {
            float m = fmaxf(fabsf(l3[a]), fabsf(h3[a]));
            q[2 * a][k] = 0.5f * (l3[a] + h3[a]);
            q[2 * a + 1][k] = 0.5f * (h3[a] - l3[a]) + m * 0x1p-20f;
        }
        if (is_inner(r, collapsed)) {
            int slot = noff[f] + j++;
            Fnext[slot] = r;
            out[k] = base_next + slot;
        } else if (r >= 0) {
            out[k] = leaf_ref(toff[r], cnt[r]);
        } else {
            out[k] = leaf_ref(toff[(n - 1) + (~r)], 1);
        }
    }
    float4* w = wide + (int64_t)kWide4F4 * (base_cur + f);
    for (int a = 0; a < 6; ++a)
        for (int k = 0; k < kWide4; k += 4) w[a * (kWide4 / 4) + k / 4] = make_float4(q[a][k], q[a][k + 1], q[a][k + 2], q[a][k + 3]);
    for (int k = 0; k < kWide4; k += 4)
        w[6 * (kWide4 / 4) + k / 4] = make_float4(__int_as_float(out[k]), __int_as_float(out[k + 1]),
                                                 __int_as_float(out[k + 2]), __int_as_float(out[k + 3]));
    w[kWide4F4 - 1] = make_float4(__int_as_float(axis), __int_as_float((1 << cntc) - 1), 0.0f, 0.0f);  // axis, valid-slot mask
}


__global__ void k_emit_tris(const float* __restrict__ verts, const uint32_t* __restrict__ sidx, int64_t n,
                            const int* __restrict__ off, float4* __restrict__ tris, float4* __restrict__ planes) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    uint32_t t = sidx[p];
    int slot = n > 1 ? off[(n - 1) + p] : 0;
    const float* v = verts + 9 * (int64_t)t;
    f3 v0 = ld3(v), e1 = ld3(v + 3) - v0, e2 = ld3(v + 6) - v0;
    tris[3 * slot + 0] = make_float4(v0.x, v0.y, v0.z, __int_as_float((int)t));
    tris[3 * slot + 1] = make_float4(e1.x, e1.y, e1.z, 0.0f);
    tris[3 * slot + 2] = make_float4(e2.x, e2.y, e2.z, 0.0f);
    // plane of the triangle MT sees, (v0, v0 + e1, v0 + e2), in float64 and rounded once: unit normal
    // n and offset n.v0 (the gather's plane-side cull evaluates f(p) = n.p - offset; a zero-area
    // triangle gets the null plane, which never culls)
    const double nx = (double)e1.y * e2.z - (double)e1.z * e2.y, ny = (double)e1.z * e2.x - (double)e1.x * e2.z,
                 nz = (double)e1.x * e2.y - (double)e1.y * e2.x;
    const double len = sqrt(nx * nx + ny * ny + nz * nz);
    const double il = len > 0.0 ? 1.0 / len : 0.0;
    planes[slot] = make_float4((float)(nx * il), (float)(ny * il), (float)(nz * il),
                               (float)((nx * v0.x + ny * v0.y + nz * v0.z) * il));
}

struct BuildWork {
    uint64_t *keys, *keys2;
    uint32_t *idx, *idx2;
    float4 *clA, *clB, *lbox, *nbox;
    int *nn, *parent_int, *parent_leaf, *flags, *cnt, *off, *totals, *icount, *pre;
    uint8_t* hidden;
    int *F0, *F1, *wexp, *nint, *noff;
    float* dpg;
    uint8_t* dpc;
    unsigned long long *mflags, *moff;
    float* cost;
    uint8_t* collapsed;
    int2* child;
    void* cub;
    size_t cub_bytes;
};

static size_t build_layout(int64_t n, char* base, BuildWork* w) {
    Bump b{base};
    w->keys = b.take<uint64_t>(n);
    w->keys2 = b.take<uint64_t>(n);
    w->idx = b.take<uint32_t>(n);
    w->idx2 = b.take<uint32_t>(n);
    w->clA = b.take<float4>(2 * n);
    w->clB = b.take<float4>(2 * n);
    w->lbox = b.take<float4>(2 * n);
    w->nbox = b.take<float4>(2 * n);
    w->nn = b.take<int>(n);
    w->parent_int = b.take<int>(n);
    w->parent_leaf = b.take<int>(n);
    w->flags = b.take<int>(n);
    w->cnt = b.take<int>(n);
    w->off = b.take<int>(2 * n);
    w->totals = b.take<int>(8);
    w->mflags = b.take<unsigned long long>(n);
    w->moff = b.take<unsigned long long>(n);
    w->cost = b.take<float>(n);
    w->collapsed = b.take<uint8_t>(n);
    w->icount = b.take<int>(n);
    w->pre = b.take<int>(n);
    w->hidden = b.take<uint8_t>(n);
    w->F0 = b.take<int>(n);
    w->F1 = b.take<int>(n);
    w->wexp = b.take<int>((size_t)kWide * n);
    w->dpg = b.take<float>(VPL_WIDE_DP ? (size_t)kWide * n : 1);
    w->dpc = b.take<uint8_t>(VPL_WIDE_DP ? (size_t)(kWide + 1) * n : 1);
    w->nint = b.take<int>(n);
    w->noff = b.take<int>(n);
    w->child = b.take<int2>(n);
    size_t c1 = 0, c2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, c1, (uint64_t*)nullptr, (uint64_t*)nullptr, (uint32_t*)nullptr,
                                    (uint32_t*)nullptr, (int)n, 0, 64);
    cub::DeviceScan::ExclusiveSum(nullptr, c2, (unsigned long long*)nullptr, (unsigned long long*)nullptr, (int)n);
    size_t c3 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, c3, (int*)nullptr, (int*)nullptr, (int)n);
    w->cub_bytes = c1 > c2 ? c1 : c2;
    if (c3 > w->cub_bytes) w->cub_bytes = c3;
    w->cub = b.take<char>(w->cub_bytes);
    return b.off;
}

static inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t); }

}  // namespace vplgi

using namespace vplgi;

extern "C" {

int32_t vpl_bvh_bytes(int64_t n_tris, size_t* bvh_bytes, size_t* work_bytes) {
    if (!bvh_bytes || !work_bytes || n_tris <= 0 || n_tris > (int64_t)1 << 28) return VPL_EINVAL;
    *bvh_bytes = bvh_layout(n_tris, nullptr);
    BuildWork w;
    *work_bytes = build_layout(n_tris, nullptr, &w);
    return VPL_OK;
}

int32_t vpl_build_bvh(const void* d_scene, void* d_bvh, size_t bvh_bytes, void* d_work, size_t work_bytes,
                      void* stream) {
    if (!d_scene || !d_bvh || !d_work) { set_error("vpl_build_bvh: null pointer"); return VPL_EINVAL; }
    cudaStream_t s = (cudaStream_t)stream;
    SceneHdr hh;
    VPL_TRY(read_scene_hdr(d_scene, s, &hh));
    const int64_t n = hh.n;
    size_t nb = 0, wb = 0;
    VPL_TRY(vpl_bvh_bytes(n, &nb, &wb));
    if (bvh_bytes < nb || work_bytes < wb) { set_error("vpl_build_bvh: buffers too small"); return VPL_ESMALL; }
    SceneView sv = scene_view(d_scene, n);
    BvhHdr bh;
    bvh_layout(n, &bh);
    VPL_CUDA(cudaMemcpyAsync(d_bvh, &bh, sizeof(bh), cudaMemcpyHostToDevice, s));
    float4* nodes = (float4*)((char*)d_bvh + bh.off_nodes);
    float4* tris = (float4*)((char*)d_bvh + bh.off_tris);
    BuildWork w;
    build_layout(n, (char*)d_work, &w);

    // Morton order of centroids over the scene box
    k_morton63<<<nblk(n, 256), 256, 0, s>>>(sv.hdr, sv.cen, n, w.keys, w.idx);
    VPL_LAUNCHED("k_morton63");
    size_t cb = w.cub_bytes;
    VPL_CUDA(cub::DeviceRadixSort::SortPairs(w.cub, cb, w.keys, w.keys2, w.idx, w.idx2, (int)n, 0, 64, s));
    k_leaf_clusters<<<nblk(n, 256), 256, 0, s>>>(sv.hdr, sv.verts, w.idx2, n, w.clA, w.lbox);
    VPL_LAUNCHED("k_leaf_clusters");

    if (n > 1) {
        // PLOC: merge mutual nearest neighbours until one cluster is left, kPlocBatch
        // iterations per host round trip (counts double-buffered in w.totals[4..7])
        int C = (int)n;
        float4 *cur = w.clA, *nxt = w.clB;
        VPL_CUDA(cudaMemsetAsync(w.parent_int, 0xFF, sizeof(int) * n, s));
        int init[4] = {(int)n, (int)n, (int)n - 2, (int)n - 2};   // C[0], C[1], next[0], next[1]
        VPL_CUDA(cudaMemcpyAsync(w.totals + 4, init, sizeof(init), cudaMemcpyHostToDevice, s));
        int* dC = w.totals + 4;      // dC[it & 1] = clusters entering iteration it
        int* dN = w.totals + 6;      // dN[it & 1] = next free node id entering iteration it
        int it = 0;
        while (C > 1) {
            const int Cub = C;
            for (int b = 0; b < kPlocBatch; ++b, ++it) {
                const int pi = it & 1, po = pi ^ 1;
                k_ploc_nn<<<nblk(Cub, kPlocBlock), kPlocBlock, 0, s>>>(cur, dC + pi, w.nn);
                VPL_LAUNCHED("k_ploc_nn");
                k_ploc_flags<<<nblk(Cub, 256), 256, 0, s>>>(w.nn, dC + pi, Cub, w.mflags);
                VPL_LAUNCHED("k_ploc_flags");
                cb = w.cub_bytes;
                VPL_CUDA(cub::DeviceScan::ExclusiveSum(w.cub, cb, w.mflags, w.moff, Cub, s));
                k_ploc_merge<<<nblk(Cub, 256), 256, 0, s>>>(cur, w.nn, dC + pi, w.mflags, w.moff, dN + pi, nxt, w.child,
                                                            w.nbox, w.parent_int, w.parent_leaf, dC + po, dN + po,
                                                            w.totals);
                VPL_LAUNCHED("k_ploc_merge");
                float4* t = cur; cur = nxt; nxt = t;
            }
            int cnow = 0;
            VPL_CUDA(cudaMemcpyAsync(&cnow, dC + (it & 1), sizeof(int), cudaMemcpyDeviceToHost, s));
            VPL_CUDA(cudaStreamSynchronize(s));
            if (cnow >= C && C > 1) { set_error("vpl_build_bvh: PLOC made no progress"); return VPL_ECUDA; }
            C = cnow;
        }
        // a finished batch may have run idle iterations (C = 1): they copy the root
        // cluster between the ping-pong buffers and change nothing else
        // SAH collapse, depth-first ordering, emission
        VPL_CUDA(cudaMemsetAsync(w.flags, 0, sizeof(int) * n, s));
        k_sah_collapse<<<nblk(n, 256), 256, 0, s>>>(n, w.child, w.nbox, w.lbox, w.parent_int, w.parent_leaf, w.flags,
                                                    w.cnt, w.cost, w.collapsed, w.icount);
        VPL_LAUNCHED("k_sah_collapse");
#if VPL_WIDE_DP
        VPL_CUDA(cudaMemsetAsync(w.flags, 0, sizeof(int) * n, s));
        k_wide_dp<<<nblk(n, 128), 128, 0, s>>>(n, w.child, w.nbox, w.parent_int, w.parent_leaf, w.flags, w.dpg, w.dpc);
        VPL_LAUNCHED("k_wide_dp");
#endif
        VPL_CUDA(cudaMemsetAsync(w.totals + 2, 0, sizeof(int), s));
        k_dfs_offsets<<<nblk(2 * n - 1, 256), 256, 0, s>>>(n, w.child, w.parent_int, w.parent_leaf, w.cnt, w.off,
                                                           w.totals + 2, w.icount, w.collapsed, w.pre, w.hidden);
        VPL_LAUNCHED("k_dfs_offsets");
        k_emit_nodes<<<nblk(n - 1, 256), 256, 0, s>>>(n, w.child, w.nbox, w.lbox, w.cnt, w.off, w.collapsed, w.pre,
                                                       w.hidden, nodes);
        VPL_LAUNCHED("k_emit_nodes");
        // wide nodes for the packet traversals, breadth-first from the root
        for (int fmt = 0; fmt < 2; ++fmt) {
            float4* wide = (float4*)((char*)d_bvh + (fmt == 0 ? bh.off_wide : bh.off_wide4));
            int zero = 0;
            VPL_CUDA(cudaMemcpyAsync(w.F0, &zero, sizeof(int), cudaMemcpyHostToDevice, s));
            int nF = 1, base = 0, levels = 0;
            int *Fc = w.F0, *Fn = w.F1;
            while (nF > 0) {
                ++levels;
                if (fmt == 0 && VPL_WIDE_DP)
                    k_wide_expand_dp<<<nblk(nF, 128), 128, 0, s>>>(Fc, nF, w.child, w.dpc, w.wexp, w.nint);
                else if (fmt == 0) k_wide_expand<kWide><<<nblk(nF, 128), 128, 0, s>>>(Fc, nF, w.child, w.nbox, w.collapsed,
                                                                              w.cnt, w.wexp, w.nint);
                else k_wide_expand<kWide4><<<nblk(nF, 128), 128, 0, s>>>(Fc, nF, w.child, w.nbox, w.collapsed,
                                                                         w.cnt, w.wexp, w.nint);
                VPL_LAUNCHED("k_wide_expand");
                cb = w.cub_bytes;
                VPL_CUDA(cub::DeviceScan::ExclusiveSum(w.cub, cb, w.nint, w.noff, nF, s));
                if (fmt == 0) k_wide_write<<<nblk(nF, 128), 128, 0, s>>>(Fc, nF, w.wexp, w.nint, w.noff, base, base + nF,
                                                                       w.nbox, w.lbox, w.collapsed, w.cnt, w.off, n,
                                                                       Fn, wide, w.totals + 3);
                else k_wide4_write<<<nblk(nF, 128), 128, 0, s>>>(Fc, nF, w.wexp, w.nint, w.noff, base, base + nF,
                                                                  w.nbox, w.lbox, w.collapsed, w.cnt, w.off, n, Fn,
                                                                  wide, w.totals + 3);
                VPL_LAUNCHED("k_wide_write");
                int next = 0;
                VPL_CUDA(cudaMemcpyAsync(&next, w.totals + 3, sizeof(int), cudaMemcpyDeviceToHost, s));
                VPL_CUDA(cudaStreamSynchronize(s));
                base += nF;
                nF = next;
                int* t = Fc; Fc = Fn; Fn = t;
            }
            int per_level = fmt == 0 ? 2 * kWide : kWide4 - 1;   // the cone traversal expands two nodes per step
            if (per_level * levels > kWarpStack) {
                set_error("vpl_build_bvh: %d wide levels exceed the packet stack (%d)", levels, kWarpStack);
                return VPL_ECUDA;
            }
        }
    }
    k_emit_tris<<<nblk(n, 256), 256, 0, s>>>(sv.verts, w.idx2, n, w.off, tris, (float4*)((char*)d_bvh + bh.off_planes));
    VPL_LAUNCHED("k_emit_tris");
    if (n > 1) {
        int depth = 0;
        VPL_CUDA(cudaMemcpyAsync(&depth, w.totals + 2, sizeof(int), cudaMemcpyDeviceToHost, s));
        VPL_CUDA(cudaStreamSynchronize(s));
        if (depth >= kStack) {
            set_error("vpl_build_bvh: tree depth %d exceeds the traversal stack (%d)", depth, kStack);
            return VPL_ECUDA;
        }
    }
    return VPL_OK;
}

}  // extern "C"
