// render.cu — a7 render_gbuffer (O12), a8 gather_indirect (Eq. 1, O13) and
// the test hooks that share their traversal code.
#include <cub/device/device_radix_sort.cuh>

#include "gather.cuh"

namespace vplgi {

constexpr double kPiR = 3.14159265358979323846;

// O12 — centre-sample pinhole ray, closest hit
__global__ void k_gbuffer(SceneView sv, BvhView bv, TileMap tm, vpl_gpoint* __restrict__ gb) {
    int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (g >= tm.n_warps()) return;
    int32_t pix = tm.pixel(g, lane);
    if (pix < 0) return;
    gb[pix] = primary_hit(sv, bv, pix);
}

// a8 — Eq. 1 gather.  Persistent: each warp takes work items —
// an 8x4 pixel block x a chunk of the Morton-ordered VPL copy — from an
// atomic queue; all lanes walk the chunk's VPLs in the same order, so the
// shadow segments of a warp form a narrow beam (gather.cuh).  fp32 two-level
// accumulation: a per-batch partial is folded into the chunk total every 256
// VPLs; the chunk totals of a block are folded in chunk order by the warp
// that finishes the block's last chunk.
// VPL clusters: 32 consecutive VPLs of the Morton-ordered copy, bounded by
// their position box and normal box (4 float4: ylo, yhi, nlo, nhi).  A lane
// can trace some VPL of the cluster only if cx = n_x.(y - x) > 0 and
// ci = n_i.(x - y) > 0 are both possible over the boxes; the bounds are
// evaluated with a relative margin far above the fp32 rounding of O13's cull,
// so a skipped cluster holds no traced pair (the image is unchanged bitwise).
#ifndef VPL_CLUSTER
#define VPL_CLUSTER 32
#endif
constexpr int kCluster = VPL_CLUSTER;   // VPLs per culling cluster (divides 256)
__device__ __forceinline__ bool cluster_may_trace(const float4* __restrict__ cb, f3 x, f3 nx) {
    const float4 ylo = __ldg(cb), yhi = __ldg(cb + 1), nlo = __ldg(cb + 2), nhi = __ldg(cb + 3);
    // max over y in the box of n_x.(y - x): per axis the larger of n*(lo - x), n*(hi - x)
    const float ax = fmaxf(nx.x * (ylo.x - x.x), nx.x * (yhi.x - x.x));
    const float ay = fmaxf(nx.y * (ylo.y - x.y), nx.y * (yhi.y - x.y));
    const float az = fmaxf(nx.z * (ylo.z - x.z), nx.z * (yhi.z - x.z));
    // max over n in the normal box, y in the position box of n.(x - y): corner products per axis
    const float dxl = x.x - yhi.x, dxh = x.x - ylo.x, dyl = x.y - yhi.y, dyh = x.y - ylo.y;
    const float dzl = x.z - yhi.z, dzh = x.z - ylo.z;
    const float bx = fmaxf(fmaxf(nlo.x * dxl, nlo.x * dxh), fmaxf(nhi.x * dxl, nhi.x * dxh));
    const float by = fmaxf(fmaxf(nlo.y * dyl, nlo.y * dyh), fmaxf(nhi.y * dyl, nhi.y * dyh));
    const float bz = fmaxf(fmaxf(nlo.z * dzl, nlo.z * dzh), fmaxf(nhi.z * dzl, nhi.z * dzh));
    const float scale = fmax3(fabsf(x.x), fabsf(x.y), fabsf(x.z)) +
                        fmax3(fmaxf(fabsf(ylo.x), fabsf(yhi.x)), fmaxf(fabsf(ylo.y), fabsf(yhi.y)),
                              fmaxf(fabsf(ylo.z), fabsf(yhi.z)));
    const float m = 1e-4f * scale;   // >> the rounding of d = y - x and of the two dots
    return (ax + ay) + az > -m && (bx + by) + bz > -m;
}
// Can any receiver with position in [xl, xh] and normal in [nl, nh] (rb = xl nl xh nh) trace VPL v, i.e.
// can cx = n_x.(y - x) > 0 and ci = n_y.(x - y) > 0 both hold?  Interval bounds per axis, with the
// cluster cull's margin (far above the fp32 rounding of O13's dots).
__device__ __forceinline__ bool vpl_may_trace(const vpl_record* __restrict__ v, const float* rb) {
    const float4 yv = __ldg((const float4*)v), nv = __ldg((const float4*)v + 1);
    const float y[3] = {yv.x, yv.y, yv.z}, ny[3] = {nv.x, nv.y, nv.z};
    float cx = 0.0f, ci = 0.0f, sx = 0.0f, sy = 0.0f;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const float xl = rb[a], nl = rb[3 + a], xh = rb[6 + a], nh = rb[9 + a];
        const float dl = y[a] - xh, dh = y[a] - xl;   // y - x over the box
        cx += fmaxf(fmaxf(nl * dl, nl * dh), fmaxf(nh * dl, nh * dh));
        ci += fmaxf(ny[a] * -dl, ny[a] * -dh);
        sx = fmaxf(sx, fmaxf(fabsf(xl), fabsf(xh)));
        sy = fmaxf(sy, fabsf(y[a]));
    }
    const float m = 1e-4f * (sx + sy);
    return cx > -m && ci > -m;
}
__global__ void k_vpl_clusters(const vpl_record* __restrict__ v, int32_t M, float4* __restrict__ cb) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;     // one thread per cluster
    if ((int64_t)c * kCluster >= M) return;
    const float inf = __int_as_float(0x7f800000);
    float4 a = make_float4(inf, inf, inf, 0.0f), b = make_float4(-inf, -inf, -inf, 0.0f);
    float4 na = a, nb = b;
    const int i1 = min(M, (c + 1) * kCluster);
    for (int i = c * kCluster; i < i1; ++i) {
        const float4* p = (const float4*)(v + i);
        const float4 y = p[0], n = p[1];
        a.x = fminf(a.x, y.x); a.y = fminf(a.y, y.y); a.z = fminf(a.z, y.z);
        b.x = fmaxf(b.x, y.x); b.y = fmaxf(b.y, y.y); b.z = fmaxf(b.z, y.z);
        na.x = fminf(na.x, n.x); na.y = fminf(na.y, n.y); na.z = fminf(na.z, n.z);
        nb.x = fmaxf(nb.x, n.x); nb.y = fmaxf(nb.y, n.y); nb.z = fmaxf(nb.z, n.z);
    }
    cb[4 * c] = a; cb[4 * c + 1] = b; cb[4 * c + 2] = na; cb[4 * c + 3] = nb;
}

// One warp per CTA: the traversal stack is then at a fixed shared-memory
// address (no per-warp base to keep live in a register), and 32 one-warp
// CTAs fill an SM at the 64-register budget.
#ifndef VPL_CLUSTER_CULL
#define VPL_CLUSTER_CULL 1   // skip 32-VPL clusters no lane of the warp can trace
#endif
#ifndef VPL_GATHER_CTAS
#define VPL_GATHER_CTAS 32
#endif
#ifndef VPL_INTERLEAVE
#define VPL_INTERLEAVE 1
#endif
#ifndef VPL_CHUNK_GROUP
#define VPL_CHUNK_GROUP 128   // VPLs per interleave group (a multiple of the cluster size that divides 256); each group's
                              // fp32 partial is folded into the chunk total
#endif
constexpr int kGroup = VPL_CHUNK_GROUP;
static_assert(kGroup % kCluster == 0 && 256 % kGroup == 0, "interleave group");
#ifndef VPL_STAGE
#define VPL_STAGE 0   // 1: each cluster's VPL records staged in shared memory by a 1-D bulk async copy (cp.async.bulk +
                      // mbarrier; single buffer, the copy overlaps the per-VPL cull) instead of warp-uniform L1 loads
#endif
#ifndef VPL_ACC_SMEM
#define VPL_ACC_SMEM 0   // 1: Eq. 1 sums accumulate in the shared-memory totals directly instead of 6 registers folded per
                         // group (measured: spills 268 -> 220 B but C4 +1.7%: off)
#endif
#ifndef VPL_VPL_CULL
#define VPL_VPL_CULL 1   // per-VPL cull against the receiver block's bounds, one VPL per lane
#endif
#ifndef VPL_TAIL_BLOCKS
#define VPL_TAIL_BLOCKS -1  // >= 0: whole-block tasks for all but the last VPL_TAIL_BLOCKS x grid blocks of a call (no partial
                            // sums for them); measured at 2: block costs vary ~10x, the long tasks unbalance the SMs (C3 226 ->
                            // 496 ms, C4 670 -> 807 ms); -1: (block, chunk) tasks only (whole-block only when M fits one chunk)
#endif
#ifndef VPL_PART_EVICT_LAST
#define VPL_PART_EVICT_LAST 1   // partial stores with an L2 evict_last policy (C4: DRAM writes 120 -> 64 MB per launch)
#endif
// Test hook (kDump, vpl_gather_dump): the production gather additionally records, for listed pixels,
// its own traced / visible bit of every pixel x VPL pair (indexed by the caller's VPL order through
// the sort permutation) — the visibility the image was computed with.
struct GatherDump {
    const int32_t* slot;   // [W*H] pixel -> dump row, -1 = not dumped
    const int32_t* perm;   // sorted position -> caller's VPL index (null: identity)
    uint32_t *tbits, *vbits;
    int32_t words;         // ceil(M / 32)
};
template <bool kCount, bool kDump = false>
__global__ void __launch_bounds__(32, VPL_GATHER_CTAS) k_gather(SceneView sv, BvhView bv, TileMap tm, const vpl_gpoint* __restrict__ gb,
                                                const vpl_record* __restrict__ vpls, int32_t M, float* __restrict__ rgb,
                                                vpl_counters* __restrict__ ctr, int* __restrict__ queue,
                                                const float4* __restrict__ clusters, int32_t chunk, int32_t n_chunks,
                                                float* __restrict__ part_out, int* __restrict__ done,
                                                int* __restrict__ slot_gen, int32_t ring, int32_t n_whole,
                                                GatherDump dump) {
    __shared__ int sstack[kWarpStack];
    __shared__ float s_acc[kSeg][3][32];   // running per-receiver totals (kept out of the register budget)
#if VPL_TAIL_BLOCKS >= 0
    __shared__ float s_tot[kSeg][3][32];   // whole-block tasks: the chunk totals folded in chunk order
#else
    float (*s_tot)[3][32] = s_acc;         // whole-block tasks have a single chunk: its total is the block's
#endif
    __shared__ float s_rb[12];             // receiver bounds of the task: lo(x, n), hi(x, n)  (VPL_VPL_CULL)
#if VPL_STAGE
    __shared__ __align__(128) float4 s_vpl[3 * kCluster];   // the current cluster's records, staged by a bulk async copy
    __shared__ __align__(8) unsigned long long s_bar;       // its mbarrier (one arrival + the copy's bytes per phase)
    const unsigned s_vpl_addr = (unsigned)__cvta_generic_to_shared(s_vpl);
    const unsigned s_bar_addr = (unsigned)__cvta_generic_to_shared(&s_bar);
    unsigned stage_phase = 0;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_bar_addr) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
#endif
    constexpr int kPart = 96 * kSeg;       // partial floats per (block, chunk): 32 lanes x kSeg receivers x 3
    const int lane = threadIdx.x;
    // Tasks: the first n_whole blocks of the call are whole-block tasks (one warp walks all the chunks of
    // the block and folds their totals in chunk order itself: no partial sums leave the SM); the
    // remaining blocks are split into (block, chunk) tasks, fine-grained enough that the dynamic queue
    // balances the SMs at the end of the launch and when a rank holds 1/8 of the frame.  Both give the
    // same fp32 sums: chunk totals from zero, folded in chunk order.
    const int64_t ntask = n_whole + (tm.n_warps() - n_whole) * n_chunks;
    const float eps = sv.hdr->eps, b2 = sv.hdr->b2;
    while (true) {
        int64_t g;
        if (lane == 0) g = atomicAdd(queue, 1);
        g = __shfl_sync(0xFFFFFFFFu, g, 0);
        if (g >= ntask) break;
        const bool whole = g < n_whole;
        const int64_t blk = whole ? g : n_whole + (g - n_whole) / n_chunks;   // 8 x 4kSeg pixel block of the call
        const int ch0 = whole ? 0 : (int)((g - n_whole) % n_chunks), ch1 = whole ? n_chunks : ch0 + 1;
        int32_t pix[kSeg];
        f3 x[kSeg], nx[kSeg];
        int tri_x[kSeg];
        unsigned act = 0;
#pragma unroll
        for (int k = 0; k < kSeg; ++k) {
            pix[k] = tm.pixel(blk, lane, k);
            x[k] = mk3(0, 0, 0); nx[k] = mk3(0, 0, 0);
            tri_x[k] = -1;
            if (pix[k] >= 0) {
                const float4* gp = (const float4*)(gb + pix[k]);
                const float4 a = gp[0], b = gp[1];
                tri_x[k] = __float_as_int(a.w);
                if (tri_x[k] >= 0 && __float_as_int(b.w) != 0) act |= 1u << k;
                x[k] = xyz(a); nx[k] = xyz(b);
            }
#if VPL_TAIL_BLOCKS >= 0
            s_tot[k][0][lane] = 0.0f; s_tot[k][1][lane] = 0.0f; s_tot[k][2][lane] = 0.0f;
#endif
        }
        if (VPL_VPL_CULL) {   // bounds of the block's front-face receivers and of their normals (uniform)
            const float inf = __int_as_float(0x7f800000);
            float lo[6] = {inf, inf, inf, inf, inf, inf}, hi[6] = {-inf, -inf, -inf, -inf, -inf, -inf};
#pragma unroll
            for (int k = 0; k < kSeg; ++k)
                if ((act >> k) & 1u) {
                    const float v[6] = {x[k].x, x[k].y, x[k].z, nx[k].x, nx[k].y, nx[k].z};
#pragma unroll
                    for (int a = 0; a < 6; ++a) { lo[a] = fminf(lo[a], v[a]); hi[a] = fmaxf(hi[a], v[a]); }
                }
            __syncwarp();
#pragma unroll
            for (int a = 0; a < 6; ++a) {
                const float l = warp_min_f32(lo[a]), h = warp_max_f32(hi[a]);
                if (lane == 0) { s_rb[a] = l; s_rb[6 + a] = h; }
            }
            __syncwarp();
        }
        HeavyState hs;   // occluder caches, list cursor, weights: touched by shade_heavy only (local memory)
#pragma unroll
        for (int k = 0; k < kSeg; ++k) hs.cache[k] = OccluderCache();
        hs.eps = eps; hs.b2 = b2;
        TravStats st;
        unsigned long long n_traced = 0, n_vis = 0, n_pairs = 0;
        for (int ch = ch0; ch < ch1; ++ch) {
        // The chunk's VPLs: groups of kGroup consecutive VPLs of the sorted copy, interleaved over the chunks
        // (group q belongs to chunk q % n_chunks), so that every chunk samples the whole VPL set and the
        // tasks of a block cost about the same — a contiguous range of the spatial order is either all
        // culled or all near, and the longest tasks set the tail of a launch.  VPL_INTERLEAVE 0: contiguous.
        const int n_groups = (M + kGroup - 1) / kGroup, gpc = chunk / kGroup;
        const int q0 = VPL_INTERLEAVE ? ch : ch * gpc, q1 = VPL_INTERLEAVE ? n_groups : min(n_groups, (ch + 1) * gpc);
        const int qs = VPL_INTERLEAVE ? n_chunks : 1;
#pragma unroll
        for (int k = 0; k < kSeg; ++k) { s_acc[k][0][lane] = 0.0f; s_acc[k][1][lane] = 0.0f; s_acc[k][2][lane] = 0.0f; }
        if (__any_sync(0xFFFFFFFFu, act != 0)) {
            for (int q = q0; q < q1; q += qs) {
                const int i0 = q * kGroup, vend = M;
                if (kCount) n_pairs += (unsigned long long)__popc(act) * (unsigned long long)(min(M, i0 + kGroup) - i0);
#if !VPL_ACC_SMEM
                float part[kSeg][3];
#pragma unroll
                for (int k = 0; k < kSeg; ++k) part[k][0] = part[k][1] = part[k][2] = 0.0f;
#endif
                const int i1 = min(vend, i0 + kGroup);
                for (int c0 = i0; c0 < i1; c0 += kCluster) {       // clusters of kCluster VPLs (i0 % 256 == 0)
                    const float4* cb = clusters ? clusters + 4 * (c0 / kCluster) : nullptr;
                    unsigned inc = act;                            // receivers that may trace the cluster
#pragma unroll
                    for (int k = 0; k < kSeg; ++k)
                        if (cb && ((inc >> k) & 1u) && !cluster_may_trace(cb, x[k], nx[k])) inc &= ~(1u << k);
                    if (cb && !__any_sync(0xFFFFFFFFu, inc != 0)) continue;   // no receiver can trace any VPL of it
                    const int c1 = min(c0 + kCluster, i1);
                    hs.cand = -1; hs.cand_end = cb ? c0 : INT_MAX;         // candidate list (lazy) and its VPL range end
                    // per-VPL cull, transposed: lane l tests VPL c0 + l against the box of the block's
                    // receivers and the box of their normals (s_rb) — can cx > 0 and ci > 0 hold for any
                    // of them?  Same conservative margin as the cluster cull; the VPL loop then visits
                    // only the VPLs some receiver may trace.
                    unsigned need = 0xFFFFFFFFu >> (32 - (c1 - c0));
#if VPL_STAGE
                    // the cluster's records (48 B each) by one 1-D bulk async copy (TMA) into shared memory;
                    // the copy overlaps the per-VPL cull below, its completion is awaited on the mbarrier
                    __syncwarp();   // the previous cluster's readers are done
                    if (lane == 0) {
                        const unsigned bytes = (unsigned)(c1 - c0) * 48u;
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_bar_addr), "r"(bytes) : "memory");
                        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                                     ::"r"(s_vpl_addr), "l"(vpls + c0), "r"(bytes), "r"(s_bar_addr) : "memory");
                    }
#endif
                    if (VPL_VPL_CULL && cb) need &= __ballot_sync(0xFFFFFFFFu, vpl_may_trace(vpls + min(c0 + lane, c1 - 1), s_rb));
#if VPL_STAGE
                    {
                        unsigned ok = 0;
                        for (int spin = 0; !ok; ++spin) {
                            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                                         : "=r"(ok) : "r"(s_bar_addr), "r"(stage_phase) : "memory");
                            if (spin > (1 << 22)) __trap();   // never hang the GPU on a lost copy
                        }
                        stage_phase ^= 1u;
                    }
#endif
                    while (need) {
                        const int i = c0 + __ffs(need) - 1;
                        need &= need - 1u;
#if VPL_STAGE
                        const float4 yv = s_vpl[3 * (i - c0)], nb = s_vpl[3 * (i - c0) + 1];
#else
                        const float4 yv = __ldg((const float4*)(vpls + i)), nb = __ldg((const float4*)(vpls + i) + 1);
#endif
                        const unsigned tv = shade<kCount>(bv, vpls, i, xyz(yv), __float_as_int(yv.w), nb, x, nx, tri_x, act,
                                                          &hs, sstack, &st, c1, inc);
                        const float* w = hs.w;
                        const unsigned tr = tv & 0xFFFFu, vis = tv >> 16;
                        if (kCount) { n_traced += __popc(tr); n_vis += __popc(vis); }
                        if (kDump) {
#pragma unroll
                            for (int k = 0; k < kSeg; ++k) {
                                const int ds = pix[k] >= 0 ? dump.slot[pix[k]] : -1;
                                if (ds >= 0) {
                                    const int o = dump.perm ? dump.perm[i] : i;
                                    const size_t wd = (size_t)ds * dump.words + (o >> 5);
                                    if (tr & (1u << k)) atomicOr(dump.tbits + wd, 1u << (o & 31));
                                    if (vis & (1u << k)) atomicOr(dump.vbits + wd, 1u << (o & 31));
                                }
                            }
                        }
                        if (vis) {
#if VPL_STAGE
                            const float4 phi = s_vpl[3 * (i - c0) + 2];
#else
                            const float4 phi = __ldg((const float4*)(vpls + i) + 2);
#endif
#pragma unroll
                            for (int k = 0; k < kSeg; ++k)
                                if (vis & (1u << k)) {
#if VPL_ACC_SMEM
                                    s_acc[k][0][lane] = fmaf(phi.x, w[k], s_acc[k][0][lane]);
                                    s_acc[k][1][lane] = fmaf(phi.y, w[k], s_acc[k][1][lane]);
                                    s_acc[k][2][lane] = fmaf(phi.z, w[k], s_acc[k][2][lane]);
#else
                                    part[k][0] = fmaf(phi.x, w[k], part[k][0]);
                                    part[k][1] = fmaf(phi.y, w[k], part[k][1]);
                                    part[k][2] = fmaf(phi.z, w[k], part[k][2]);
#endif
                                }
                        }
                    }
                }
#pragma unroll
                for (int k = 0; k < kSeg; ++k) {
#if !VPL_ACC_SMEM
                    s_acc[k][0][lane] += part[k][0]; s_acc[k][1][lane] += part[k][1]; s_acc[k][2][lane] += part[k][2];
#endif
                }
            }
        }
#if VPL_TAIL_BLOCKS >= 0
        if (whole) {   // the same fold as the chunked path's: totals from 0.0f, chunk totals added in chunk order
#pragma unroll
            for (int k = 0; k < kSeg; ++k) {
                s_tot[k][0][lane] += s_acc[k][0][lane]; s_tot[k][1][lane] += s_acc[k][1][lane];
                s_tot[k][2][lane] += s_acc[k][2][lane];
            }
        }
#endif
        }   // chunks of the task
        const float sc = (float)(1.0 / kPiR);
        if (whole) {
#pragma unroll
            for (int k = 0; k < kSeg; ++k)
                if (pix[k] >= 0) {
                    const bool on = (act >> k) & 1u;
                    const f3 rho = xyz(((const float4*)(gb + pix[k]))[2]);
                    float* o = rgb + 3 * (int64_t)pix[k];
                    o[0] = on ? s_tot[k][0][lane] * rho.x * sc : 0.0f;
                    o[1] = on ? s_tot[k][1][lane] * rho.y * sc : 0.0f;
                    o[2] = on ? s_tot[k][2][lane] * rho.z * sc : 0.0f;
                }
        } else {
            const int ch = ch0;
            // chunk partial sums, (slot, chunk, receiver, lane)-contiguous in a ring of `ring` block slots
            // (the call's block ordinal modulo ring: a few MB stay L2-resident); the warp that completes a
            // block's last chunk folds them in chunk order (fp32), writes the pixels, discards the partial
            // lines (never written back to HBM) and hands the slot to the block `ring` later.
            const int64_t lb = blk - n_whole;
            const int slot = (int)(lb % ring), gen = (int)(lb / ring);
            float* pb = part_out + ((int64_t)slot * n_chunks) * kPart;
            if (lane == 0) {   // the slot's previous block (dispensed earlier, so running) must be folded
                int cur;
                while (true) {
                    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(cur) : "l"(slot_gen + slot) : "memory");
                    if (cur >= gen) break;
                    __nanosleep(256);
                }
            }
            __syncwarp();
#pragma unroll
            for (int k = 0; k < kSeg; ++k) {
                float* o = pb + ch * kPart + 96 * k + 3 * lane;
#if VPL_PART_EVICT_LAST
                uint64_t pol;   // keep the partial lines in L2 until the fold discards them
                asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
                asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(o), "f"(s_acc[k][0][lane]), "l"(pol) : "memory");
                asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(o + 1), "f"(s_acc[k][1][lane]), "l"(pol) : "memory");
                asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(o + 2), "f"(s_acc[k][2][lane]), "l"(pol) : "memory");
#else
                o[0] = s_acc[k][0][lane]; o[1] = s_acc[k][1][lane]; o[2] = s_acc[k][2][lane];
#endif
            }
            __threadfence();
            __syncwarp();
            int prev = 0;
            if (lane == 0) prev = atomicAdd(done + slot, 1);
            prev = __shfl_sync(0xFFFFFFFFu, prev, 0);
            if (prev == n_chunks - 1) {
                __threadfence();
#pragma unroll
                for (int k = 0; k < kSeg; ++k) {
                    float acc[3] = {0.0f, 0.0f, 0.0f};
                    for (int c = 0; c < n_chunks; ++c) {
                        const float* q = pb + c * kPart + 96 * k + 3 * lane;
                        acc[0] += __ldcg(q); acc[1] += __ldcg(q + 1); acc[2] += __ldcg(q + 2);
                    }
                    if (pix[k] >= 0) {
                        const bool on = (act >> k) & 1u;
                        const f3 rho = xyz(((const float4*)(gb + pix[k]))[2]);
                        float* out = rgb + 3 * (int64_t)pix[k];
                        out[0] = on ? acc[0] * rho.x * sc : 0.0f;
                        out[1] = on ? acc[1] * rho.y * sc : 0.0f;
                        out[2] = on ? acc[2] * rho.z * sc : 0.0f;
                    }
                }
                __syncwarp();
                for (int l = lane; l < (kPart / 32) * n_chunks; l += 32)
                    asm volatile("discard.global.L2 [%0], 128;" ::"l"(pb + 32 * l) : "memory");
                __syncwarp();
                if (lane == 0) {
                    done[slot] = 0;
                    __threadfence();
                    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(slot_gen + slot), "r"(gen + 1) : "memory");
                }
            }
        }
        if (kCount) {
            unsigned long long v[20] = {n_pairs, n_traced, n_vis, st.boxes, st.tris, st.wrays, st.wsteps,
                                        st.cones, st.cpk, st.rpk, st.chits, st.ctests, st.lists, st.entries,
                                        st.lfail, st.fsteps, st.lsteps, st.fmt, st.fmt_hit, st.pculled};
#pragma unroll
            for (int q = 0; q < 20; ++q) {
                unsigned long long a = v[q];
                for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xFFFFFFFFu, a, o);
                if (lane == 0) atomicAdd(&ctr->pairs + q, a);
            }
        }
    }
}

// test hook: traced / visible bits of listed pixels x all VPLs, through the
// gather's own traversal engine in the caller's VPL order (lanes = 32
// consecutive listed pixels, receiver slot 0; no clusters, no lists)
__global__ void k_visdump(SceneView sv, BvhView bv, const vpl_gpoint* __restrict__ gb, const vpl_record* __restrict__ vpls,
                          int32_t M, const int32_t* __restrict__ pixels, int32_t n_px, uint32_t* __restrict__ tbits,
                          uint32_t* __restrict__ vbits) {
    __shared__ int s_stack[2][kWarpStack];
    int* sstack = s_stack[threadIdx.x >> 5];
    int64_t words = (M + 31) / 32;
    HeavyState hs;
#pragma unroll
    for (int q = 0; q < kSeg; ++q) hs.cache[q] = OccluderCache();
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    if ((k - lane) >= n_px) return;                      // whole warp out of range
    bool inb = k < n_px;
    const vpl_gpoint* gp = gb + (inb ? pixels[k] : 0);
    f3 x[kSeg], nx[kSeg];
    int tri_x[kSeg];
    x[0] = ld3(gp->pos); nx[0] = ld3(gp->nrm); tri_x[0] = gp->tri;
    if (kSeg > 1) { x[kSeg - 1] = x[0]; nx[kSeg - 1] = nx[0]; tri_x[kSeg - 1] = -1; }
    const unsigned act = (inb && gp->tri >= 0 && gp->front) ? 1u : 0u;
    const float eps = sv.hdr->eps, b2 = sv.hdr->b2;
    hs.eps = eps; hs.b2 = b2;
    for (int64_t wd = 0; wd < words; ++wd) {
        uint32_t tb = 0, vb = 0;
        const int i0 = (int)(wd * 32), i1 = min(M, i0 + 32);
        for (int i = i0; i < i1; ++i) {
            const float4 yv = __ldg((const float4*)(vpls + i)), nb = __ldg((const float4*)(vpls + i) + 1);
            hs.cand = -1; hs.cand_end = INT_MAX;
            const unsigned tv = shade<false>(bv, vpls, i, xyz(yv), __float_as_int(yv.w), nb, x, nx, tri_x, act, &hs,
                                             sstack, nullptr, i1, act);
            tb |= (tv & 1u) << (i - i0);
            vb |= ((tv >> 16) & 1u) << (i - i0);
        }
        if (inb) { tbits[k * words + wd] = tb; vbits[k * words + wd] = vb; }
    }
}

__global__ void k_closest_batch(BvhView bv, const float* __restrict__ o, const float* __restrict__ d, int64_t n,
                                float tmin, float tmax, int32_t* __restrict__ tri, float* __restrict__ tout) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    Ray r = make_ray(ld3(o + 3 * i), ld3(d + 3 * i), tmin, tmax);
    float t;
    int h = bvh_closest(bv, r, t);
    tri[i] = h;
    tout[i] = h >= 0 ? t : 0.0f;
}

__global__ void k_occluded_batch(SceneView sv, BvhView bv, const float* __restrict__ a, const float* __restrict__ b,
                                 int64_t n, uint8_t* __restrict__ occ) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    occ[i] = segment_occluded<false>(bv, ld3(a + 3 * i), ld3(b + 3 * i), sv.hdr->eps, nullptr);
}

__global__ void k_philox_batch(const uint32_t* __restrict__ in, int64_t n, uint32_t* __restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t* c = in + 6 * i;
    uint32_t r[4];
    Philox::block(c[0], c[1], c[2], c[3], c[4], c[5], r);
    for (int k = 0; k < 4; ++k) out[4 * i + k] = r[k];
}

static inline int nb(int64_t n, int t) { return (int)((n + t - 1) / t); }

// Gather-side VPL order: Eq. 1 is a sum over the VPL set, so the gather may
// visit the VPLs in any fixed order.  It visits them in Morton order of
// their positions (30-bit code over the VPL bounding box) so consecutive
// VPLs are close: the occluder cache hits more often and groups of nearby
// VPLs share one beam (gather.cuh).  The array order of vpl_generate_vpls
// (the oracle-checked output) is not touched; the sorted copy lives in the
// gather's work buffer.
__device__ __forceinline__ uint32_t spread10(uint32_t x) {
    x &= 0x3FFu;
    x = (x | (x << 16)) & 0x030000FFu;
    x = (x | (x << 8)) & 0x0300F00Fu;
    x = (x | (x << 4)) & 0x030C30C3u;
    x = (x | (x << 2)) & 0x09249249u;
    return x;
}
__global__ void k_vpl_bbox(const vpl_record* __restrict__ v, int32_t M, unsigned* __restrict__ box) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= M) return;
    const float* p = (const float*)(v + i);
    for (int a = 0; a < 3; ++a) {
        atomicMin(box + a, (unsigned)fkey(p[a]) ^ 0x80000000u);
        atomicMax(box + 3 + a, (unsigned)fkey(p[a]) ^ 0x80000000u);
    }
}
__global__ void k_vpl_morton(const vpl_record* __restrict__ v, int32_t M, const unsigned* __restrict__ box,
                             uint32_t* __restrict__ keys, int32_t* __restrict__ idx) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= M) return;
    const float* p = (const float*)(v + i);
    uint32_t c = 0;
    for (int a = 0; a < 3; ++a) {
        float lo = fkey_inv((int)(box[a] ^ 0x80000000u)), hi = fkey_inv((int)(box[3 + a] ^ 0x80000000u));
        float ext = hi - lo;
        float q = ext > 0.0f ? (p[a] - lo) * (1024.0f / ext) : 0.0f;
        c |= spread10(min((uint32_t)fmaxf(q, 0.0f), 1023u)) << a;
    }
    keys[i] = c;
    idx[i] = i;
}
__global__ void k_vpl_permute(const vpl_record* __restrict__ v, const int32_t* __restrict__ idx, int32_t M,
                              vpl_record* __restrict__ out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= M) return;
    const float4* src = (const float4*)(v + idx[i]);
    float4* dst = (float4*)(out + i);
    dst[0] = src[0]; dst[1] = src[1]; dst[2] = src[2];
}

// O14 — direct term L_e of Eq. 1 (reading R21): per pixel, S
// uniform samples on every area light (Philox stream 4, item = pixel,
// draws 2(lS+s), 2(lS+s)+1), E_c += L_c ((A cx) cl) / (r2 r2) if visible,
// out = (rho (E inv_S)) / pi — the same exact-fp32 form as Eq. 2 (O8), so
// the result is bitwise the oracle's.  One thread per pixel, exact any-hit
// on the binary BVH.
__global__ void k_direct(SceneView sv, BvhView bv, TileMap tm, const vpl_gpoint* __restrict__ gb, int32_t S,
                         uint64_t seed, float inv_S, int32_t accumulate, float* __restrict__ rgb) {
    int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (g >= tm.n_warps()) return;
    int32_t pix = tm.pixel(g, lane);
    if (pix < 0) return;
    const SceneHdr* h = sv.hdr;
    const float4* gp = (const float4*)(gb + pix);
    const float4 a = gp[0], b = gp[1], c = gp[2];
    const bool ok = __float_as_int(a.w) >= 0 && __float_as_int(b.w) != 0;
    float E[3] = {0.0f, 0.0f, 0.0f}, Pt[3] = {0.0f, 0.0f, 0.0f};
    if (ok) {
        const f3 x = xyz(a), nx = xyz(b);
        Philox ph(seed, 4u, (uint32_t)pix);
        for (int l = 0; l < h->nL; ++l) {
            const float* L = h->lights + 16 * l;
            if (light_is_point(L)) {   // R27: no samples, Phi cx / ((r2 sqrt r2) 4 pi) V
                const f3 y = ld3(L);
                const f3 d = y - x;
                const float r2 = dot(d, d);
                const float cx = dot(nx, d);
                if (cx > 0.0f && !segment_occluded<false>(bv, x, y, h->eps, nullptr)) {
                    const float gg = point_g(cx, r2);
                    Pt[0] += L[13] * gg; Pt[1] += L[14] * gg; Pt[2] += L[15] * gg;
                }
                continue;
            }
            const f3 corner = ld3(L), eu = ld3(L + 3), ev = ld3(L + 6), nl = ld3(L + 9);
            for (int q = 0; q < S; ++q) {
                const uint32_t j = 2u * (uint32_t)(l * S + q);
                const float u = u01(ph.at(j)), v = u01(ph.at(j + 1));
                const f3 y = (corner + u * eu) + v * ev;
                const f3 d = y - x;
                const float r2 = dot(d, d);
                const float cx = dot(nx, d);
                const float cl = -dot(nl, d);
                if (cx > 0.0f && cl > 0.0f && !segment_occluded<false>(bv, x, y, h->eps, nullptr)) {
                    const float gg = ((L[12] * cx) * cl) / (r2 * r2);
                    E[0] += L[13] * gg; E[1] += L[14] * gg; E[2] += L[15] * gg;
                }
            }
        }
    }
    const float INV_PI = (float)(1.0 / kPiR);
    float* o = rgb + 3 * (int64_t)pix;
    const float r0 = ok ? (c.x * ((E[0] * inv_S) + Pt[0])) * INV_PI : 0.0f;
    const float r1 = ok ? (c.y * ((E[1] * inv_S) + Pt[1])) * INV_PI : 0.0f;
    const float r2o = ok ? (c.z * ((E[2] * inv_S) + Pt[2])) * INV_PI : 0.0f;
    if (accumulate) { o[0] += r0; o[1] += r1; o[2] += r2o; }
    else { o[0] = r0; o[1] = r1; o[2] = r2o; }
}

// NEXT f1 — image error against a reference (the RMSE harness of the
// paper's equal-sample comparisons): fp64 sums of (a - r)^2, r^2,
// |a - r|, |r| over n floats.  Deterministic: each block reduces a fixed
// strided subset in a fixed tree order, one block then adds the partials in
// block order.
constexpr int kErrBlocks = 592, kErrThreads = 256;
__global__ void __launch_bounds__(kErrThreads) k_image_err(const float* __restrict__ a, const float* __restrict__ r,
                                                           int64_t n, double* __restrict__ part) {
    __shared__ double sh[4][kErrThreads];
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t i = blockIdx.x * (int64_t)kErrThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kErrThreads) {
        const double x = a[i], y = r[i], d = x - y;
        acc[0] += d * d; acc[1] += y * y; acc[2] += fabs(d); acc[3] += fabs(y);
    }
    for (int q = 0; q < 4; ++q) sh[q][threadIdx.x] = acc[q];
    __syncthreads();
    for (int w = kErrThreads / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w)
            for (int q = 0; q < 4; ++q) sh[q][threadIdx.x] += sh[q][threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x < 4) part[4 * blockIdx.x + threadIdx.x] = sh[threadIdx.x][0];
}
__global__ void k_image_err_final(const double* __restrict__ part, int nb, double* __restrict__ out) {
    if (threadIdx.x >= 4) return;
    double t = 0.0;
    for (int b = 0; b < nb; ++b) t += part[4 * b + threadIdx.x];
    out[threadIdx.x] = t;
}

// VPL chunking of the gather's work items: depends on M only (so any tile split
// reproduces the same sums): chunk = max(CHUNK_MIN, ceil(M / CHUNKS) rounded up to 256); 128 chunks
// put the C4 load-balance efficiency at 8 ranks at 95% (tools/shard_sim.py)
#ifndef VPL_GATHER_CHUNKS
#define VPL_GATHER_CHUNKS 128
#endif
#ifndef VPL_GATHER_CHUNK_MIN
#define VPL_GATHER_CHUNK_MIN 256
#endif
static inline void gather_chunks(int32_t M, int32_t* chunk, int32_t* n_chunks) {
    int64_t c = ((int64_t)M + VPL_GATHER_CHUNKS - 1) / VPL_GATHER_CHUNKS;
    c = (c + 255) / 256 * 256;
    if (c < VPL_GATHER_CHUNK_MIN) c = VPL_GATHER_CHUNK_MIN;
    *chunk = (int32_t)c;
    *n_chunks = M > 0 ? (int32_t)(((int64_t)M + c - 1) / c) : 1;
}

struct GatherWork {
    int* queue;
    int* slot_gen;
    int32_t ring;
    unsigned* box;
    float4* clusters;
    float* part;
    int* done;
    uint32_t *keys, *keys2;
    int32_t *idx, *idx2;
    vpl_record* sorted;
    void* cub;
    size_t cub_bytes;
};
// partial-sum ring: block slots reused modulo VPL_PART_RING (C4: 4096 x 128 chunks x 384 B = 201 MB
// allocated instead of 3.2 GB for the whole frame; 512 slots made warps wait on straggler chunks: +30%)
#ifndef VPL_PART_RING
#define VPL_PART_RING 4096
#endif

static size_t gather_layout(int32_t M, int32_t W, int32_t H, char* base, GatherWork* w) {
    Bump b{base};
    w->queue = b.take<int>(1);
    int32_t chunk, nch;
    gather_chunks(M, &chunk, &nch);
    const size_t nblk = (size_t)((W + 7) / 8) * (size_t)((H + 3) / 4);   // 8x4 blocks of a full frame
    w->ring = (int32_t)(nblk < (size_t)VPL_PART_RING ? (nblk > 0 ? nblk : 1) : VPL_PART_RING);
    w->part = b.take<float>(nch > 1 ? (size_t)w->ring * (size_t)nch * 96 * kSeg : 1);
    w->done = b.take<int>(w->ring);
    w->slot_gen = b.take<int>(w->ring);
    w->box = b.take<unsigned>(6);
    size_t m = (size_t)(M > 0 ? M : 1);
    w->keys = b.take<uint32_t>(m);
    w->keys2 = b.take<uint32_t>(m);
    w->idx = b.take<int32_t>(m);
    w->idx2 = b.take<int32_t>(m);
    w->sorted = b.take<vpl_record>(m);
    w->clusters = b.take<float4>(4 * ((m + kCluster - 1) / kCluster));
    size_t c = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, c, (uint32_t*)nullptr, (uint32_t*)nullptr, (int32_t*)nullptr,
                                    (int32_t*)nullptr, (int)m, 0, 30);
    w->cub_bytes = c;
    w->cub = b.take<char>(c);
    return b.off;
}

static int32_t make_tilemap(const SceneHdr& hh, const int32_t* d_tiles, int32_t n_tiles, int32_t tw, int32_t th,
                            TileMap* tm) {
    if ((!d_tiles && n_tiles != 0) || n_tiles < 0 || tw <= 0 || th <= 0 || tw % 8 || th % 4) {
        set_error("bad tile arguments (tile_w %% 8 == 0, tile_h %% 4 == 0 required)");
        return VPL_EINVAL;
    }
    tm->tiles = d_tiles;
    tm->n_tiles = n_tiles;
    tm->tw = tw; tm->th = th;
    tm->W = hh.W; tm->H = hh.H;
    tm->tiles_x = (hh.W + tw - 1) / tw;
    tm->bx_per_tile = tw / 8;
    tm->blocks_per_tile = (tw / 8) * (th / 4);
    return VPL_OK;
}

}  // namespace vplgi

using namespace vplgi;

extern "C" {

int32_t vpl_render_gbuffer(const void* d_scene, const void* d_bvh, const int32_t* d_tiles, int32_t n_tiles,
                           int32_t tile_w, int32_t tile_h, vpl_gpoint* d_gbuf, void* stream) {
    if (!d_scene || !d_bvh || !d_gbuf) { set_error("vpl_render_gbuffer: null pointer"); return VPL_EINVAL; }
    cudaStream_t s = (cudaStream_t)stream;
    SceneHdr hh;
    VPL_TRY(read_scene_hdr(d_scene, s, &hh));
    TileMap tm;
    VPL_TRY(make_tilemap(hh, d_tiles, n_tiles, tile_w, tile_h, &tm));
    if (n_tiles == 0) return VPL_OK;
    int64_t threads = tm.n_warps() * 32;
    k_gbuffer<<<nb(threads, 128), 128, 0, s>>>(scene_view(d_scene, hh.n), bvh_view(d_bvh, hh.n), tm, d_gbuf);
    VPL_LAUNCHED("k_gbuffer");
    return VPL_OK;
}

int32_t vpl_gather_bytes(int32_t n_vpls, int32_t width, int32_t height, size_t* work_bytes) {
    if (!work_bytes || n_vpls < 0 || width < 0 || height < 0) return VPL_EINVAL;
    GatherWork w;
    *work_bytes = gather_layout(n_vpls, width, height, nullptr, &w);
    return VPL_OK;
}

static int32_t gather_impl(const void* d_scene, const void* d_bvh, const vpl_gpoint* d_gbuf, const vpl_record* d_vpls,
                           int32_t n_vpls, const int32_t* d_tiles, int32_t n_tiles, int32_t tile_w, int32_t tile_h,
                           float* d_rgb, vpl_counters* d_ctr, void* d_work, size_t work_bytes, void* stream,
                           GatherDump dump, int32_t flags = 0) {
    if (!d_scene || !d_bvh || !d_gbuf || !d_rgb || !d_work || n_vpls < 0 || (n_vpls > 0 && !d_vpls)) {
        set_error("vpl_gather_indirect: bad arguments");
        return VPL_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    SceneHdr hh;
    VPL_TRY(read_scene_hdr(d_scene, s, &hh));
    GatherWork w;
    if (work_bytes < gather_layout(n_vpls, hh.W, hh.H, nullptr, &w)) {
        set_error("vpl_gather_indirect: work buffer smaller than vpl_gather_bytes(n_vpls, W, H)");
        return VPL_ESMALL;
    }
    gather_layout(n_vpls, hh.W, hh.H, (char*)d_work, &w);
    int32_t chunk, n_chunks;
    gather_chunks(n_vpls, &chunk, &n_chunks);
    TileMap tm;
    VPL_TRY(make_tilemap(hh, d_tiles, n_tiles, tile_w, tile_h, &tm));
    tm.bh = 4 * kSeg;   // warps cover 8 x 4kSeg blocks (rows past a tile's end are masked)
    tm.blocks_per_tile = (tile_w / 8) * ((tile_h + tm.bh - 1) / tm.bh);
    if (n_tiles == 0) return VPL_OK;
    int* queue = w.queue;
    VPL_CUDA(cudaMemsetAsync(queue, 0, sizeof(int), s));
    if (n_chunks > 1) {
        VPL_CUDA(cudaMemsetAsync(w.done, 0, sizeof(int) * (size_t)w.ring, s));
        VPL_CUDA(cudaMemsetAsync(w.slot_gen, 0, sizeof(int) * (size_t)w.ring, s));
    }
    const vpl_record* vp = d_vpls;
    dump.perm = nullptr;
    if (n_vpls > 1) {
        const unsigned init[6] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0u, 0u, 0u};
        VPL_CUDA(cudaMemcpyAsync(w.box, init, sizeof(init), cudaMemcpyHostToDevice, s));
        k_vpl_bbox<<<nb(n_vpls, 256), 256, 0, s>>>(d_vpls, n_vpls, w.box);
        VPL_LAUNCHED("k_vpl_bbox");
        k_vpl_morton<<<nb(n_vpls, 256), 256, 0, s>>>(d_vpls, n_vpls, w.box, w.keys, w.idx);
        VPL_LAUNCHED("k_vpl_morton");
        size_t cb = w.cub_bytes;
        VPL_CUDA(cub::DeviceRadixSort::SortPairs(w.cub, cb, w.keys, w.keys2, w.idx, w.idx2, n_vpls, 0, 30, s));
        k_vpl_permute<<<nb(n_vpls, 256), 256, 0, s>>>(d_vpls, w.idx2, n_vpls, w.sorted);
        VPL_LAUNCHED("k_vpl_permute");
        vp = w.sorted;
        dump.perm = w.idx2;
    }
    const float4* clusters = nullptr;
#if VPL_CLUSTER_CULL
    if (n_vpls > 0 && !(flags & VPL_GATHER_NO_CULL)) {
        const int ncl = (n_vpls + kCluster - 1) / kCluster;
        k_vpl_clusters<<<nb(ncl, 128), 128, 0, s>>>(vp, n_vpls, w.clusters);
        VPL_LAUNCHED("k_vpl_clusters");
        clusters = w.clusters;
    }
#endif
    int dev = 0, sms = 148;
    VPL_CUDA(cudaGetDevice(&dev));
    VPL_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    int grid = sms * VPL_GATHER_CTAS;  // persistent: VPL_GATHER_CTAS one-warp CTAs per SM
    // whole-block tasks for all but the last VPL_TAIL_BLOCKS x grid blocks of the call (the chunked tail balances
    // the SMs; a rank with fewer blocks than that runs chunked tasks only, as does a dump run)
    const int64_t nblk = tm.n_warps();
    int64_t n_whole = n_chunks == 1 ? nblk : nblk - (int64_t)VPL_TAIL_BLOCKS * grid;
    if (n_whole < 0 || (VPL_TAIL_BLOCKS < 0 && n_chunks > 1)) n_whole = 0;
    if (n_whole > INT32_MAX) n_whole = INT32_MAX;
    SceneView sv = scene_view(d_scene, hh.n);
    BvhView bv = bvh_view(d_bvh, hh.n);
    bv.box_pad = hh.box_pad;
    if (flags & VPL_GATHER_NO_CULL) bv.planes = nullptr;   // reference run: no cluster cull, no lists, no plane-side cull
#ifdef VPL_CARVEOUT
    // shared-memory carveout preference (percent of the unified L1/shared array; tuning builds only)
    VPL_CUDA(cudaFuncSetAttribute(k_gather<false>, cudaFuncAttributePreferredSharedMemoryCarveout, VPL_CARVEOUT));
    VPL_CUDA(cudaFuncSetAttribute(k_gather<true>, cudaFuncAttributePreferredSharedMemoryCarveout, VPL_CARVEOUT));
#endif
    if (dump.slot)
        k_gather<true, true><<<grid, 32, 0, s>>>(sv, bv, tm, d_gbuf, vp, n_vpls, d_rgb, d_ctr, queue, clusters, chunk,
                                                  n_chunks, w.part, w.done, w.slot_gen, w.ring, (int32_t)n_whole, dump);
    else if (d_ctr)
        k_gather<true><<<grid, 32, 0, s>>>(sv, bv, tm, d_gbuf, vp, n_vpls, d_rgb, d_ctr, queue, clusters, chunk,
                                            n_chunks, w.part, w.done, w.slot_gen, w.ring, (int32_t)n_whole, dump);
    else
        k_gather<false><<<grid, 32, 0, s>>>(sv, bv, tm, d_gbuf, vp, n_vpls, d_rgb, nullptr, queue, clusters, chunk,
                                             n_chunks, w.part, w.done, w.slot_gen, w.ring, (int32_t)n_whole, dump);
    VPL_LAUNCHED("k_gather");

    return VPL_OK;
}

int32_t vpl_gather_indirect(const void* d_scene, const void* d_bvh, const vpl_gpoint* d_gbuf, const vpl_record* d_vpls,
                            int32_t n_vpls, const int32_t* d_tiles, int32_t n_tiles, int32_t tile_w, int32_t tile_h,
                            float* d_rgb, vpl_counters* d_ctr, void* d_work, size_t work_bytes, void* stream) {
    GatherDump dump{nullptr, nullptr, nullptr, nullptr, 0};
    return gather_impl(d_scene, d_bvh, d_gbuf, d_vpls, n_vpls, d_tiles, n_tiles, tile_w, tile_h, d_rgb, d_ctr, d_work,
                       work_bytes, stream, dump);
}

int32_t vpl_gather_dump(const void* d_scene, const void* d_bvh, const vpl_gpoint* d_gbuf, const vpl_record* d_vpls,
                        int32_t n_vpls, const int32_t* d_tiles, int32_t n_tiles, int32_t tile_w, int32_t tile_h,
                        float* d_rgb, vpl_counters* d_ctr, void* d_work, size_t work_bytes,
                        const int32_t* d_pixel_slot, uint32_t* d_traced_bits, uint32_t* d_vis_bits, int32_t flags,
                        void* stream) {
    if ((d_pixel_slot && (!d_traced_bits || !d_vis_bits)) || n_vpls <= 0 || (flags & ~VPL_GATHER_NO_CULL)) {
        set_error("vpl_gather_dump: bad arguments");
        return VPL_EINVAL;
    }
    GatherDump dump{d_pixel_slot, nullptr, d_traced_bits, d_vis_bits, (n_vpls + 31) / 32};
    return gather_impl(d_scene, d_bvh, d_gbuf, d_vpls, n_vpls, d_tiles, n_tiles, tile_w, tile_h, d_rgb, d_ctr, d_work,
                       work_bytes, stream, dump, flags);
}


int32_t vpl_render_direct(const void* d_scene, const void* d_bvh, const vpl_gpoint* d_gbuf, const int32_t* d_tiles,
                          int32_t n_tiles, int32_t tile_w, int32_t tile_h, int32_t samples, uint64_t seed,
                          int32_t accumulate, float* d_rgb, void* stream) {
    if (!d_scene || !d_bvh || !d_gbuf || !d_rgb || samples <= 0) {
        set_error("vpl_render_direct: bad arguments");
        return VPL_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    SceneHdr hh;
    VPL_TRY(read_scene_hdr(d_scene, s, &hh));
    TileMap tm;
    VPL_TRY(make_tilemap(hh, d_tiles, n_tiles, tile_w, tile_h, &tm));
    if (n_tiles == 0) return VPL_OK;
    const float inv_S = (float)(1.0 / (double)samples);
    int64_t threads = tm.n_warps() * 32;
    k_direct<<<nb(threads, 128), 128, 0, s>>>(scene_view(d_scene, hh.n), bvh_view(d_bvh, hh.n), tm, d_gbuf, samples,
                                             seed, inv_S, accumulate, d_rgb);
    VPL_LAUNCHED("k_direct");
    return VPL_OK;
}

int32_t vpl_image_error(const float* d_img, const float* d_ref, int64_t n, double* d_out, void* d_work,
                        size_t work_bytes, void* stream) {
    if (!d_out || !d_work || n < 0 || (n > 0 && (!d_img || !d_ref))) {
        set_error("vpl_image_error: bad arguments");
        return VPL_EINVAL;
    }
    if (work_bytes < sizeof(double) * 4 * kErrBlocks) { set_error("vpl_image_error: work too small"); return VPL_ESMALL; }
    cudaStream_t s = (cudaStream_t)stream;
    k_image_err<<<kErrBlocks, kErrThreads, 0, s>>>(d_img, d_ref, n, (double*)d_work);
    VPL_LAUNCHED("k_image_err");
    k_image_err_final<<<1, 32, 0, s>>>((const double*)d_work, kErrBlocks, d_out);
    VPL_LAUNCHED("k_image_err_final");
    return VPL_OK;
}

int32_t vpl_visibility_dump(const void* d_scene, const void* d_bvh, const vpl_gpoint* d_gbuf, const vpl_record* d_vpls,
                            int32_t n_vpls, const int32_t* d_pixels, int32_t n_pixels, uint32_t* d_traced_bits,
                            uint32_t* d_vis_bits, void* stream) {
    if (!d_scene || !d_bvh || !d_gbuf || !d_pixels || !d_traced_bits || !d_vis_bits || n_vpls <= 0 || n_pixels < 0)
        return VPL_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    SceneHdr hh;
    VPL_TRY(read_scene_hdr(d_scene, s, &hh));
    if (n_pixels == 0) return VPL_OK;
    BvhView bv = bvh_view(d_bvh, hh.n);
    bv.box_pad = hh.box_pad;   // margin of the plane-side cull
    k_visdump<<<nb(n_pixels, 64), 64, 0, s>>>(scene_view(d_scene, hh.n), bv, d_gbuf, d_vpls, n_vpls, d_pixels, n_pixels,
                                           d_traced_bits, d_vis_bits);
    VPL_LAUNCHED("k_visdump");
    return VPL_OK;
}

int32_t vpl_closest_hit_batch(const void* d_scene, const void* d_bvh, const float* d_o, const float* d_dir, int64_t n,
                              float tmin, float tmax, int32_t* d_tri, float* d_t, void* stream) {
    if (!d_scene || !d_bvh || !d_o || !d_dir || !d_tri || !d_t || n < 0) return VPL_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    SceneHdr hh;
    VPL_TRY(read_scene_hdr(d_scene, s, &hh));
    if (n == 0) return VPL_OK;
    k_closest_batch<<<nb(n, 128), 128, 0, s>>>(bvh_view(d_bvh, hh.n), d_o, d_dir, n, tmin, tmax, d_tri, d_t);
    VPL_LAUNCHED("k_closest_batch");
    return VPL_OK;
}

int32_t vpl_occluded_batch(const void* d_scene, const void* d_bvh, const float* d_a, const float* d_b, int64_t n,
                           uint8_t* d_occ, void* stream) {
    if (!d_scene || !d_bvh || !d_a || !d_b || !d_occ || n < 0) return VPL_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    SceneHdr hh;
    VPL_TRY(read_scene_hdr(d_scene, s, &hh));
    if (n == 0) return VPL_OK;
    k_occluded_batch<<<nb(n, 128), 128, 0, s>>>(scene_view(d_scene, hh.n), bvh_view(d_bvh, hh.n), d_a, d_b, n, d_occ);
    VPL_LAUNCHED("k_occluded_batch");
    return VPL_OK;
}

int32_t vpl_philox_batch(const uint32_t* d_in, int64_t n, uint32_t* d_out, void* stream) {
    if (!d_in || !d_out || n < 0) return VPL_EINVAL;
    if (n == 0) return VPL_OK;
    k_philox_batch<<<nb(n, 128), 128, 0, (cudaStream_t)stream>>>(d_in, n, d_out);
    VPL_LAUNCHED("k_philox_batch");
    return VPL_OK;
}

}  // extern "C"
