// reject.cu — NEXT f3, the rejection-sampling comparator (P:29-32 [r3]:
// "reject those VPLs that contribute less than the average value to the
// resulting image"; SPEC generate_rejection_vpls S:252-260; O15,
// reading R23).  Input: a pilot VPL set (plain IR: vpl_generate_vpls with every
// patch FAR).  Each candidate is scored by its Eq. 1 summand at 64 probe
// pixels (luminance, exact fp32 in probe order, exact visibility); candidate
// i is accepted with probability p_i = max(0.05, min(1, s_i / mean)) (Philox
// stream 6), scanning in index order until the budget is met, and its flux is
// weighted by (pilot / scanned) / p_i.  Every decision is taken on the same
// fp32 scores and fp64 arithmetic as the oracle, so the output is bitwise the
// oracle's.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "common.cuh"

namespace vplgi {

constexpr int kProbes = 64;

// probe b: block (b % 8, b / 8) of an 8 x 8 grid, offset floor(U(draw 0/1 of stream 5, item b) * size)
__global__ void k_probe_points(SceneView sv, BvhView bv, uint64_t seed, int32_t* __restrict__ pix,
                               vpl_gpoint* __restrict__ probes) {
    int b = threadIdx.x;
    if (b >= kProbes) return;
    const int W = sv.hdr->W, H = sv.hdr->H;
    int bx = b % 8, by = b / 8;
    int x0 = bx * W / 8, x1 = (bx + 1) * W / 8, y0 = by * H / 8, y1 = (by + 1) * H / 8;
    Philox ph(seed, 5u, (uint32_t)b);
    float u = u01(ph.at(0)), v = u01(ph.at(1));
    int px = x0 + (int)(u * (float)(x1 - x0));
    int py = y0 + (int)(v * (float)(y1 - y0));
    int p = py * W + px;
    pix[b] = p;
    probes[b] = primary_hit(sv, bv, p);
}

__device__ __forceinline__ float lum3(float a, float b, float c) { return ((a + b) + c) / 3.0f; }

// warp per candidate: lane q and q + 32 evaluate probes q, q + 32; lane 0 adds
// the 64 terms in probe order (the oracle's fp32 sequence)
__global__ void __launch_bounds__(128) k_reject_score(SceneView sv, BvhView bv, const vpl_gpoint* __restrict__ probes,
                                                      const vpl_record* __restrict__ pilot, int64_t np_,
                                                      float* __restrict__ scores) {
    __shared__ vpl_gpoint sp[kProbes];
    for (int k = threadIdx.x; k < kProbes; k += blockDim.x) sp[k] = probes[k];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const float eps = sv.hdr->eps, b2 = sv.hdr->b2;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < np_; i += nwarps) {
        const float4* v = (const float4*)(pilot + i);
        const float4 a = __ldg(v), bn = __ldg(v + 1), fl = __ldg(v + 2);
        const f3 y = xyz(a), ny = xyz(bn);
        const int tri_i = __float_as_int(a.w);
        const float li = lum3(fl.x, fl.y, fl.z);
        float t2[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const vpl_gpoint& g = sp[lane + 32 * h];
            float t = 0.0f;
            if (g.tri >= 0 && g.front && g.tri != tri_i) {
                const f3 x = ld3(g.pos), nx = ld3(g.nrm);
                const f3 d = y - x;
                const float r2 = dot(d, d);
                const float cx = dot(nx, d);
                const float ci = -dot(ny, d);
                if (cx > 0.0f && ci > 0.0f && !segment_occluded<false>(bv, x, y, eps, nullptr)) {
                    const float w = (cx * ci) / (r2 * (r2 > b2 ? r2 : b2));
                    t = (w * li) * lum3(g.alb[0], g.alb[1], g.alb[2]);
                }
            }
            t2[h] = t;
        }
        float acc = 0.0f;
#pragma unroll
        for (int h = 0; h < 2; ++h)
            for (int q = 0; q < 32; ++q) acc += __shfl_sync(0xFFFFFFFFu, t2[h], q);
        if (lane == 0) scores[i] = acc;
    }
}

// fp64 sum of the scores in index order (the oracle's sequence), one thread
__global__ void k_reject_mean(const float* __restrict__ scores, int64_t np_, double* __restrict__ mean) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double s = 0.0;
    for (int64_t i = 0; i < np_; ++i) s += (double)scores[i];
    *mean = np_ > 0 ? s / (double)np_ : 0.0;
}

constexpr double kRejPMin = 0.05;

// p_i = max(P_MIN, min(1, s_i / mean)) (fp64), accept iff (double)U(stream 6, item i, draw 0) < p_i
__global__ void k_reject_accept(const float* __restrict__ scores, int64_t np_, const double* __restrict__ mean,
                                uint64_t seed, int32_t* __restrict__ flag, double* __restrict__ prob,
                                int64_t* __restrict__ scanned) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i == 0) *scanned = np_;
    if (i >= np_) return;
    const double m = *mean;
    double p = m > 0.0 ? (double)scores[i] / m : 1.0;
    if (p > 1.0) p = 1.0;
    if (p < kRejPMin) p = kRejPMin;
    Philox ph(seed, 6u, (uint32_t)i);
    const double u = (double)u01(ph.at(0));
    flag[i] = u < p;
    prob[i] = p;
}

// the scanned prefix ends at the budget-th acceptance (unique)
__global__ void k_reject_prefix(const int32_t* __restrict__ flag, const int32_t* __restrict__ pos, int64_t np_,
                                int64_t B, int64_t* __restrict__ scanned, int64_t* __restrict__ accepted) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= np_) return;
    if (i == np_ - 1) {
        const int64_t tot = (int64_t)pos[i] + flag[i];
        *accepted = tot < B ? tot : B;
    }
    if (flag[i] && pos[i] == B - 1) *scanned = i + 1;
}

__global__ void k_reject_emit(const vpl_record* __restrict__ pilot, int64_t np_, int64_t B,
                              const int32_t* __restrict__ flag, const int32_t* __restrict__ pos,
                              const double* __restrict__ prob, const int64_t* __restrict__ scanned,
                              vpl_record* __restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= np_ || !flag[i] || pos[i] >= B) return;
    const float f = (float)(((double)np_ / (double)*scanned) / prob[i]);
    const float4* s4 = (const float4*)(pilot + i);
    float4* d4 = (float4*)(out + pos[i]);
    const float4 c = s4[2];
    d4[0] = s4[0];
    d4[1] = s4[1];
    d4[2] = make_float4(c.x * f, c.y * f, c.z * f, c.w);
}

// ---------------------------------------------------------------- NEXT f4: Metropolis comparator (O16)
// pool = the pilot along its Morton curve (O4's quantisation over the pilot position box)
__global__ void k_mh_bbox(const vpl_record* __restrict__ v, int64_t n, unsigned* __restrict__ box) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float* p = (const float*)(v + i);
    for (int a = 0; a < 3; ++a) {
        atomicMin(box + a, (unsigned)fkey(p[a]) ^ 0x80000000u);
        atomicMax(box + 3 + a, (unsigned)fkey(p[a]) ^ 0x80000000u);
    }
}
__device__ __forceinline__ uint32_t morton3_10(uint32_t qx, uint32_t qy, uint32_t qz) {
    uint32_t c = 0;
    for (int b = 0; b < 10; ++b)
        c |= (((qx >> b) & 1u) << (3 * b)) | (((qy >> b) & 1u) << (3 * b + 1)) | (((qz >> b) & 1u) << (3 * b + 2));
    return c;
}
__global__ void k_mh_morton(const vpl_record* __restrict__ v, int64_t n, const unsigned* __restrict__ box,
                            uint32_t* __restrict__ key, int32_t* __restrict__ idx) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float* p = (const float*)(v + i);
    uint32_t q[3];
    for (int a = 0; a < 3; ++a) {
        const float lo = fkey_inv((int)(box[a] ^ 0x80000000u)), hi = fkey_inv((int)(box[3 + a] ^ 0x80000000u));
        const float ext = hi - lo;
        const float scale = ext > 0.0f ? 1024.0f / ext : 0.0f;
        const uint32_t qa = (uint32_t)((p[a] - lo) * scale);
        q[a] = qa < 1023u ? qa : 1023u;
    }
    key[i] = morton3_10(q[0], q[1], q[2]);
    idx[i] = (int32_t)i;
}
// f_j = max(s_pool[j], 0.05 mean) (1 if mean = 0); mean_f = fp64 sum in pool order / n (one thread)
__global__ void k_mh_target(const float* __restrict__ scores, const int32_t* __restrict__ pool, int64_t n,
                            const double* __restrict__ mean, double* __restrict__ f) {
    int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= n) return;
    const double m = *mean;
    const double v = m > 0.0 ? (double)scores[pool[j]] : 1.0;
    const double fl = 0.05 * m;
    f[j] = v > fl ? v : fl;
}
__global__ void k_mh_meanf(const double* __restrict__ f, int64_t n, double* __restrict__ mean_f) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double t = 0.0;
    for (int64_t j = 0; j < n; ++j) t += f[j];
    *mean_f = t / (double)n;
}
// one thread per chain (Philox stream 7, item = chain, draws in sequence); mutations: a large
// step (probability 0.3) to a uniform pool index, else a local step along the Morton curve
__global__ void k_mh_chains(const vpl_record* __restrict__ pilot, const int32_t* __restrict__ pool,
                            const double* __restrict__ f, const double* __restrict__ mean_f, int64_t n,
                            int64_t chains, int64_t per_chain, int64_t burn, int64_t R, uint64_t seed,
                            vpl_record* __restrict__ out, unsigned long long* __restrict__ accepted) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= chains) return;
    Philox ph(seed, 7u, (uint32_t)c);
    const uint32_t x0 = ph.next();
    int64_t cur = (int64_t)(((uint64_t)x0 * (uint64_t)n) >> 32);
    const double scale = (double)n / (double)(chains * per_chain);
    const double mf = *mean_f;
    unsigned long long acc = 0;
    for (int64_t t = 0; t < burn + per_chain; ++t) {
        const double sel = (double)u01(ph.next());
        const uint32_t xk = ph.next();
        int64_t nxt;
        if (sel < 0.3) {                            // large step: uniform over the pool
            nxt = (int64_t)(((uint64_t)xk * (uint64_t)n) >> 32);
        } else {                                    // small step: local Morton neighbour
            const int64_t k = (int64_t)(((uint64_t)xk * (uint64_t)(2 * R)) >> 32);
            const int64_t delta = k < R ? k - R : k - R + 1;
            nxt = ((cur + delta) % n + n) % n;
        }
        const double u = (double)u01(ph.next());
        if (u < f[nxt] / f[cur]) { cur = nxt; ++acc; }
        if (t >= burn) {
            const float w = (float)(scale * (mf / f[cur]));
            const float4* s4 = (const float4*)(pilot + pool[cur]);
            float4* d4 = (float4*)(out + c * per_chain + (t - burn));
            const float4 fl = s4[2];
            d4[0] = s4[0];
            d4[1] = s4[1];
            d4[2] = make_float4(fl.x * w, fl.y * w, fl.z * w, fl.w);
        }
    }
    atomicAdd(accepted, acc);
}

struct RejectWork {
    int32_t* probe_pix;
    vpl_gpoint* probes;
    float* scores;
    double *mean, *prob, *mean_f;
    int64_t* scanned;
    int32_t *flag, *pos, *idx, *pool;
    uint32_t *key, *key2;
    unsigned* box;
    void* cub;
    size_t cub_bytes;
};

static size_t reject_layout(int64_t np_, char* base, RejectWork* w) {
    Bump b{base};
    size_t m = (size_t)(np_ > 0 ? np_ : 1);
    w->probe_pix = b.take<int32_t>(kProbes);
    w->probes = b.take<vpl_gpoint>(kProbes);
    w->scores = b.take<float>(m);
    w->mean = b.take<double>(1);
    w->prob = b.take<double>(m);
    w->scanned = b.take<int64_t>(1);
    w->mean_f = b.take<double>(1);
    w->flag = b.take<int32_t>(m);
    w->pos = b.take<int32_t>(m);
    w->idx = b.take<int32_t>(m);
    w->pool = b.take<int32_t>(m);
    w->key = b.take<uint32_t>(m);
    w->key2 = b.take<uint32_t>(m);
    w->box = b.take<unsigned>(8);
    size_t c1 = 0, c2 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, c1, (int32_t*)nullptr, (int32_t*)nullptr, (int)m);
    cub::DeviceRadixSort::SortPairs(nullptr, c2, (uint32_t*)nullptr, (uint32_t*)nullptr, (int32_t*)nullptr,
                                    (int32_t*)nullptr, (int)m, 0, 30);
    w->cub_bytes = c1 > c2 ? c1 : c2;
    w->cub = b.take<char>(w->cub_bytes);
    return b.off;
}

static inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t); }

}  // namespace vplgi

using namespace vplgi;

extern "C" {

int32_t vpl_rejection_bytes(int64_t n_pilot, size_t* work_bytes) {
    if (!work_bytes || n_pilot < 0 || n_pilot > INT32_MAX) return VPL_EINVAL;
    RejectWork w;
    *work_bytes = reject_layout(n_pilot, nullptr, &w);
    return VPL_OK;
}

int32_t vpl_generate_rejection(const void* d_scene, const void* d_bvh, const vpl_record* d_pilot, int64_t n_pilot,
                               int64_t budget, uint64_t seed, vpl_record* d_out, float* d_scores, double* d_mean,
                               int64_t* d_accepted, int64_t* d_scanned, int32_t* d_probe_pixels, void* d_work,
                               size_t work_bytes, void* stream) {
    if (!d_scene || !d_bvh || !d_out || !d_accepted || !d_work || n_pilot <= 0 || n_pilot > INT32_MAX ||
        budget <= 0 || !d_pilot) {
        set_error("vpl_generate_rejection: bad arguments");
        return VPL_EINVAL;
    }
    RejectWork w;
    if (work_bytes < reject_layout(n_pilot, nullptr, &w)) {
        set_error("vpl_generate_rejection: work smaller than vpl_rejection_bytes(n_pilot)");
        return VPL_ESMALL;
    }
    reject_layout(n_pilot, (char*)d_work, &w);
    cudaStream_t s = (cudaStream_t)stream;
    SceneHdr hh;
    VPL_TRY(read_scene_hdr(d_scene, s, &hh));
    SceneView sv = scene_view(d_scene, hh.n);
    BvhView bv = bvh_view(d_bvh, hh.n);
    const int64_t B = budget < n_pilot ? budget : n_pilot;
    float* scores = d_scores ? d_scores : w.scores;
    double* mean = d_mean ? d_mean : w.mean;
    int64_t* scanned = d_scanned ? d_scanned : w.scanned;

    k_probe_points<<<1, kProbes, 0, s>>>(sv, bv, seed, w.probe_pix, w.probes);
    VPL_LAUNCHED("k_probe_points");
    if (d_probe_pixels) VPL_CUDA(cudaMemcpyAsync(d_probe_pixels, w.probe_pix, sizeof(int32_t) * kProbes,
                                                 cudaMemcpyDeviceToDevice, s));
    int dev = 0, sms = 148;
    VPL_CUDA(cudaGetDevice(&dev));
    VPL_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int64_t want = (n_pilot + 3) / 4, cap = (int64_t)sms * 16;
    const int grid = (int)(want < cap ? want : cap);
    k_reject_score<<<grid, 128, 0, s>>>(sv, bv, w.probes, d_pilot, n_pilot, scores);
    VPL_LAUNCHED("k_reject_score");
    k_reject_mean<<<1, 32, 0, s>>>(scores, n_pilot, mean);
    VPL_LAUNCHED("k_reject_mean");
    k_reject_accept<<<nblk(n_pilot, 256), 256, 0, s>>>(scores, n_pilot, mean, seed, w.flag, w.prob, scanned);
    VPL_LAUNCHED("k_reject_accept");
    size_t cb = w.cub_bytes;
    VPL_CUDA(cub::DeviceScan::ExclusiveSum(w.cub, cb, w.flag, w.pos, (int)n_pilot, s));
    k_reject_prefix<<<nblk(n_pilot, 256), 256, 0, s>>>(w.flag, w.pos, n_pilot, B, scanned, d_accepted);
    VPL_LAUNCHED("k_reject_prefix");
    k_reject_emit<<<nblk(n_pilot, 256), 256, 0, s>>>(d_pilot, n_pilot, B, w.flag, w.pos, w.prob, scanned, d_out);
    VPL_LAUNCHED("k_reject_emit");
    return VPL_OK;
}

int32_t vpl_generate_metropolis(const void* d_scene, const void* d_bvh, const vpl_record* d_pilot, int64_t n_pilot,
                                int64_t chains, int64_t per_chain, int64_t burn, int64_t radius, uint64_t seed,
                                vpl_record* d_out, float* d_scores, int32_t* d_pool, uint64_t* d_accepted,
                                void* d_work, size_t work_bytes, void* stream) {
    if (!d_scene || !d_bvh || !d_pilot || !d_out || !d_accepted || !d_work || n_pilot < 2 || n_pilot > INT32_MAX ||
        chains < 1 || per_chain < 1 || burn < 0 || radius < 1 || radius > INT32_MAX) {
        set_error("vpl_generate_metropolis: bad arguments");
        return VPL_EINVAL;
    }
    RejectWork w;
    if (work_bytes < reject_layout(n_pilot, nullptr, &w)) {
        set_error("vpl_generate_metropolis: work smaller than vpl_rejection_bytes(n_pilot)");
        return VPL_ESMALL;
    }
    reject_layout(n_pilot, (char*)d_work, &w);
    cudaStream_t s = (cudaStream_t)stream;
    SceneHdr hh;
    VPL_TRY(read_scene_hdr(d_scene, s, &hh));
    SceneView sv = scene_view(d_scene, hh.n);
    BvhView bv = bvh_view(d_bvh, hh.n);
    float* scores = d_scores ? d_scores : w.scores;
    k_probe_points<<<1, kProbes, 0, s>>>(sv, bv, seed, w.probe_pix, w.probes);
    VPL_LAUNCHED("k_probe_points");
    int dev = 0, sms = 148;
    VPL_CUDA(cudaGetDevice(&dev));
    VPL_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int64_t want = (n_pilot + 3) / 4, cap = (int64_t)sms * 16;
    k_reject_score<<<(int)(want < cap ? want : cap), 128, 0, s>>>(sv, bv, w.probes, d_pilot, n_pilot, scores);
    VPL_LAUNCHED("k_reject_score");
    k_reject_mean<<<1, 32, 0, s>>>(scores, n_pilot, w.mean);
    VPL_LAUNCHED("k_reject_mean");
    const unsigned init[6] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0u, 0u, 0u};
    VPL_CUDA(cudaMemcpyAsync(w.box, init, sizeof(init), cudaMemcpyHostToDevice, s));
    k_mh_bbox<<<nblk(n_pilot, 256), 256, 0, s>>>(d_pilot, n_pilot, w.box);
    VPL_LAUNCHED("k_mh_bbox");
    k_mh_morton<<<nblk(n_pilot, 256), 256, 0, s>>>(d_pilot, n_pilot, w.box, w.key, w.idx);
    VPL_LAUNCHED("k_mh_morton");
    size_t cb = w.cub_bytes;
    VPL_CUDA(cub::DeviceRadixSort::SortPairs(w.cub, cb, w.key, w.key2, w.idx, w.pool, (int)n_pilot, 0, 30, s));
    if (d_pool) VPL_CUDA(cudaMemcpyAsync(d_pool, w.pool, sizeof(int32_t) * n_pilot, cudaMemcpyDeviceToDevice, s));
    k_mh_target<<<nblk(n_pilot, 256), 256, 0, s>>>(scores, w.pool, n_pilot, w.mean, w.prob);
    VPL_LAUNCHED("k_mh_target");
    k_mh_meanf<<<1, 32, 0, s>>>(w.prob, n_pilot, w.mean_f);
    VPL_LAUNCHED("k_mh_meanf");
    VPL_CUDA(cudaMemsetAsync(d_accepted, 0, sizeof(uint64_t), s));
    k_mh_chains<<<nblk(chains, 64), 64, 0, s>>>(d_pilot, w.pool, w.prob, w.mean_f, n_pilot, chains, per_chain, burn,
                                                radius, seed, d_out, (unsigned long long*)d_accepted);
    VPL_LAUNCHED("k_mh_chains");
    return VPL_OK;
}

}  // extern "C"
