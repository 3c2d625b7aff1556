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

struct RejectWork {
    int32_t* probe_pix;
    vpl_gpoint* probes;
    float* scores;
    double *mean, *prob;
    int64_t* scanned;
    int32_t *flag, *pos;
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
    w->flag = b.take<int32_t>(m);
    w->pos = b.take<int32_t>(m);
    size_t c1 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, c1, (int32_t*)nullptr, (int32_t*)nullptr, (int)m);
    w->cub_bytes = c1;
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

}  // extern "C"
