// generate.cu — a4-a6 generate_vpls: the paper's hybrid VPL generation
// (P:44-65 near part: light-visible filter, Morton order, area prefix f and
// its inverse g, K equal-area strata, a uniform point per stratum, Eq. 2
// flux; P:35 / P:46 step 3 far part: sparse instant-radiosity walks keeping
// only far deposits).  Bit-exact with DESIGN.md §3 O3-O11.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include <vector>

#include "common.cuh"

namespace vplgi {

constexpr uint32_t kStreamNear = 0, kStreamWalk = 1;
constexpr double kPi = 3.14159265358979323846;

__device__ __forceinline__ f3 light_corner(const float* L) { return ld3(L); }
__device__ __forceinline__ f3 light_eu(const float* L) { return ld3(L + 3); }
__device__ __forceinline__ f3 light_ev(const float* L) { return ld3(L + 6); }
__device__ __forceinline__ f3 light_n(const float* L) { return ld3(L + 9); }

__global__ void k_count_labels(const uint8_t* __restrict__ labels, int64_t n, unsigned long long* cnt /*[2]*/) {
    unsigned long long nn = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        nn += labels[i] != 0;
    for (int o = 16; o > 0; o >>= 1) nn += __shfl_xor_sync(0xFFFFFFFFu, nn, o);
    if ((threadIdx.x & 31) == 0 && nn) atomicAdd(cnt, nn);
}

// O3 — lit <=> near, facing some light, centroid -> light centre unoccluded (R6)
__global__ void k_lit(SceneView sv, BvhView bv, const uint8_t* __restrict__ labels, int64_t n,
                      uint8_t* __restrict__ lit) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint8_t r = 0;
    if (labels[i]) {
        const SceneHdr* h = sv.hdr;
        f3 c = xyz(sv.cen[i]), nn = xyz(sv.nrm[i]);
        float eps = h->eps;
        for (int l = 0; l < h->nL && !r; ++l) {
            const float* L = h->lights + 16 * l;
            f3 cl = (light_corner(L) + 0.5f * light_eu(L)) + 0.5f * light_ev(L);
            if (dot(nn, cl - c) > 0.0f && (light_is_point(L) || dot(light_n(L), c - cl) > 0.0f) &&
                !segment_occluded<false>(bv, c, cl, eps, nullptr))
                r = 1;
        }
    }
    lit[i] = r;
}

__device__ __forceinline__ uint32_t fenc(float f) {
    uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float fdec(uint32_t u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u);
}

__global__ void k_init_bbox(uint32_t* enc) {
    if (threadIdx.x < 3) { enc[threadIdx.x] = 0xFFFFFFFFu; enc[3 + threadIdx.x] = 0u; }
}

__global__ void k_lit_bbox(SceneView sv, const int32_t* __restrict__ lit_idx, const int32_t* __restrict__ d_m,
                           uint32_t* __restrict__ enc) {
    int64_t m = *d_m;
    uint32_t lo[3] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu}, hi[3] = {0u, 0u, 0u};
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x) {
        float4 c = sv.cen[lit_idx[j]];
        float cc[3] = {c.x, c.y, c.z};
        for (int a = 0; a < 3; ++a) {
            uint32_t e = fenc(cc[a]);
            lo[a] = min(lo[a], e);
            hi[a] = max(hi[a], e);
        }
    }
    for (int a = 0; a < 3; ++a)
        for (int o = 16; o > 0; o >>= 1) {
            lo[a] = min(lo[a], __shfl_xor_sync(0xFFFFFFFFu, lo[a], o));
            hi[a] = max(hi[a], __shfl_xor_sync(0xFFFFFFFFu, hi[a], o));
        }
    if ((threadIdx.x & 31) == 0)
        for (int a = 0; a < 3; ++a) { atomicMin(enc + a, lo[a]); atomicMax(enc + 3 + a, hi[a]); }
}

__device__ __forceinline__ uint32_t spread10(uint32_t x) {
    x &= 0x3FFu;
    x = (x | (x << 16)) & 0x030000FFu;
    x = (x | (x << 8)) & 0x0300F00Fu;
    x = (x | (x << 4)) & 0x030C30C3u;
    x = (x | (x << 2)) & 0x09249249u;
    return x;
}

// O4 — 30-bit Morton code over the lit-near centroid bbox
__global__ void k_morton30(SceneView sv, const int32_t* __restrict__ lit_idx, int64_t m,
                           const uint32_t* __restrict__ enc, uint32_t* __restrict__ codes) {
    int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= m) return;
    float4 c = sv.cen[lit_idx[j]];
    float cc[3] = {c.x, c.y, c.z};
    uint32_t q[3];
    for (int a = 0; a < 3; ++a) {
        float lo = fdec(enc[a]), hi = fdec(enc[3 + a]);
        float ext = hi - lo;
        float scale = ext > 0.0f ? 1024.0f / ext : 0.0f;
        uint32_t qa = (uint32_t)((cc[a] - lo) * scale);
        q[a] = qa < 1023u ? qa : 1023u;
    }
    codes[j] = spread10(q[0]) | (spread10(q[1]) << 1) | (spread10(q[2]) << 2);
}

__global__ void k_iota(int32_t* __restrict__ a, int64_t n) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) a[i] = (int32_t)i;
}

__global__ void k_gather_aq(SceneView sv, const int32_t* __restrict__ order, int64_t m, uint64_t* __restrict__ a) {
    int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j < m) a[j] = sv.aq[order[j]];
}

// O6-O8 — one VPL per stratum k (Eq. 2)
__global__ void k_strata(SceneView sv, BvhView bv, const int32_t* __restrict__ order, const uint64_t* __restrict__ P,
                         int64_t m, int64_t K, float D, uint64_t seed, vpl_record* __restrict__ out) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= K) return;
    const SceneHdr* h = sv.hdr;
    uint64_t F = P[m - 1];
    Philox rng(seed, kStreamNear, (uint32_t)k);
    uint32_t x = rng.at(0);
    unsigned __int128 num = ((((unsigned __int128)(uint64_t)k) << 32) + x) * (unsigned __int128)F;
    unsigned __int128 den = ((unsigned __int128)(uint64_t)K) << 32;
    uint64_t sk = (uint64_t)(num / den);
    // g(s_k): first j with P[j] > s_k (upper bound)
    int64_t lo = 0, hi = m - 1;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (P[mid] > sk) hi = mid; else lo = mid + 1;
    }
    int t = order[lo];
    float u1 = u01(rng.at(1)), u2 = u01(rng.at(2));
    const float* v = sv.verts + 9 * (int64_t)t;
    f3 v0 = ld3(v), v1 = ld3(v + 3), v2 = ld3(v + 6);
    float su = sqrtf(u1);
    float b1 = 1.0f - su;
    float b2 = u2 * su;
    float b0 = (1.0f - b1) - b2;
    f3 p = (b1 * v0 + b2 * v1) + b0 * v2;
    f3 nn = xyz(sv.nrm[t]);
    float E[3] = {0.0f, 0.0f, 0.0f};
    float eps = h->eps;
    for (int l = 0; l < h->nL; ++l) {
        const float* L = h->lights + 16 * l;
        float u3 = u01(rng.at(3 + 2 * l)), u4 = u01(rng.at(4 + 2 * l));
        f3 y = (light_corner(L) + u3 * light_eu(L)) + u4 * light_ev(L);
        f3 d = y - p;
        float r2 = dot(d, d);
        float cp = dot(nn, d);
        if (light_is_point(L)) {   // R27: Eq. 2's point form, Phi cos(omega) / (4 pi r^2) V
            if (cp > 0.0f && !segment_occluded<false>(bv, p, y, eps, nullptr)) {
                float g = point_g(cp, r2);
                E[0] += L[13] * g;
                E[1] += L[14] * g;
                E[2] += L[15] * g;
            }
            continue;
        }
        float cl = -dot(light_n(L), d);
        if (cp > 0.0f && cl > 0.0f && !segment_occluded<false>(bv, p, y, eps, nullptr)) {
            float g = ((L[12] * cp) * cl) / (r2 * r2);
            E[0] += L[13] * g;
            E[1] += L[14] * g;
            E[2] += L[15] * g;
        }
    }
    const float INV_PI = (float)(1.0 / kPi);
    float4 a = sv.alb[t];
    vpl_record r;
    r.pos[0] = p.x; r.pos[1] = p.y; r.pos[2] = p.z;
    r.tri = t;
    r.nrm[0] = nn.x; r.nrm[1] = nn.y; r.nrm[2] = nn.z;
    r.tag_depth = 0;
    r.flux[0] = (a.x * (D * E[0])) * INV_PI;
    r.flux[1] = (a.y * (D * E[1])) * INV_PI;
    r.flux[2] = (a.z * (D * E[2])) * INV_PI;
    r.walk = (int32_t)k;
    out[k] = r;
}

// Malley cosine direction with the Duff et al. orthonormal basis (O10)
__device__ __forceinline__ f3 malley(Philox& rng, f3 n) {
    float a = 0.0f, b = 0.0f, q = 0.0f;
    bool found = false;
    for (int att = 0; att < 64; ++att) {
        float ua = u01(rng.next());
        float ub = u01(rng.next());
        a = 2.0f * ua - 1.0f;
        b = 2.0f * ub - 1.0f;
        q = a * a + b * b;
        if (q < 1.0f) { found = true; break; }
    }
    if (!found) { a = 0.0f; b = 0.0f; q = 0.0f; }
    float z = sqrtf(1.0f - q);
    float sg = copysignf(1.0f, n.z);
    float ia = -1.0f / (sg + n.z);
    float bb = (n.x * n.y) * ia;
    f3 t1 = mk3(1.0f + sg * ((n.x * n.x) * ia), sg * bb, -sg * n.x);
    f3 t2 = mk3(bb, sg + (n.y * n.y) * ia, -n.y);
    return mk3((a * t1.x + b * t2.x) + z * n.x, (a * t1.y + b * t2.y) + z * n.y, (a * t1.z + b * t2.z) + z * n.z);
}

// Uniform direction on the sphere for a point light's emission (R27): rejection in the cube,
// a, b, c = 2U - 1 until 0 < a*a + b*b + c*c <= 1 (<= 64 attempts, else (0, 0, 1)); not normalised
__device__ __forceinline__ f3 sphere_dir(Philox& rng) {
    for (int att = 0; att < 64; ++att) {
        float a = 2.0f * u01(rng.next()) - 1.0f;
        float b = 2.0f * u01(rng.next()) - 1.0f;
        float c = 2.0f * u01(rng.next()) - 1.0f;
        float q = (a * a + b * b) + c * c;
        if (q > 0.0f && q <= 1.0f) return mk3(a, b, c);
    }
    return mk3(0.0f, 0.0f, 1.0f);
}

// O10 — one sparse-IR walk per thread (P:15, P:35, P:46 step 3; R9-R11)
__global__ void k_walks(SceneView sv, BvhView bv, const uint8_t* __restrict__ labels, int64_t w0, int64_t nb,
                        int max_depth, int rr, uint64_t seed, vpl_record* __restrict__ dep, int32_t* __restrict__ cnt) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nb) return;
    const SceneHdr* h = sv.hdr;
    uint32_t w = (uint32_t)(w0 + i);
    Philox rng(seed, kStreamWalk, w);
    uint32_t x0 = rng.next();
    int l = (int)(((uint64_t)x0 * (uint64_t)h->nL) >> 32);
    const float* L = h->lights + 16 * l;
    float beta[3];
    // beta0 = power of light l x n_L: pi A L (area light), Phi (point light, R27)
    for (int c = 0; c < 3; ++c)
        beta[c] = light_is_point(L) ? (float)((double)L[13 + c] * (double)h->nL)
                                    : (float)(kPi * (double)L[12] * (double)L[13 + c] * (double)h->nL);
    float u1 = u01(rng.next()), u2 = u01(rng.next());
    f3 o = (light_corner(L) + u1 * light_eu(L)) + u2 * light_ev(L);   // point light: e_u = e_v = 0
    f3 dir = light_is_point(L) ? sphere_dir(rng) : malley(rng, light_n(L));
    const float INV_PI = (float)(1.0 / kPi);
    float eps = h->eps;
    int c_out = 0;
    vpl_record* mine = dep + i * max_depth;
    for (int d = 1; d <= max_depth; ++d) {
        Ray ray = make_ray(o, dir, eps, __int_as_float(0x7f800000));
        float t;
        int hh = bvh_closest(bv, ray, t);
        if (hh < 0) break;
        f3 nh = xyz(sv.nrm[hh]);
        if (dot(nh, dir) >= 0.0f) break;
        f3 x = o + t * dir;
        float4 rho = sv.alb[hh];
        if (!labels[hh]) {
            vpl_record r;
            r.pos[0] = x.x; r.pos[1] = x.y; r.pos[2] = x.z;
            r.tri = hh;
            r.nrm[0] = nh.x; r.nrm[1] = nh.y; r.nrm[2] = nh.z;
            r.tag_depth = 1 | (d << 8);
            r.flux[0] = (rho.x * beta[0]) * INV_PI;
            r.flux[1] = (rho.y * beta[1]) * INV_PI;
            r.flux[2] = (rho.z * beta[2]) * INV_PI;
            r.walk = (int32_t)w;
            mine[c_out++] = r;
        }
        if (d == max_depth) break;
        if (rr) {
            float q = ((rho.x + rho.y) + rho.z) / 3.0f;
            float xi = u01(rng.next());
            if (!(xi < q)) break;
            beta[0] = (beta[0] * rho.x) / q;
            beta[1] = (beta[1] * rho.y) / q;
            beta[2] = (beta[2] * rho.z) / q;
        } else {
            beta[0] = beta[0] * rho.x;
            beta[1] = beta[1] * rho.y;
            beta[2] = beta[2] * rho.z;
        }
        dir = malley(rng, nh);
        o = x;
    }
    cnt[i] = c_out;
}

// copy the first deposits of walks [0, cut] (take_last of walk `cut`) in (w, d) order
__global__ void k_walk_compact(const vpl_record* __restrict__ dep, const int32_t* __restrict__ cnt,
                               const int32_t* __restrict__ off, int64_t nb, int max_depth, int64_t cut, int take_last,
                               vpl_record* __restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nb || i > cut) return;
    int c = cnt[i];
    if (i == cut) c = min(c, take_last);
    for (int k = 0; k < c; ++k) out[off[i] + k] = dep[i * max_depth + k];
}

__global__ void k_div_flux(vpl_record* __restrict__ v, int64_t n, float fw) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    v[i].flux[0] = v[i].flux[0] / fw;
    v[i].flux[1] = v[i].flux[1] / fw;
    v[i].flux[2] = v[i].flux[2] / fw;
}

constexpr int64_t kWalkBatchMax = 1 << 20;

struct GenWork {
    unsigned long long* counts;   // [2]
    uint8_t* lit;
    int32_t* lit_idx;
    int32_t* iota;
    int32_t* d_m;
    uint32_t* enc;                // [6]
    uint32_t *codes, *codes2;
    int32_t* order;
    uint64_t *aq_sorted, *P;
    vpl_record* dep;
    int32_t *cnt, *off;
    void* cub;
    size_t cub_bytes;
};

static size_t gen_layout(int64_t n, int max_depth, char* base, GenWork* w) {
    Bump b{base};
    w->counts = b.take<unsigned long long>(2);
    w->lit = b.take<uint8_t>(n);
    w->lit_idx = b.take<int32_t>(n);
    w->iota = b.take<int32_t>(n);
    w->d_m = b.take<int32_t>(1);
    w->enc = b.take<uint32_t>(6);
    w->codes = b.take<uint32_t>(n);
    w->codes2 = b.take<uint32_t>(n);
    w->order = b.take<int32_t>(n);
    w->aq_sorted = b.take<uint64_t>(n);
    w->P = b.take<uint64_t>(n);
    int md = max_depth > 0 ? max_depth : 1;
    w->dep = b.take<vpl_record>((size_t)kWalkBatchMax * md);
    w->cnt = b.take<int32_t>(kWalkBatchMax);
    w->off = b.take<int32_t>(kWalkBatchMax);
    size_t c1 = 0, c2 = 0, c3 = 0, c4 = 0;
    cub::DeviceSelect::Flagged(nullptr, c1, (int32_t*)nullptr, (uint8_t*)nullptr, (int32_t*)nullptr, (int32_t*)nullptr, (int)n);
    cub::DeviceRadixSort::SortPairs(nullptr, c2, (uint32_t*)nullptr, (uint32_t*)nullptr, (int32_t*)nullptr,
                                    (int32_t*)nullptr, (int)n, 0, 30);
    cub::DeviceScan::InclusiveSum(nullptr, c3, (uint64_t*)nullptr, (uint64_t*)nullptr, (int)n);
    cub::DeviceScan::ExclusiveSum(nullptr, c4, (int32_t*)nullptr, (int32_t*)nullptr, (int)kWalkBatchMax);
    size_t c = c1;
    if (c2 > c) c = c2;
    if (c3 > c) c = c3;
    if (c4 > c) c = c4;
    w->cub_bytes = c;
    w->cub = b.take<char>(c);
    return b.off;
}

static inline int nblk(int64_t n, int t) { return (int)((n + t - 1) / t); }

}  // namespace vplgi

using namespace vplgi;

extern "C" {

int32_t vpl_generate_bytes(const vpl_gen_params* p, int64_t n_tris, int64_t max_out, size_t* work_bytes) {
    if (!p || !work_bytes || n_tris <= 0 || max_out < 0 || p->max_depth < 0 || p->max_depth > 64) return VPL_EINVAL;
    GenWork w;
    *work_bytes = gen_layout(n_tris, (int)p->max_depth, nullptr, &w);
    return VPL_OK;
}

int32_t vpl_generate_vpls(const void* d_scene, const void* d_bvh, const uint8_t* d_labels, const vpl_gen_params* p,
                          vpl_record* d_vpls, int64_t max_out, vpl_gen_info* info, void* d_work, size_t work_bytes,
                          void* stream) {
    if (!d_scene || !d_bvh || !d_labels || !p || !info || !d_work || (max_out > 0 && !d_vpls)) {
        set_error("vpl_generate_vpls: null pointer");
        return VPL_EINVAL;
    }
    if (p->M < 0 || p->K_near < 0 || p->K_near > p->M || p->max_depth < 0 || p->max_depth > 64 ||
        p->n_walks_fixed < 0) {
        set_error("vpl_generate_vpls: bad parameters");
        return VPL_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    SceneHdr hh;
    VPL_TRY(read_scene_hdr(d_scene, s, &hh));
    const int64_t n = hh.n;
    size_t need = 0;
    VPL_TRY(vpl_generate_bytes(p, n, max_out, &need));
    if (work_bytes < need) { set_error("vpl_generate_vpls: work %zu < %zu", work_bytes, need); return VPL_ESMALL; }
    SceneView sv = scene_view(d_scene, n);
    BvhView bv = bvh_view(d_bvh, n);
    GenWork w;
    gen_layout(n, (int)p->max_depth, (char*)d_work, &w);
    memset(info, 0, sizeof(*info));
    const int md = (int)p->max_depth;

    // near / far patch counts
    VPL_CUDA(cudaMemsetAsync(w.counts, 0, 2 * sizeof(unsigned long long), s));
    k_count_labels<<<min(nblk(n, 256), 148 * 4), 256, 0, s>>>(d_labels, n, w.counts);
    VPL_LAUNCHED("k_count_labels");
    unsigned long long h_cnt[2];
    VPL_CUDA(cudaMemcpyAsync(h_cnt, w.counts, sizeof(h_cnt), cudaMemcpyDeviceToHost, s));
    VPL_CUDA(cudaStreamSynchronize(s));
    info->n_near = (int64_t)h_cnt[0];
    info->n_far_tris = n - info->n_near;

    // ---- near part
    int64_t m = 0;
    uint64_t F = 0;
    if (p->K_near > 0 && p->n_walks_fixed == 0 && info->n_near > 0) {
        k_lit<<<nblk(n, 128), 128, 0, s>>>(sv, bv, d_labels, n, w.lit);
        VPL_LAUNCHED("k_lit");
        size_t cb = w.cub_bytes;
        k_iota<<<nblk(n, 256), 256, 0, s>>>(w.iota, n);
        VPL_LAUNCHED("k_iota");
        VPL_CUDA(cub::DeviceSelect::Flagged(w.cub, cb, w.iota, w.lit, w.lit_idx, w.d_m, (int)n, s));
        int32_t hm = 0;
        VPL_CUDA(cudaMemcpyAsync(&hm, w.d_m, sizeof(hm), cudaMemcpyDeviceToHost, s));
        VPL_CUDA(cudaStreamSynchronize(s));
        m = hm;
        if (m > 0) {
            k_init_bbox<<<1, 32, 0, s>>>(w.enc);
            VPL_LAUNCHED("k_init_bbox");
            k_lit_bbox<<<min(nblk(m, 256), 148 * 4), 256, 0, s>>>(sv, w.lit_idx, w.d_m, w.enc);
            VPL_LAUNCHED("k_lit_bbox");
            k_morton30<<<nblk(m, 256), 256, 0, s>>>(sv, w.lit_idx, m, w.enc, w.codes);
            VPL_LAUNCHED("k_morton30");
            cb = w.cub_bytes;
            VPL_CUDA(cub::DeviceRadixSort::SortPairs(w.cub, cb, w.codes, w.codes2, w.lit_idx, w.order, (int)m, 0, 30, s));
            k_gather_aq<<<nblk(m, 256), 256, 0, s>>>(sv, w.order, m, w.aq_sorted);
            VPL_LAUNCHED("k_gather_aq");
            cb = w.cub_bytes;
            VPL_CUDA(cub::DeviceScan::InclusiveSum(w.cub, cb, w.aq_sorted, w.P, (int)m, s));
            VPL_CUDA(cudaMemcpyAsync(&F, w.P + (m - 1), sizeof(F), cudaMemcpyDeviceToHost, s));
            VPL_CUDA(cudaStreamSynchronize(s));
        }
    }
    info->n_lit = m;
    int64_t K = p->K_near, Mf = p->M - p->K_near;
    if (p->n_walks_fixed > 0) K = 0;
    else if (m == 0) { K = 0; Mf = p->M; info->flags |= VPL_FLAG_EMPTY_NEAR; }
    else if (info->n_far_tris == 0) { K = p->M; Mf = 0; info->flags |= VPL_FLAG_EMPTY_FAR; }
    if (K > max_out || (p->n_walks_fixed == 0 && K + Mf > max_out)) {
        set_error("vpl_generate_vpls: max_out %lld < %lld", (long long)max_out, (long long)(K + Mf));
        return VPL_ESMALL;
    }
    info->K = K;
    if (K > 0) {
        float D = (float)((double)F / (double)K / 1099511627776.0);
        k_strata<<<nblk(K, 128), 128, 0, s>>>(sv, bv, w.order, w.P, m, K, D, p->seed, d_vpls);
        VPL_LAUNCHED("k_strata");
    }

    // ---- far part (P:35, P:46 step 3)
    int64_t n_out = K, walks = 0;
    std::vector<int32_t> hc;
    if (md > 0 && (p->n_walks_fixed > 0 || Mf > 0)) {
        const bool fixed = p->n_walks_fixed > 0;
        const int64_t Wmax = fixed ? p->n_walks_fixed : 1024 * Mf;
        int64_t have = 0;
        bool done = false;
        for (int64_t w0 = 0; w0 < Wmax && !done;) {
            int64_t want = fixed ? Wmax - w0 : std::max<int64_t>(4096, 2 * (Mf - have));
            int64_t nb = std::min<int64_t>(std::min<int64_t>(want, Wmax - w0), kWalkBatchMax);
            k_walks<<<nblk(nb, 64), 64, 0, s>>>(sv, bv, d_labels, w0, nb, md, (int)p->rr, p->seed, w.dep, w.cnt);
            VPL_LAUNCHED("k_walks");
            size_t cb = w.cub_bytes;
            VPL_CUDA(cub::DeviceScan::ExclusiveSum(w.cub, cb, w.cnt, w.off, (int)nb, s));
            hc.resize(nb);
            VPL_CUDA(cudaMemcpyAsync(hc.data(), w.cnt, sizeof(int32_t) * nb, cudaMemcpyDeviceToHost, s));
            VPL_CUDA(cudaStreamSynchronize(s));
            int64_t cut = nb - 1, take_last = hc[nb - 1], got = 0;
            if (fixed) {
                for (int64_t i = 0; i < nb; ++i) got += hc[i];
                walks = w0 + nb;
            } else {
                int64_t need_more = Mf - have;
                int64_t acc = 0;
                for (int64_t i = 0; i < nb; ++i) {
                    walks = w0 + i + 1;
                    if (acc + hc[i] >= need_more) {
                        cut = i;
                        take_last = need_more - acc;
                        got = need_more;
                        done = true;
                        break;
                    }
                    acc += hc[i];
                }
                if (!done) got = acc;
            }
            if (n_out + got > max_out) { set_error("vpl_generate_vpls: max_out too small for fixed walks"); return VPL_ESMALL; }
            if (got > 0) {
                k_walk_compact<<<nblk(nb, 128), 128, 0, s>>>(w.dep, w.cnt, w.off, nb, md, cut, (int)take_last,
                                                             d_vpls + n_out);
                VPL_LAUNCHED("k_walk_compact");
            }
            n_out += got;
            have += got;
            w0 += nb;
        }
        if (!fixed && !done) info->flags |= VPL_FLAG_WALK_BUDGET_UNMET;
        if (walks > 0 && n_out > K) {
            k_div_flux<<<nblk(n_out - K, 256), 256, 0, s>>>(d_vpls + K, n_out - K, (float)walks);
            VPL_LAUNCHED("k_div_flux");
        }
    }
    info->M_far = n_out - K;
    info->n_walks = walks;
    info->n_out = n_out;
    VPL_CUDA(cudaStreamSynchronize(s));
    return VPL_OK;
}

}  // extern "C"
