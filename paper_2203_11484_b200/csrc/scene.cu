// scene.cu — a1 scene_upload (O1), a3 classify_near_far (O2), a2 build_bvh (LBVH).
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"

namespace vplgi {

__device__ __forceinline__ uint32_t fenc(float f) {
    uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float fdec(uint32_t u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u);
}

__global__ void k_scene_init(SceneHdr* h, int64_t n, int32_t nL, const vpl_light* lights_dev_unused) {
    (void)lights_dev_unused;
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        for (int a = 0; a < 3; ++a) { h->bbox_enc[a] = 0xFFFFFFFFu; h->bbox_enc[3 + a] = 0u; }
        h->bad = ~0ull;
    }
}

// O1 — per-triangle prep and the degenerate check
__global__ void k_tri_prep(const float* __restrict__ vin, const float* __restrict__ ain, int64_t n, SceneHdr* h,
                           float* __restrict__ verts, float4* __restrict__ nrm, float4* __restrict__ alb,
                           float4* __restrict__ cen, uint64_t* __restrict__ aq) {
    uint32_t lo[3] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu}, hi[3] = {0u, 0u, 0u};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float* v = vin + 9 * i;
        float vv[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) { vv[k] = v[k]; verts[9 * i + k] = vv[k]; }
        f3 v0 = mk3(vv[0], vv[1], vv[2]), v1 = mk3(vv[3], vv[4], vv[5]), v2 = mk3(vv[6], vv[7], vv[8]);
        f3 e1 = v1 - v0, e2 = v2 - v0;
        f3 c = cross(e1, e2);
        float len = sqrtf(dot(c, c));
        float area = 0.5f * len;
        nrm[i] = make_float4(c.x / len, c.y / len, c.z / len, area);
        f3 ce = (v0 + v1) + v2;
        cen[i] = make_float4(ce.x / 3.0f, ce.y / 3.0f, ce.z / 3.0f, 0.0f);
        alb[i] = make_float4(ain[3 * i], ain[3 * i + 1], ain[3 * i + 2], 0.0f);
        uint64_t q = __double2ull_rn((double)area * 1099511627776.0);  // exact scale, round half even
        aq[i] = q;
        if (!(area > 0.0f) || q == 0ull) atomicMin(&h->bad, (unsigned long long)i);
#pragma unroll
        for (int k = 0; k < 9; ++k) {
            uint32_t e = fenc(vv[k]);
            lo[k % 3] = min(lo[k % 3], e);
            hi[k % 3] = max(hi[k % 3], e);
        }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        for (int o = 16; o > 0; o >>= 1) {
            lo[a] = min(lo[a], __shfl_xor_sync(0xFFFFFFFFu, lo[a], o));
            hi[a] = max(hi[a], __shfl_xor_sync(0xFFFFFFFFu, hi[a], o));
        }
    }
    if ((threadIdx.x & 31) == 0) {
        for (int a = 0; a < 3; ++a) {
            atomicMin(&h->bbox_enc[a], lo[a]);
            atomicMax(&h->bbox_enc[3 + a], hi[a]);
        }
    }
}

// scene constants in double, rounded once (O0; R12, R13)
__global__ void k_scene_consts(SceneHdr* h, int64_t* d_bad) {
    if (threadIdx.x || blockIdx.x) return;
    float m = 0.0f;
    for (int a = 0; a < 3; ++a) {
        h->bbox_lo[a] = fdec(h->bbox_enc[a]);
        h->bbox_hi[a] = fdec(h->bbox_enc[3 + a]);
        m = fmaxf(m, fmaxf(fabsf(h->bbox_lo[a]), fabsf(h->bbox_hi[a])));
    }
    double dx = (double)h->bbox_hi[0] - (double)h->bbox_lo[0];
    double dy = (double)h->bbox_hi[1] - (double)h->bbox_lo[1];
    double dz = (double)h->bbox_hi[2] - (double)h->bbox_lo[2];
    double diag = sqrt(dx * dx + dy * dy + dz * dz);
    h->diag = diag;
    h->eps = (float)(1e-4 * diag);
    h->b2 = (float)((0.01 * diag) * (0.01 * diag));
    h->box_pad = m * 0x1p-16f;  // conservative BVH box padding
    if (d_bad) *d_bad = h->bad == ~0ull ? -1 : (int64_t)h->bad;
}

// O2 — near iff the centroid is strictly inside the frustum and closer than T
__global__ void k_classify(const SceneHdr* __restrict__ h, const float4* __restrict__ cen, int64_t n, float T2,
                           uint8_t* __restrict__ labels, unsigned long long* __restrict__ n_near) {
    const float* c = h->cam;
    f3 pos = ld3(c), fwd = ld3(c + 3), up = ld3(c + 6), right = ld3(c + 9);
    float tx = c[12], ty = c[13];
    unsigned long long cnt = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        f3 d = xyz(cen[i]) - pos;
        float z = dot(d, fwd), x = dot(d, right), y = dot(d, up);
        bool near = (z > 0.0f) && (fabsf(x) < z * tx) && (fabsf(y) < z * ty) && (dot(d, d) < T2);
        labels[i] = (uint8_t)near;
        cnt += near;
    }
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, o);
    if (n_near && (threadIdx.x & 31) == 0 && cnt) atomicAdd(n_near, cnt);
}

__global__ void k_tri_data(SceneView sv, int64_t n, float* __restrict__ nrm, float* __restrict__ cen,
                           float* __restrict__ area, uint64_t* __restrict__ aq) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    float4 a = sv.nrm[i], c = sv.cen[i];
    nrm[3 * i] = a.x; nrm[3 * i + 1] = a.y; nrm[3 * i + 2] = a.z;
    area[i] = a.w;
    cen[3 * i] = c.x; cen[3 * i + 1] = c.y; cen[3 * i + 2] = c.z;
    aq[i] = sv.aq[i];
}

__global__ void k_i64_from_ull(const unsigned long long* a, int64_t* b) {
    if (threadIdx.x == 0 && blockIdx.x == 0) *b = (int64_t)*a;
}

// ------------------------------------------------------------------ LBVH (Karras 2012)
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
    f3 c = xyz(cen[i]);
    const float* lo = h->bbox_lo;
    const float* hi = h->bbox_hi;
    float q[3] = {c.x, c.y, c.z};
    uint32_t qi[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        float ext = hi[a] - lo[a];
        float s = ext > 0.0f ? 2097152.0f / ext : 0.0f;
        float f = fmaxf((q[a] - lo[a]) * s, 0.0f);
        qi[a] = min((uint32_t)f, 2097151u);
    }
    keys[i] = spread21(qi[0]) | (spread21(qi[1]) << 1) | (spread21(qi[2]) << 2);
    idx[i] = (uint32_t)i;
}

__device__ __forceinline__ int delta(const uint64_t* __restrict__ k, int64_t n, int64_t i, int64_t j) {
    if (j < 0 || j >= n) return -1;
    uint64_t a = k[i], b = k[j];
    if (a == b) return 64 + __clz((uint32_t)(i ^ j));
    return __clzll(a ^ b);
}

// child refs: >= 0 internal node, ~p leaf at sorted position p
__global__ void k_karras(const uint64_t* __restrict__ k, int64_t n, int2* __restrict__ child,
                         int32_t* __restrict__ parent_int, int32_t* __restrict__ parent_leaf) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n - 1) return;
    int d = (delta(k, n, i, i + 1) - delta(k, n, i, i - 1)) >= 0 ? 1 : -1;
    int dmin = delta(k, n, i, i - d);
    int64_t lmax = 2;
    while (delta(k, n, i, i + lmax * d) > dmin) lmax <<= 1;
    int64_t l = 0;
    for (int64_t t = lmax >> 1; t >= 1; t >>= 1)
        if (delta(k, n, i, i + (l + t) * d) > dmin) l += t;
    int64_t j = i + l * d;
    int dnode = delta(k, n, i, j);
    int64_t s = 0;
    int64_t t = l;
    do {
        t = (t + 1) >> 1;
        if (delta(k, n, i, i + (s + t) * d) > dnode) s += t;
    } while (t > 1);
    int64_t g = i + s * d + min(d, 0);
    int left = (min(i, j) == g) ? ~(int)g : (int)g;
    int right = (max(i, j) == g + 1) ? ~(int)(g + 1) : (int)(g + 1);
    child[i] = make_int2(left, right);
    if (left >= 0) parent_int[left] = (int)i; else parent_leaf[~left] = (int)i;
    if (right >= 0) parent_int[right] = (int)i; else parent_leaf[~right] = (int)i;
    if (i == 0) parent_int[0] = -1;
}

struct Box { float lo[3], hi[3]; };

__device__ __forceinline__ void store_box(float* dst, const Box& b) {
    for (int a = 0; a < 3; ++a) { __stcg(dst + a, b.lo[a]); __stcg(dst + 3 + a, b.hi[a]); }
}
__device__ __forceinline__ Box load_box(const float* src) {
    Box b;
    for (int a = 0; a < 3; ++a) { b.lo[a] = __ldcg(src + a); b.hi[a] = __ldcg(src + 3 + a); }
    return b;
}

// bottom-up refit: the second child to arrive computes the union
__global__ void k_refit(const SceneHdr* __restrict__ h, const float* __restrict__ verts, const uint32_t* __restrict__ sidx,
                        int64_t n, const int2* __restrict__ child, const int32_t* __restrict__ parent_int,
                        const int32_t* __restrict__ parent_leaf, int32_t* __restrict__ flags,
                        float* __restrict__ leafbox, float* __restrict__ intbox) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    float pad = h->box_pad;
    const float* v = verts + 9 * (int64_t)sidx[p];
    Box b;
    for (int a = 0; a < 3; ++a) {
        b.lo[a] = fminf(fminf(v[a], v[3 + a]), v[6 + a]) - pad;
        b.hi[a] = fmaxf(fmaxf(v[a], v[3 + a]), v[6 + a]) + pad;
    }
    store_box(leafbox + 6 * p, b);
    if (n == 1) return;
    __threadfence();
    int node = parent_leaf[p];
    while (node >= 0) {
        if (atomicAdd(&flags[node], 1) == 0) return;
        __threadfence();
        int2 c = child[node];
        Box a = c.x >= 0 ? load_box(intbox + 6 * c.x) : load_box(leafbox + 6 * (~c.x));
        Box bb = c.y >= 0 ? load_box(intbox + 6 * c.y) : load_box(leafbox + 6 * (~c.y));
        Box u;
        for (int k = 0; k < 3; ++k) { u.lo[k] = fminf(a.lo[k], bb.lo[k]); u.hi[k] = fmaxf(a.hi[k], bb.hi[k]); }
        store_box(intbox + 6 * node, u);
        __threadfence();
        node = parent_int[node];
    }
}

__global__ void k_pack_nodes(int64_t n, const int2* __restrict__ child, const float* __restrict__ leafbox,
                             const float* __restrict__ intbox, float4* __restrict__ nodes) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n - 1) return;
    int2 c = child[i];
    const float* a = c.x >= 0 ? intbox + 6 * c.x : leafbox + 6 * (~c.x);
    const float* b = c.y >= 0 ? intbox + 6 * c.y : leafbox + 6 * (~c.y);
    nodes[4 * i + 0] = make_float4(a[0], a[3], a[1], a[4]);
    nodes[4 * i + 1] = make_float4(b[0], b[3], b[1], b[4]);
    nodes[4 * i + 2] = make_float4(a[2], a[5], b[2], b[5]);
    nodes[4 * i + 3] = make_float4(__int_as_float(c.x), __int_as_float(c.y), 0.0f, 0.0f);
}

__global__ void k_pack_tris(const float* __restrict__ verts, const uint32_t* __restrict__ sidx, int64_t n,
                            float4* __restrict__ tris) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    uint32_t t = sidx[p];
    const float* v = verts + 9 * (int64_t)t;
    f3 v0 = ld3(v), e1 = ld3(v + 3) - v0, e2 = ld3(v + 6) - v0;
    tris[3 * p + 0] = make_float4(v0.x, v0.y, v0.z, __int_as_float((int)t));
    tris[3 * p + 1] = make_float4(e1.x, e1.y, e1.z, 0.0f);
    tris[3 * p + 2] = make_float4(e2.x, e2.y, e2.z, 0.0f);
}

struct BuildWork {
    uint64_t *keys, *keys2;
    uint32_t *idx, *idx2;
    int2* child;
    int32_t *parent_int, *parent_leaf, *flags;
    float *leafbox, *intbox;
    void* cub_tmp;
    size_t cub_bytes;
};

static size_t build_layout(int64_t n, char* base, BuildWork* w) {
    Bump b{base};
    w->keys = b.take<uint64_t>(n);
    w->keys2 = b.take<uint64_t>(n);
    w->idx = b.take<uint32_t>(n);
    w->idx2 = b.take<uint32_t>(n);
    w->child = b.take<int2>(n);
    w->parent_int = b.take<int32_t>(n);
    w->parent_leaf = b.take<int32_t>(n);
    w->flags = b.take<int32_t>(n);
    w->leafbox = b.take<float>(6 * n);
    w->intbox = b.take<float>(6 * n);
    size_t cub = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, cub, (uint64_t*)nullptr, (uint64_t*)nullptr, (uint32_t*)nullptr,
                                    (uint32_t*)nullptr, (int)n, 0, 64);
    w->cub_bytes = cub;
    w->cub_tmp = b.take<char>(cub);
    return b.off;
}

static inline int blocks_for(int64_t n, int t) { return (int)((n + t - 1) / t); }

}  // namespace vplgi

using namespace vplgi;

extern "C" {

int32_t vpl_scene_bytes(int64_t n_tris, int32_t n_lights, size_t* bytes) {
    if (!bytes || n_tris <= 0 || n_tris > (int64_t)1 << 30 || n_lights < 1 || n_lights > kMaxLights) {
        set_error("vpl_scene_bytes: bad arguments (n_tris=%lld, n_lights=%d)", (long long)n_tris, n_lights);
        return VPL_EINVAL;
    }
    *bytes = scene_layout(n_tris, nullptr);
    return VPL_OK;
}

int32_t vpl_scene_upload(const float* d_verts, const float* d_albedo, int64_t n_tris, const vpl_light* h_lights,
                         int32_t n_lights, const vpl_camera* h_cam, void* d_scene, size_t scene_bytes,
                         int64_t* d_bad, void* stream) {
    size_t need = 0;
    VPL_TRY(vpl_scene_bytes(n_tris, n_lights, &need));
    if (!d_verts || !d_albedo || !h_lights || !h_cam || !d_scene) { set_error("vpl_scene_upload: null pointer"); return VPL_EINVAL; }
    if (scene_bytes < need) { set_error("vpl_scene_upload: scene buffer %zu < %zu", scene_bytes, need); return VPL_ESMALL; }
    if (h_cam->width <= 0 || h_cam->height <= 0) { set_error("vpl_scene_upload: bad resolution"); return VPL_EINVAL; }
    VPL_TRY(check_arch());
    cudaStream_t s = (cudaStream_t)stream;
    SceneHdr hh;
    memset(&hh, 0, sizeof(hh));
    scene_layout(n_tris, &hh);
    hh.n = n_tris; hh.nL = n_lights; hh.W = h_cam->width; hh.H = h_cam->height;
    memcpy(hh.cam, h_cam->pos, 3 * sizeof(float));
    memcpy(hh.cam + 3, h_cam->fwd, 3 * sizeof(float));
    memcpy(hh.cam + 6, h_cam->up, 3 * sizeof(float));
    memcpy(hh.cam + 9, h_cam->right, 3 * sizeof(float));
    hh.cam[12] = h_cam->tan_x; hh.cam[13] = h_cam->tan_y;
    memcpy(hh.lights, h_lights, sizeof(vpl_light) * n_lights);
    static_assert(sizeof(vpl_light) == 16 * sizeof(float), "light row layout");
    SceneHdr* dh = (SceneHdr*)d_scene;
    // pageable H2D cudaMemcpyAsync stages the source before returning
    VPL_CUDA(cudaMemcpyAsync(dh, &hh, sizeof(SceneHdr), cudaMemcpyHostToDevice, s));
    k_scene_init<<<1, 32, 0, s>>>(dh, n_tris, n_lights, nullptr);
    VPL_LAUNCHED("k_scene_init");
    char* b = (char*)d_scene;
    int grid = min(blocks_for(n_tris, 256), 148 * 8);
    k_tri_prep<<<grid, 256, 0, s>>>(d_verts, d_albedo, n_tris, dh, (float*)(b + hh.off_verts),
                                    (float4*)(b + hh.off_nrm), (float4*)(b + hh.off_alb),
                                    (float4*)(b + hh.off_cen), (uint64_t*)(b + hh.off_aq));
    VPL_LAUNCHED("k_tri_prep");
    k_scene_consts<<<1, 32, 0, s>>>(dh, d_bad);
    VPL_LAUNCHED("k_scene_consts");
    return VPL_OK;
}

int32_t vpl_scene_consts(const void* d_scene, double* diag, float* eps, float* b2, void* stream) {
    if (!d_scene || !diag || !eps || !b2) return VPL_EINVAL;
    SceneHdr hh;
    cudaStream_t s = (cudaStream_t)stream;
    VPL_CUDA(cudaMemcpyAsync(&hh, d_scene, sizeof(hh), cudaMemcpyDeviceToHost, s));
    VPL_CUDA(cudaStreamSynchronize(s));
    *diag = hh.diag; *eps = hh.eps; *b2 = hh.b2;
    return VPL_OK;
}

int32_t vpl_scene_tri_data(const void* d_scene, float* d_nrm, float* d_cen, float* d_area, uint64_t* d_aq,
                           void* stream) {
    if (!d_scene || !d_nrm || !d_cen || !d_area || !d_aq) return VPL_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    SceneHdr hh;
    VPL_TRY(read_scene_hdr(d_scene, s, &hh));
    k_tri_data<<<blocks_for(hh.n, 256), 256, 0, s>>>(scene_view(d_scene, hh.n), hh.n, d_nrm, d_cen, d_area, d_aq);
    VPL_LAUNCHED("k_tri_data");
    return VPL_OK;
}

int32_t vpl_classify_near_far(const void* d_scene, double T, uint8_t* d_labels, int64_t* d_n_near, void* stream) {
    if (!d_scene || !d_labels || !(T > 0.0)) { set_error("vpl_classify_near_far: bad arguments"); return VPL_EINVAL; }
    cudaStream_t s = (cudaStream_t)stream;
    SceneHdr hh;
    VPL_TRY(read_scene_hdr(d_scene, s, &hh));
    SceneView sv = scene_view(d_scene, hh.n);
    float T2 = (float)(T * T);
    unsigned long long* cnt = nullptr;
    if (d_n_near) {
        // count into the caller's int64 slot through an unsigned alias
        cnt = (unsigned long long*)d_n_near;
        VPL_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), s));
    }
    int grid = min(blocks_for(hh.n, 256), 148 * 8);
    k_classify<<<grid, 256, 0, s>>>(sv.hdr, sv.cen, hh.n, T2, d_labels, cnt);
    VPL_LAUNCHED("k_classify");
    return VPL_OK;
}

int32_t vpl_bvh_bytes(int64_t n_tris, size_t* bvh_bytes, size_t* work_bytes) {
    if (!bvh_bytes || !work_bytes || n_tris <= 0) return VPL_EINVAL;
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
    int64_t n = hh.n;
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
    k_morton63<<<blocks_for(n, 256), 256, 0, s>>>(sv.hdr, sv.cen, n, w.keys, w.idx);
    VPL_LAUNCHED("k_morton63");
    size_t cb = w.cub_bytes;
    VPL_CUDA(cub::DeviceRadixSort::SortPairs(w.cub_tmp, cb, w.keys, w.keys2, w.idx, w.idx2, (int)n, 0, 64, s));
    if (n > 1) {
        VPL_CUDA(cudaMemsetAsync(w.flags, 0, sizeof(int32_t) * n, s));
        k_karras<<<blocks_for(n - 1, 256), 256, 0, s>>>(w.keys2, n, w.child, w.parent_int, w.parent_leaf);
        VPL_LAUNCHED("k_karras");
    }
    k_refit<<<blocks_for(n, 256), 256, 0, s>>>(sv.hdr, sv.verts, w.idx2, n, w.child, w.parent_int, w.parent_leaf,
                                               w.flags, w.leafbox, w.intbox);
    VPL_LAUNCHED("k_refit");
    if (n > 1) {
        k_pack_nodes<<<blocks_for(n - 1, 256), 256, 0, s>>>(n, w.child, w.leafbox, w.intbox, nodes);
        VPL_LAUNCHED("k_pack_nodes");
    }
    k_pack_tris<<<blocks_for(n, 256), 256, 0, s>>>(sv.verts, w.idx2, n, tris);
    VPL_LAUNCHED("k_pack_tris");
    return VPL_OK;
}

}  // extern "C"
