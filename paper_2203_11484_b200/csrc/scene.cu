// scene.cu — a1 scene_upload (O1) and a3 classify_near_far (O2).
#include "common.cuh"

#ifndef VPL_BOX_PAD
#define VPL_BOX_PAD 0x1p-16f   // BVH box padding relative to max |coordinate|
#endif
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
    h->box_pad = m * VPL_BOX_PAD;  // conservative BVH box padding
    if (d_bad) *d_bad = h->bad == ~0ull ? -1 : (int64_t)h->bad;
}

// (knob definitions must precede use; see the top of this file)
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

}  // extern "C"
