/*
 * vplgi.h — C ABI of the B200-native (sm_100a) hybrid-VPL many-light gather
 * of arXiv 2203.11484 ("A hybrid VPL sampling", PAPER.md = P:n line refs).
 *
 * Library: paper_2203_11484_b200/libvplgi.so.  Every function returns an
 * int32_t status (VPL_OK = 0, negative on error; see vpl_status_string and
 * vpl_last_error for the message).  No torch types cross this boundary.
 *
 * Ownership: every d_* pointer is caller-owned device memory on the current
 * CUDA device (the Python binding allocates them as torch tensors); h_*
 * pointers are caller-owned host memory read or written during the call
 * only.  The library never allocates device memory and keeps no pointer
 * after a call returns.  Work is enqueued on `stream` (a cudaStream_t passed
 * as void*; NULL = legacy default stream); outputs are valid once the stream
 * is synchronised.  Only vpl_generate_vpls synchronises the stream itself
 * (it loops on the host over batches of random walks, P:46 step 3).
 * Calls are reentrant on disjoint buffers; the only global state is a
 * thread-local last-error string.
 *
 * Errors: VPL_EINVAL (null pointer, bad size or range), VPL_ESMALL (a buffer
 * smaller than its size query), VPL_ECUDA (launch/runtime error), VPL_EARCH
 * (device is not sm_100).  Data-dependent outcomes (degenerate triangle,
 * empty near set, unmet walk budget) are reported through output values,
 * never through the status code.
 *
 * Arithmetic: the bit-exact steps follow DESIGN.md §3 (O0-O12) — IEEE fp32
 * without FMA contraction; the gather (O13) accumulates in fp32.
 */
#ifndef VPLGI_H
#define VPLGI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define VPL_API __attribute__((visibility("default")))
#else
#define VPL_API
#endif

#define VPL_ABI_VERSION 4   /* 4: vpl_counters.plane_culled; 3: vpl_counters.cand_*, filter_steps; 2: vpl_gather_bytes(M, W, H), vpl_counters.cache_tests, f1-f4 entry points */
#define VPL_MAX_LIGHTS 64

enum {
    VPL_OK = 0,
    VPL_EINVAL = -1,
    VPL_ESMALL = -2,
    VPL_ECUDA = -3,
    VPL_EARCH = -4,
};

/* flags in vpl_gen_info.flags */
enum {
    VPL_FLAG_EMPTY_NEAR = 1,        /* no lit near patch: K := 0, M_far := M */
    VPL_FLAG_EMPTY_FAR = 2,         /* no far patch: K := M */
    VPL_FLAG_WALK_BUDGET_UNMET = 4, /* 1024*M_far walks did not yield M_far far deposits */
};

/* Area light (BJ:7-11 use 0.5 x 0.5 m quads; R2): the parallelogram
 * corner + a*e_u + b*e_v (a, b in [0,1]) emitting radiance `radiance` on the
 * side of `normal`; `area` = |e_u x e_v|.  16 floats, the row layout of
 * scenegen's light array.
 * Point light (Eq. 2's literal form P:51-56; reading R27):
 * area == 0 marks an isotropic point light at `corner` (e_u = e_v = 0,
 * `normal` ignored) whose `radiance` field holds its power Phi (W per
 * channel): near VPLs get Phi cos(omega)/(4 pi r^2) V per unit represented
 * area (times rho/pi), walks start with power Phi n_L in a uniform
 * direction on the sphere, and the direct term needs no light samples. */
typedef struct {
    float corner[3], e_u[3], e_v[3], normal[3], area, radiance[3];
} vpl_light;

/* Pinhole camera: orthonormal fwd/up/right, tan_y = tan(vfov/2),
 * tan_x = tan_y * W / H; pixel (px, py), py = 0 the top row. */
typedef struct {
    float pos[3], fwd[3], up[3], right[3], tan_x, tan_y;
    int32_t width, height;
} vpl_camera;

/* VPL record, 48 bytes (3 x float4).  tri = original triangle index;
 * tag_depth = tag | depth << 8 (tag 0 = near/patch VPL, 1 = far/walk VPL);
 * walk = walk index (far) or stratum index k (near).  flux Phi is the value
 * of Eq. 1's L_i: radiance at x is rho_x/pi * sum Phi * cx ci / ... */
typedef struct {
    float pos[3];
    int32_t tri;
    float nrm[3];
    int32_t tag_depth;
    float flux[3];
    int32_t walk;
} vpl_record;

/* G-buffer point, 48 bytes (3 x float4): hit position, geometric normal,
 * albedo, distance t, triangle (-1 = miss) and front (1 = front-face hit). */
typedef struct {
    float pos[3];
    int32_t tri;
    float nrm[3];
    int32_t front;
    float alb[3];
    float t;
} vpl_gpoint;

/* generate_vpls knobs (BJ:7-11; DESIGN.md §3 O6-O11) */
typedef struct {
    int64_t M;             /* total VPL budget (Eq. 1's M) */
    int64_t K_near;        /* requested patch-stratified VPLs (K of P:65) */
    int64_t max_depth;     /* D_max of the sparse-IR walk */
    int64_t rr;            /* 1 = Russian roulette (R10) */
    int64_t n_walks_fixed; /* 0 = budget mode (R11); > 0 = run exactly this many walks, keep all deposits */
    uint64_t seed;         /* Philox key */
} vpl_gen_params;

typedef struct {
    int64_t n_near, n_lit, K, M_far, n_walks, flags, n_far_tris, n_out;
} vpl_gen_info;

/* gather counters (nullable output of vpl_gather_indirect; DESIGN.md §5
 * turns them into algorithmic op counts for the roofline) */
typedef struct {
    unsigned long long pairs;        /* front-hit pixels x VPLs considered (Eq. 1 terms) */
    unsigned long long traced;       /* pairs that passed the cosine test and got a shadow ray */
    unsigned long long visible;      /* traced pairs found unoccluded */
    unsigned long long box_tests;    /* per-ray slab tests (ray x child box, 4-wide nodes) */
    unsigned long long tri_tests;    /* exact Moller-Trumbore tests (ray x triangle) */
    unsigned long long warp_rays;    /* packets that needed a traversal (>= 1 unresolved lane) */
    unsigned long long warp_steps;   /* warp-level traversal iterations (node or leaf visits) */
    unsigned long long cone_tests;   /* beam x child box tests of real (non-empty) children of 16-wide nodes */
    unsigned long long cone_packets; /* packets traversed with the cone test */
    unsigned long long ray_packets;  /* packets traversed with per-ray tests (loose cones) */
    unsigned long long cache_hits;   /* traced lanes resolved by the occluder cache */
    unsigned long long cache_tests;  /* exact MT tests spent in the occluder cache (part of tri_tests) */
    unsigned long long cand_lists;   /* VPL clusters whose candidate-triangle list was built */
    unsigned long long cand_entries; /* total entries of those lists */
    unsigned long long cand_fails;   /* clusters whose list could not be used (loose beam or overflow) */
    unsigned long long filter_steps; /* per-VPL candidate-filter iterations (32 candidates each) */
    unsigned long long cand_steps;   /* traversal steps spent building the lists (part of warp_steps) */
    unsigned long long filter_mt;    /* warp-level MT tests issued by the list filter */
    unsigned long long filter_mt_hits; /* ... of which found an occluder for some lane */
    unsigned long long plane_culled; /* box-hit candidate triangles dropped by the plane-side cull before MT */
} vpl_counters;

/* -------------------------------------------------------------------- */
VPL_API int32_t vpl_abi_version(void);
VPL_API const char* vpl_status_string(int32_t status);
VPL_API const char* vpl_last_error(void);
/* number of kernels this library has launched in the process (all threads) */
VPL_API uint64_t vpl_launch_count(void);
/* multiProcessorCount and the sm major.minor of the current device */
VPL_API int32_t vpl_device_info(int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor);

/* -------------------------------------------------------------------- */
/* a1  scene_upload (O1)
 * Copies the N triangles (d_verts float[N*9] = v0 v1 v2 xyz, d_albedo
 * float[N*3] RGB in [0,1]), the lights and the camera into the caller's
 * scene blob (size from vpl_scene_bytes) and derives per-triangle normal,
 * area, centroid, 40-bit fixed-point area, the scene bbox and the constants
 * diag, eps = 1e-4*diag (R13) and b^2 = (0.01*diag)^2 (R12).
 * d_bad (nullable, device int64): receives the lowest degenerate triangle
 * index or -1. */
VPL_API int32_t vpl_scene_bytes(int64_t n_tris, int32_t n_lights, size_t* bytes);
VPL_API int32_t vpl_scene_upload(const float* d_verts, const float* d_albedo, int64_t n_tris,
                         const vpl_light* h_lights, int32_t n_lights, const vpl_camera* h_cam,
                         void* d_scene, size_t scene_bytes, int64_t* d_bad, void* stream);
/* test hook: per-triangle derived data (O1) into caller device arrays
 * d_nrm float[N*3], d_cen float[N*3], d_area float[N], d_aq uint64[N] */
VPL_API int32_t vpl_scene_tri_data(const void* d_scene, float* d_nrm, float* d_cen, float* d_area, uint64_t* d_aq,
                           void* stream);
/* copies the scene constants back (synchronises the stream) */
VPL_API int32_t vpl_scene_consts(const void* d_scene, double* diag, float* eps, float* b2, void* stream);

/* -------------------------------------------------------------------- */
/* a2  build_bvh (the paper has no acceleration structure)
 * Deterministic PLOC build (search radius VPL_PLOC_RADIUS, 128 by default, bvh.cu) over the 63-bit Morton order
 * of the centroids, SAH leaf collapse, then a 16-wide (beam traversal) and a
 * 4-wide (per-ray traversal) collapse of the same tree; boxes padded by
 * 2^-16 * max|coord| so every box test is conservative w.r.t. the exact
 * Moller-Trumbore tests of O9; per triangle also its plane (unit normal and
 * offset, rounded once from float64) for the gather's plane-side cull.
 * Same scene in, same bytes out.
 * d_bvh: vpl_bvh_bytes(...).bvh bytes; d_work: .work bytes (scratch). */
VPL_API int32_t vpl_bvh_bytes(int64_t n_tris, size_t* bvh_bytes, size_t* work_bytes);
VPL_API int32_t vpl_build_bvh(const void* d_scene, void* d_bvh, size_t bvh_bytes, void* d_work, size_t work_bytes,
                      void* stream);

/* -------------------------------------------------------------------- */
/* a3  classify_near_far (O2)
 * d_labels uint8[N]: 1 = near (centroid strictly inside the view frustum and
 * closer than T metres), 0 = far.  d_n_near (nullable, device int64). */
VPL_API int32_t vpl_classify_near_far(const void* d_scene, double T, uint8_t* d_labels, int64_t* d_n_near,
                              void* stream);

/* -------------------------------------------------------------------- */
/* a4-a6  generate_vpls (P:44-65 near part, P:35/P:46 far part; O3-O11)
 * d_labels: near/far labels (a3's output, or any caller labels — all-zero
 * with n_walks_fixed > 0 yields plain instant radiosity).
 * d_vpls: vpl_record[max_out]; on return h_info->n_out records are valid
 * (near in stratum order, then far in (walk, depth) order).
 * d_work: vpl_generate_bytes(...) bytes.  Synchronises `stream`. */
VPL_API int32_t vpl_generate_bytes(const vpl_gen_params* h_p, int64_t n_tris, int64_t max_out, size_t* work_bytes);
VPL_API int32_t vpl_generate_vpls(const void* d_scene, const void* d_bvh, const uint8_t* d_labels,
                          const vpl_gen_params* h_p, vpl_record* d_vpls, int64_t max_out,
                          vpl_gen_info* h_info, void* d_work, size_t work_bytes, void* stream);

/* -------------------------------------------------------------------- */
/* Pixel tiles (multi-GPU sharding unit): the image is cut into
 * tile_w x tile_h tiles numbered row-major (tiles_x = ceil(W/tile_w));
 * d_tiles int32[n_tiles] lists the tiles a call processes.  tile_w must be a
 * multiple of 8 and tile_h of 4 (a warp covers an 8x4 pixel block). */

/* a7  render_gbuffer (O12): centre-sample primary rays,
 * closest hit; writes d_gbuf[py*W + px] for the listed tiles only. */
VPL_API int32_t vpl_render_gbuffer(const void* d_scene, const void* d_bvh, const int32_t* d_tiles, int32_t n_tiles,
                           int32_t tile_w, int32_t tile_h, vpl_gpoint* d_gbuf, void* stream);

/* a8  gather_indirect (Eq. 1; O13): indirect-only linear radiance
 * d_rgb float[H*W*3] for the listed tiles (others untouched).  Miss or
 * back-face pixels get 0.  d_ctr (nullable) accumulates counters.
 * n_tiles = 0 is a no-op (d_tiles may then be null), as for every per-tile call.
 * d_work: vpl_gather_bytes(n_vpls, W, H) bytes (tile queue, a Morton-ordered
 * copy of the VPLs — Eq. 1 is a sum over the set, the gather visits it in
 * spatial order; the caller's array is not modified — VPL cluster bounds and,
 * when M > 256, per-chunk partial sums: the work items are (8x8 pixel block,
 * VPL chunk) pairs, chunk = max(256, ceil(M/128) rounded up to 256) VPLs —
 * groups of 128 consecutive sorted VPLs dealt round-robin to the chunks —
 * folded in chunk order by the warp that completes a block's last chunk, so
 * the image depends on M only, never on the tile split; the partial sums live
 * in a ring of 4096 block slots reused in block order).  Visibility of each
 * traced pair is the exact O9 any-hit: the 16-wide BVH is culled with
 * conservative beams (padded boxes); per run of 16 consecutive sorted VPLs a
 * list of candidate triangles is gathered once with the run's beam; a list
 * entry whose plane no pending segment can cross inside (eps, L - eps) is
 * skipped before its MT tests. */
VPL_API int32_t vpl_gather_bytes(int32_t n_vpls, int32_t width, int32_t height, size_t* work_bytes);
VPL_API int32_t vpl_gather_indirect(const void* d_scene, const void* d_bvh, const vpl_gpoint* d_gbuf,
                            const vpl_record* d_vpls, int32_t n_vpls, const int32_t* d_tiles, int32_t n_tiles,
                            int32_t tile_w, int32_t tile_h, float* d_rgb, vpl_counters* d_ctr, void* d_work,
                            size_t work_bytes, void* stream);

/* test hook: the production gather (same launch as vpl_gather_indirect,
 * counter build) that also records its own traced / visible bit of every
 * (listed pixel, VPL) pair.  d_pixel_slot: int32[W*H] (nullable: no bits),
 * the dump row of each pixel or -1; d_traced_bits / d_vis_bits:
 * uint32[rows * ceil(n_vpls/32)], zeroed by the caller, bit i%32 of word i/32
 * = VPL i of d_vpls (the caller's order).  d_ctr nullable.  flags:
 * VPL_GATHER_NO_CULL runs without the VPL-cluster cull, the candidate
 * lists and the plane-side cull (plain per-VPL beam traversal, an exact MT
 * for every triangle box the beam reaches), so the counters of the two runs
 * can be compared. */
enum { VPL_GATHER_NO_CULL = 1 };
VPL_API int32_t vpl_gather_dump(const void* d_scene, const void* d_bvh, const vpl_gpoint* d_gbuf,
                                const vpl_record* d_vpls, int32_t n_vpls, const int32_t* d_tiles, int32_t n_tiles,
                                int32_t tile_w, int32_t tile_h, float* d_rgb, vpl_counters* d_ctr, void* d_work,
                                size_t work_bytes, const int32_t* d_pixel_slot, uint32_t* d_traced_bits,
                                uint32_t* d_vis_bits, int32_t flags, void* stream);

/* NEXT f2  render_direct: the direct term L_e of Eq. 1 ("L_e(y)
 * represents direct illumination"; SPEC shade_direct S:327-335; O14,
 * reading R21) for the listed tiles: per pixel, `samples` uniform points on
 * every area light drawn from Philox stream 4 (item = pixel index, draws
 * 2(l*samples+s) and +1), exact fp32 Eq. 2-form irradiance with exact any-hit
 * visibility, out = rho/pi * E/samples.  d_rgb float[H*W*3]: written
 * (accumulate = 0) or added to (accumulate = 1, e.g. onto the gather's
 * indirect image); miss / back-face pixels get 0 (or are left unchanged).
 * Errors: VPL_EINVAL for null pointers or samples <= 0. */
VPL_API int32_t vpl_render_direct(const void* d_scene, const void* d_bvh, const vpl_gpoint* d_gbuf,
                          const int32_t* d_tiles, int32_t n_tiles, int32_t tile_w, int32_t tile_h,
                          int32_t samples, uint64_t seed, int32_t accumulate, float* d_rgb, void* stream);

/* NEXT f1  image_error: the RMSE harness of the paper's equal-sample
 * comparisons ("RMS" against a > 200k-VPL reference).
 * d_out double[4] = { sum (img - ref)^2, sum ref^2, sum |img - ref|, sum |ref| }
 * over n floats (fp64, deterministic order).  d_work: >= 4 * 592 doubles
 * (18,944 bytes).  d_img / d_ref may be null when n = 0 (all sums 0).
 * Errors: VPL_EINVAL null / n < 0, VPL_ESMALL short work. */
VPL_API int32_t vpl_image_error(const float* d_img, const float* d_ref, int64_t n, double* d_out, void* d_work,
                        size_t work_bytes, void* stream);

/* NEXT f3  generate_rejection: the rejection-sampling comparator (P:29-32
 * [r3], "reject those VPLs that contribute less than the average value to
 * the resulting image"; O15, reading R23).
 * d_pilot: n_pilot candidate records (plain IR: vpl_generate_vpls with every
 * patch FAR).  64 probe pixels (8 x 8 blocks, offsets from Philox stream 5,
 * item = block) get their G-buffer points (O12); candidate i scores
 * s_i = sum over probes, in order, of its Eq. 1 summand as luminance (exact
 * fp32, exact visibility); mean = fp64 sum / n_pilot;
 * p_i = max(0.05, min(1, s_i / mean)); i is accepted iff
 * U(Philox stream 6, item i, draw 0) < p_i, scanning in index order until
 * `budget` are accepted (scanned = index of the last + 1, else n_pilot);
 * kept flux *= (float)((n_pilot / scanned) / p_i).  Outputs: d_out (up to
 * min(budget, n_pilot) records, the accepted ones in index order),
 * d_accepted int64 (their number); nullable: d_scores float[n_pilot],
 * d_mean double, d_scanned int64, d_probe_pixels int32[64].  d_work:
 * vpl_rejection_bytes(n_pilot) bytes.  Errors: VPL_EINVAL (null, n_pilot <= 0
 * or > 2^31 - 1, budget <= 0), VPL_ESMALL (short work). */
VPL_API int32_t vpl_rejection_bytes(int64_t n_pilot, size_t* work_bytes);
VPL_API int32_t vpl_generate_rejection(const void* d_scene, const void* d_bvh, const vpl_record* d_pilot,
                               int64_t n_pilot, int64_t budget, uint64_t seed, vpl_record* d_out,
                               float* d_scores, double* d_mean, int64_t* d_accepted, int64_t* d_scanned,
                               int32_t* d_probe_pixels, void* d_work, size_t work_bytes, void* stream);

/* NEXT f4  generate_metropolis: the Metropolis comparator (P:31-32 [r2],
 * "distributes VPLs according to Metropolis-Hastings sampling"; SPEC
 * S:261-269; O16, reading R24 — the paper gives no mutation
 * details).  Pool = the pilot candidates along their Morton curve (O4
 * quantisation over the pilot position box, ties by index); target
 * f_j = max(s_pool[j], 0.05 * mean) with the probe scores s of
 * vpl_generate_rejection (probes from `seed`).  `chains` chains (Philox
 * stream 7, item = chain) start at (x0 * n_pilot) >> 32, propose
 * j' = j + delta (mod n_pilot), delta uniform in [-radius, radius] \ {0},
 * accept iff U < f_j' / f_j (fp64), and after `burn` steps emit every state:
 * d_out[c * per_chain + t] = pilot[pool[j]] with flux *=
 * (float)((n_pilot / (chains * per_chain)) * (mean_f / f_j)).
 * d_accepted uint64: accepted proposals; d_scores float[n_pilot] and d_pool
 * int32[n_pilot] nullable.  d_work: vpl_rejection_bytes(n_pilot) bytes.
 * Errors: VPL_EINVAL (null, n_pilot < 2, chains / per_chain / radius < 1,
 * burn < 0), VPL_ESMALL (short work). */
VPL_API int32_t vpl_generate_metropolis(const void* d_scene, const void* d_bvh, const vpl_record* d_pilot,
                                int64_t n_pilot, int64_t chains, int64_t per_chain, int64_t burn, int64_t radius,
                                uint64_t seed, vpl_record* d_out, float* d_scores, int32_t* d_pool,
                                uint64_t* d_accepted, void* d_work, size_t work_bytes, void* stream);

/* -------------------------------------------------------------------- */
/* test hooks: same traversal code as the gather / the walks */
/* bits per listed pixel: ceil(n_vpls/32) words each of traced and visible */
VPL_API int32_t vpl_visibility_dump(const void* d_scene, const void* d_bvh, const vpl_gpoint* d_gbuf,
                            const vpl_record* d_vpls, int32_t n_vpls, const int32_t* d_pixels, int32_t n_pixels,
                            uint32_t* d_traced_bits, uint32_t* d_vis_bits, void* stream);
/* closest hit of n rays (o, dir float[n*3]) in (tmin, tmax): d_tri int32 (-1 miss), d_t float */
VPL_API int32_t vpl_closest_hit_batch(const void* d_scene, const void* d_bvh, const float* d_o, const float* d_dir,
                              int64_t n, float tmin, float tmax, int32_t* d_tri, float* d_t, void* stream);
/* segment occlusion of n point pairs (O9 unoccluded: eps-shrunk segment,
 * division-free any hit of DESIGN.md R25): d_occ uint8 */
VPL_API int32_t vpl_occluded_batch(const void* d_scene, const void* d_bvh, const float* d_a, const float* d_b,
                           int64_t n, uint8_t* d_occ, void* stream);
/* Philox4x32-10 of n (ctr, key) pairs: d_in uint32[n*6], d_out uint32[n*4] */
VPL_API int32_t vpl_philox_batch(const uint32_t* d_in, int64_t n, uint32_t* d_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* VPLGI_H */
