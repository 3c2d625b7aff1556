/*
 * oracle.c — plain, slow, obviously-correct CPU oracle for the hybrid-VPL
 * many-light gather of arXiv 2203.11484 (PAPER.md = P, line numbers P:n).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code with the CUDA path (paper_2203_11484_b200/csrc) and includes
 * none of its headers; both sides implement DESIGN.md §3 independently.
 *
 * Arithmetic contract (DESIGN.md §3 O0): IEEE binary32, round-to-nearest,
 * compiled with -ffp-contract=off (no FMA contraction), no fast-math, only
 * + - * / sqrt on floats.  Every loop follows the paper's definition; the
 * only library primitives are qsort (the Morton sort of P:62-63) and libm
 * nearbyint/sqrt in double for host constants.  Visibility and closest hit
 * are brute force over all triangles (no BVH).  Loops over independent
 * rays/pixels/walks are OpenMP-parallel; no per-pixel sum is reordered.
 *
 * Parity pins: see tests/test_oracle_*.py (closed forms, invariants, Philox
 * vs the CUDA toolkit's host Philox, brute-force tiny scenes).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_ABI 1
/* ORACLE_O0 = 1 builds the frozen O0 variant (liboracle_o0.so): SURVEY      */
/* §8(c) O0/O9 exactly as SPEC S:134-150 writes Moller-Trumbore — no fused  */
/* multiply-add anywhere, inv = 1/det for the any hit too, dir = d/dist     */
/* componentwise, and O13's cosine terms as plain dots.  The default build  */
/* keeps readings R25/R26.  Both are the same real-number    */
/* predicates; tests compare the CUDA path with both within BJ:5's budget.  */
#ifndef ORACLE_O0
#define ORACLE_O0 0
#endif
#define PI_D 3.14159265358979323846 /* pi, rounded once to double */

typedef struct { float x, y, z; } f3;

static inline f3 mk(float x, float y, float z) { f3 r = {x, y, z}; return r; }
static inline f3 add(f3 a, f3 b) { return mk(a.x + b.x, a.y + b.y, a.z + b.z); }
static inline f3 sub(f3 a, f3 b) { return mk(a.x - b.x, a.y - b.y, a.z - b.z); }
static inline f3 scl(float s, f3 a) { return mk(s * a.x, s * a.y, s * a.z); }
/* dot(a,b) = (a.x*b.x + a.y*b.y) + a.z*b.z  (O0) */
static inline float dot(f3 a, f3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
static inline f3 cross(f3 a, f3 b) {
    return mk(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
static inline f3 ld3(const float* p) { return mk(p[0], p[1], p[2]); }

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon et al., SC'11): 10 rounds, multipliers 0xD2511F53,  */
/* 0xCD9E8D57, Weyl key bumps 0x9E3779B9, 0xBB67AE85.                        */
/* ------------------------------------------------------------------------ */
void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; r++) {
        if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        uint32_t n1 = (uint32_t)p1;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        uint32_t n3 = (uint32_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Draw j of (stream, item): counter = (j>>2, item, stream, 0), key = seed
 * split into (lo, hi); lane j & 3 (DESIGN.md §3 O0).                        */
uint32_t oracle_draw(uint64_t seed, uint32_t stream, uint32_t item, uint32_t j) {
    uint32_t ctr[4] = {j >> 2, item, stream, 0u};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t out[4];
    oracle_philox4x32_10(ctr, key, out);
    return out[j & 3u];
}
/* u32 -> float in [0, 1 - 2^-24], exact */
static inline float u01(uint32_t x) { return (float)(x >> 8) * 0x1p-24f; }

enum { STREAM_NEAR = 0, STREAM_WALK = 1, STREAM_DIRECT = 4, STREAM_PROBE = 5, STREAM_REJECT = 6, STREAM_MH = 7 };

/* ------------------------------------------------------------------------ */
/* Scene                                                                     */
/* ------------------------------------------------------------------------ */
typedef struct {
    int64_t n;
    int nL, W, H;
    /* SoA copies for brute-force intersection */
    float *v0x, *v0y, *v0z, *e1x, *e1y, *e1z, *e2x, *e2y, *e2z;
    float *nrm;   /* [3n] unit normal (O1) */
    float *cen;   /* [3n] centroid (O1) */
    float *area;  /* [n] */
    uint64_t *aq; /* [n] 40-bit fixed-point area */
    float *alb;   /* [3n] */
    float *vert;  /* [9n] */
    float lights[16 * 64];
    float cam[14];
    int64_t bad;  /* -1 or first degenerate triangle */
    double diag;
    float eps, b2;
} OScene;

/* O1 — per-triangle prep. */
static void tri_prep(OScene* s, int64_t i) {
    const float* v = s->vert + 9 * i;
    f3 v0 = ld3(v), v1 = ld3(v + 3), v2 = ld3(v + 6);
    f3 e1 = sub(v1, v0), e2 = sub(v2, v0);
    s->v0x[i] = v0.x; s->v0y[i] = v0.y; s->v0z[i] = v0.z;
    s->e1x[i] = e1.x; s->e1y[i] = e1.y; s->e1z[i] = e1.z;
    s->e2x[i] = e2.x; s->e2y[i] = e2.y; s->e2z[i] = e2.z;
    f3 c = cross(e1, e2);
    float len = sqrtf(dot(c, c));
    float area = 0.5f * len;
    s->area[i] = area;
    s->nrm[3 * i + 0] = c.x / len;
    s->nrm[3 * i + 1] = c.y / len;
    s->nrm[3 * i + 2] = c.z / len;
    f3 ce = add(add(v0, v1), v2);
    s->cen[3 * i + 0] = ce.x / 3.0f;
    s->cen[3 * i + 1] = ce.y / 3.0f;
    s->cen[3 * i + 2] = ce.z / 3.0f;
    double a40 = (double)area * 1099511627776.0; /* exact: power-of-two scale */
    s->aq[i] = (uint64_t)nearbyint(a40);           /* round half to even     */
}

void oracle_scene_free(OScene* s) {
    if (!s) return;
    float* arrs[] = {s->v0x, s->v0y, s->v0z, s->e1x, s->e1y, s->e1z, s->e2x, s->e2y, s->e2z,
                     s->nrm, s->cen, s->area, s->alb, s->vert};
    for (unsigned k = 0; k < sizeof(arrs) / sizeof(arrs[0]); k++) free(arrs[k]);
    free(s->aq);
    free(s);
}

OScene* oracle_scene_new(const float* verts, const float* albedo, int64_t n, const float* lights,
                         int nL, const float* cam, int W, int H) {
    if (n <= 0 || nL < 0 || nL > 64) return NULL;
    OScene* s = (OScene*)calloc(1, sizeof(OScene));
    s->n = n; s->nL = nL; s->W = W; s->H = H;
    float** soa[] = {&s->v0x, &s->v0y, &s->v0z, &s->e1x, &s->e1y, &s->e1z, &s->e2x, &s->e2y, &s->e2z,
                     &s->area};
    for (unsigned k = 0; k < sizeof(soa) / sizeof(soa[0]); k++) *soa[k] = (float*)malloc(sizeof(float) * n);
    s->nrm = (float*)malloc(sizeof(float) * 3 * n);
    s->cen = (float*)malloc(sizeof(float) * 3 * n);
    s->alb = (float*)malloc(sizeof(float) * 3 * n);
    s->vert = (float*)malloc(sizeof(float) * 9 * n);
    s->aq = (uint64_t*)malloc(sizeof(uint64_t) * n);
    memcpy(s->vert, verts, sizeof(float) * 9 * n);
    memcpy(s->alb, albedo, sizeof(float) * 3 * n);
    if (nL) memcpy(s->lights, lights, sizeof(float) * 16 * nL);
    memcpy(s->cam, cam, sizeof(float) * 14);
    s->bad = -1;
    for (int64_t i = 0; i < n; i++) {
        tri_prep(s, i);
        if (s->bad < 0 && (!(s->area[i] > 0.0f) || s->aq[i] == 0)) s->bad = i;
    }
    /* scene diagonal over all vertices (R12/R13 constants, in double) */
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = 0; i < 3 * n; i++)
        for (int a = 0; a < 3; a++) {
            float x = s->vert[3 * i + a];
            if (x < lo[a]) lo[a] = x;
            if (x > hi[a]) hi[a] = x;
        }
    double dx = (double)hi[0] - (double)lo[0], dy = (double)hi[1] - (double)lo[1],
           dz = (double)hi[2] - (double)lo[2];
    s->diag = sqrt(dx * dx + dy * dy + dz * dz);
    s->eps = (float)(1e-4 * s->diag);                               /* R13 */
    s->b2 = (float)((0.01 * s->diag) * (0.01 * s->diag));           /* R12 */
    return s;
}

int64_t oracle_scene_bad(const OScene* s) { return s->bad; }
void oracle_scene_consts(const OScene* s, double* diag, float* eps, float* b2) {
    *diag = s->diag; *eps = s->eps; *b2 = s->b2;
}
void oracle_tri_data(const OScene* s, float* nrm, float* cen, float* area, uint64_t* aq) {
    memcpy(nrm, s->nrm, sizeof(float) * 3 * s->n);
    memcpy(cen, s->cen, sizeof(float) * 3 * s->n);
    memcpy(area, s->area, sizeof(float) * s->n);
    memcpy(aq, s->aq, sizeof(uint64_t) * s->n);
}

/* ------------------------------------------------------------------------ */
/* O9 — Moller-Trumbore, brute force over every triangle.                    */
/* closest hit: u = a_u/det, v = a_v/det, t = a_t/det (inv = 1/det),        */
/*   hit(i) <=> det != 0 & u>=0 & u<=1 & v>=0 & u+v<=1 & tmin<t & t<tmax    */
/* any hit (V of Eq. 1, reading R25): the same predicate without the        */
/* division — a_u, a_v, a_t sign-normalised by det (exact negations), D=|det|*/
/* — and its cross and dot products as fused multiply-adds (R26):           */
/*   cross(a,b).x = fma(a.y, b.z, -(a.z*b.y)) (cyclic), dot(a,b) =          */
/*   fma(a.z, b.z, fma(a.y, b.y, a.x*b.x))                                  */
/*   hit(i) <=> a_u>=0 & a_u<=D & a_v>=0 & a_u+a_v<=D & a_t>tmin*D & a_t<tmax*D */
/* ------------------------------------------------------------------------ */
#define CHUNK 2048

#if ORACLE_O0
/* O0 any hit: SPEC S:134-150 verbatim (inv = 1/det, no fma) */
static int any_hit_chunk(const OScene* s, f3 o, f3 d, float tmin, float tmax, int64_t i0, int64_t i1) {
    int hit = 0;
    for (int64_t i = i0; i < i1; i++) {
        f3 e1 = mk(s->e1x[i], s->e1y[i], s->e1z[i]), e2 = mk(s->e2x[i], s->e2y[i], s->e2z[i]);
        f3 pv = cross(d, e2);
        float det = dot(e1, pv);
        float inv = 1.0f / det;
        f3 sv = sub(o, mk(s->v0x[i], s->v0y[i], s->v0z[i]));
        float u = dot(sv, pv) * inv;
        f3 q = cross(sv, e1);
        float v = dot(d, q) * inv;
        float t = dot(e2, q) * inv;
        hit |= (det != 0.0f) & (u >= 0.0f) & (u <= 1.0f) & (v >= 0.0f) & ((u + v) <= 1.0f) & (t > tmin) & (t < tmax);
    }
    return hit;
}
#else
static int any_hit_chunk(const OScene* s, f3 o, f3 d, float tmin, float tmax, int64_t i0, int64_t i1) {
    int hit = 0;
    for (int64_t i = i0; i < i1; i++) {
        float e1x = s->e1x[i], e1y = s->e1y[i], e1z = s->e1z[i];
        float e2x = s->e2x[i], e2y = s->e2y[i], e2z = s->e2z[i];
        /* R26: fused multiply-adds in the stated order (fmaf is IEEE fma, one rounding) */
        float pvx = fmaf(d.y, e2z, -(d.z * e2y));
        float pvy = fmaf(d.z, e2x, -(d.x * e2z));
        float pvz = fmaf(d.x, e2y, -(d.y * e2x));
        float det = fmaf(e1z, pvz, fmaf(e1y, pvy, e1x * pvx));
        float sx = o.x - s->v0x[i], sy = o.y - s->v0y[i], sz = o.z - s->v0z[i];
        float au = fmaf(sz, pvz, fmaf(sy, pvy, sx * pvx));
        float qx = fmaf(sy, e1z, -(sz * e1y));
        float qy = fmaf(sz, e1x, -(sx * e1z));
        float qz = fmaf(sx, e1y, -(sy * e1x));
        float av = fmaf(d.z, qz, fmaf(d.y, qy, d.x * qx));
        float at = fmaf(e2z, qz, fmaf(e2y, qy, e2x * qx));
        if (det < 0.0f) { au = -au; av = -av; at = -at; }   /* sign-normalise (exact) */
        float D = fabsf(det);
        int h = (au >= 0.0f) & (au <= D) & (av >= 0.0f) & ((au + av) <= D) & (at > tmin * D) & (at < tmax * D);
        hit |= h;
    }
    return hit;
}
#endif

static int any_hit(const OScene* s, f3 o, f3 d, float tmin, float tmax) {
    for (int64_t i0 = 0; i0 < s->n; i0 += CHUNK) {
        int64_t i1 = i0 + CHUNK < s->n ? i0 + CHUNK : s->n;
        if (any_hit_chunk(s, o, d, tmin, tmax, i0, i1)) return 1;
    }
    return 0;
}

/* per-triangle hit t as an order-preserving key (t > tmin >= 0 so t > 0):  */
/* bits(t) for a hit, 0xFFFFFFFF for a miss                                   */
static uint32_t min_key_chunk(const OScene* s, f3 o, f3 d, float tmin, float tmax, int64_t i0, int64_t i1) {
    uint32_t best = 0xFFFFFFFFu;
    for (int64_t i = i0; i < i1; i++) {
        float e1x = s->e1x[i], e1y = s->e1y[i], e1z = s->e1z[i];
        float e2x = s->e2x[i], e2y = s->e2y[i], e2z = s->e2z[i];
        float pvx = d.y * e2z - d.z * e2y;
        float pvy = d.z * e2x - d.x * e2z;
        float pvz = d.x * e2y - d.y * e2x;
        float det = (e1x * pvx + e1y * pvy) + e1z * pvz;
        float inv = 1.0f / det;
        float sx = o.x - s->v0x[i], sy = o.y - s->v0y[i], sz = o.z - s->v0z[i];
        float u = ((sx * pvx + sy * pvy) + sz * pvz) * inv;
        float qx = sy * e1z - sz * e1y;
        float qy = sz * e1x - sx * e1z;
        float qz = sx * e1y - sy * e1x;
        float v = ((d.x * qx + d.y * qy) + d.z * qz) * inv;
        float t = ((e2x * qx + e2y * qy) + e2z * qz) * inv;
        int h = (det != 0.0f) & (u >= 0.0f) & (u <= 1.0f) & (v >= 0.0f) & ((u + v) <= 1.0f) &
                (t > tmin) & (t < tmax);
        uint32_t tb;
        memcpy(&tb, &t, 4);
        uint32_t key = h ? tb : 0xFFFFFFFFu;
        best = key < best ? key : best;
    }
    return best;
}

/* closest hit = lexicographic min of (t, original index) (O9, R15) */
static int64_t closest_hit(const OScene* s, f3 o, f3 d, float tmin, float tmax, float* t_out) {
    uint32_t best = 0xFFFFFFFFu;
    int64_t best_chunk = -1;
    for (int64_t i0 = 0; i0 < s->n; i0 += CHUNK) {
        int64_t i1 = i0 + CHUNK < s->n ? i0 + CHUNK : s->n;
        uint32_t k = min_key_chunk(s, o, d, tmin, tmax, i0, i1);
        if (k < best) { best = k; best_chunk = i0; }
    }
    if (best_chunk < 0) return -1;
    int64_t i1 = best_chunk + CHUNK < s->n ? best_chunk + CHUNK : s->n;
    for (int64_t i = best_chunk; i < i1; i++)
        if (min_key_chunk(s, o, d, tmin, tmax, i, i + 1) == best) {
            memcpy(t_out, &best, 4);
            return i;
        }
    return -1; /* unreachable */
}

/* unoccluded(a, b) (O9): segment shrunk by eps at both ends */
static int occluded(const OScene* s, f3 a, f3 b) {
    f3 d = sub(b, a);
    float dist = sqrtf(dot(d, d));
#if ORACLE_O0
    f3 dir = mk(d.x / dist, d.y / dist, d.z / dist);   /* O9: dir = d / dist */
#else
    float inv = 1.0f / dist;                       /* R25: one division, three products */
    f3 dir = mk(d.x * inv, d.y * inv, d.z * inv);
#endif
    float tmin = s->eps, tmax = dist - s->eps;
    if (!(tmax > tmin)) return 0;
    return any_hit(s, a, dir, tmin, tmax);
}

/* exported single-query helpers (used by the pins) */
int64_t oracle_closest_hit(const OScene* s, const float* o, const float* d, float tmin, float tmax, float* t) {
    return closest_hit(s, ld3(o), ld3(d), tmin, tmax, t);
}
int oracle_occluded(const OScene* s, const float* a, const float* b) { return occluded(s, ld3(a), ld3(b)); }
void oracle_occluded_batch(const OScene* s, const float* a, const float* b, int64_t n, uint8_t* out) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < n; i++) out[i] = (uint8_t)occluded(s, ld3(a + 3 * i), ld3(b + 3 * i));
}
void oracle_closest_batch(const OScene* s, const float* o, const float* d, int64_t n, float tmin, float tmax,
                          int64_t* idx, float* t) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < n; i++) {
        float tt = 0.0f;
        idx[i] = closest_hit(s, ld3(o + 3 * i), ld3(d + 3 * i), tmin, tmax, &tt);
        t[i] = tt;
    }
}

/* ------------------------------------------------------------------------ */
/* O2 — near/far classification: centroid strictly inside the view    */
/* frustum AND closer than T.  cam = pos fwd up right tan_x tan_y.           */
/* ------------------------------------------------------------------------ */
void oracle_classify(const OScene* s, double T, uint8_t* labels, int64_t* n_near) {
    const float* c = s->cam;
    f3 pos = ld3(c), fwd = ld3(c + 3), up = ld3(c + 6), right = ld3(c + 9);
    float tx = c[12], ty = c[13];
    float T2 = (float)(T * T);
    int64_t cnt = 0;
    for (int64_t i = 0; i < s->n; i++) {
        f3 d = sub(ld3(s->cen + 3 * i), pos);
        float z = dot(d, fwd), x = dot(d, right), y = dot(d, up);
        int near = (z > 0.0f) && (fabsf(x) < z * tx) && (fabsf(y) < z * ty) && (dot(d, d) < T2);
        labels[i] = (uint8_t)near;
        cnt += near;
    }
    *n_near = cnt;
}

/* ------------------------------------------------------------------------ */
/* VPL generation (P:44-65 near part; P:35, P:46 step 3 far part).           */
/* ------------------------------------------------------------------------ */
typedef struct {
    int64_t M, K_near, max_depth, rr, n_walks_fixed;
    uint64_t seed;
} OParams;

typedef struct {
    int64_t n_near, n_lit, K, M_far, n_walks, flags, n_far_tris, n_out;
} OInfo;

enum { FLAG_EMPTY_NEAR = 1, FLAG_EMPTY_FAR = 2, FLAG_WALK_BUDGET_UNMET = 4 };

typedef struct {
    float pos[3], nrm[3], flux[3];
    int32_t tri, tag, depth, walk;
} OVpl; /* tag 0 = near (patch), 1 = far (walk) */

static inline f3 light_corner(const float* L) { return ld3(L); }
static inline f3 light_eu(const float* L) { return ld3(L + 3); }
static inline f3 light_ev(const float* L) { return ld3(L + 6); }
static inline f3 light_n(const float* L) { return ld3(L + 9); }
/* Point lights (reading R27, "the light sources are all point lights",
 * Eq. 2's literal form P:51-56): a light row with area == 0 is an isotropic
 * point light at `corner` (e_u = e_v = 0) whose `radiance` field holds its
 * power Phi (W per channel, R3).  It has no facing side. */
static inline int light_is_point(const float* L) { return L[12] == 0.0f; }
/* Eq. 2's geometry term for a point light without D (R1: omega_i and r
 * relative to the light): cos(omega) / (4 pi r^2) = cp / ((r2 * sqrt(r2)) * 4pi),
 * cp = n.d (unnormalised d = light - x, so cos(omega) = cp / r). */
static inline float point_g(float cp, float r2) {
    const float FOUR_PI = (float)(4.0 * PI_D);
    return cp / ((r2 * sqrtf(r2)) * FOUR_PI);
}
/* light centre = (corner + 0.5*e_u) + 0.5*e_v (O3) */
static inline f3 light_centre(const float* L) {
    return add(add(light_corner(L), scl(0.5f, light_eu(L))), scl(0.5f, light_ev(L)));
}

/* O3 — a near triangle is lit iff some light faces it, it faces the light,
 * and the centroid -> light-centre segment is unoccluded (R6). */
void oracle_lit(const OScene* s, const uint8_t* labels, uint8_t* lit) {
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t i = 0; i < s->n; i++) {
        lit[i] = 0;
        if (!labels[i]) continue;
        f3 c = ld3(s->cen + 3 * i), n = ld3(s->nrm + 3 * i);
        for (int l = 0; l < s->nL; l++) {
            const float* L = s->lights + 16 * l;
            f3 cl = light_centre(L);
            if (dot(n, sub(cl, c)) > 0.0f && (light_is_point(L) || dot(light_n(L), sub(c, cl)) > 0.0f) &&
                !occluded(s, c, cl)) {
                lit[i] = 1;
                break;
            }
        }
    }
}

/* O4 — 30-bit Morton code, bit i of qx -> 3i, qy -> 3i+1, qz -> 3i+2 */
uint32_t oracle_morton3(uint32_t qx, uint32_t qy, uint32_t qz) {
    uint32_t code = 0;
    for (int b = 0; b < 10; b++) {
        code |= ((qx >> b) & 1u) << (3 * b);
        code |= ((qy >> b) & 1u) << (3 * b + 1);
        code |= ((qz >> b) & 1u) << (3 * b + 2);
    }
    return code;
}

typedef struct { uint32_t code; int64_t idx; } MKey;
static int mkey_cmp(const void* a, const void* b) {
    const MKey *x = (const MKey*)a, *y = (const MKey*)b;
    if (x->code != y->code) return x->code < y->code ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

/* O4 + O5: order the lit-near set along the Morton curve and build
 * the inclusive prefix f(i) of fixed-point areas.  Returns n_lit.    */
int64_t oracle_near_table(const OScene* s, const uint8_t* lit, int64_t* order, uint64_t* P, uint32_t* codes) {
    int64_t m = 0;
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = 0; i < s->n; i++)
        if (lit[i]) {
            m++;
            for (int a = 0; a < 3; a++) {
                float x = s->cen[3 * i + a];
                if (x < lo[a]) lo[a] = x;
                if (x > hi[a]) hi[a] = x;
            }
        }
    if (m == 0) return 0;
    float scale[3];
    for (int a = 0; a < 3; a++) {
        float ext = hi[a] - lo[a];
        scale[a] = ext > 0.0f ? 1024.0f / ext : 0.0f;
    }
    MKey* keys = (MKey*)malloc(sizeof(MKey) * m);
    int64_t k = 0;
    for (int64_t i = 0; i < s->n; i++)
        if (lit[i]) {
            uint32_t q[3];
            for (int a = 0; a < 3; a++) {
                uint32_t qa = (uint32_t)((s->cen[3 * i + a] - lo[a]) * scale[a]);
                q[a] = qa < 1023u ? qa : 1023u;
            }
            keys[k].code = oracle_morton3(q[0], q[1], q[2]);
            keys[k].idx = i;
            k++;
        }
    qsort(keys, m, sizeof(MKey), mkey_cmp);
    uint64_t acc = 0;
    for (int64_t j = 0; j < m; j++) {
        order[j] = keys[j].idx;
        if (codes) codes[j] = keys[j].code;
        acc += s->aq[keys[j].idx];
        P[j] = acc; /* f(j) = sum_{i<=j} s_i */
    }
    free(keys);
    return m;
}

/* O6 — stratum k: s_k = floor((k*2^32 + x) * F / (K*2^32)), x = raw draw 0;
 * j = g(s_k) = first index with P[j] > s_k.           */
uint64_t oracle_stratum(uint64_t seed, int64_t k, int64_t K, uint64_t F) {
    uint32_t x = oracle_draw(seed, STREAM_NEAR, (uint32_t)k, 0);
    unsigned __int128 num = (((unsigned __int128)(uint64_t)k << 32) + x) * (unsigned __int128)F;
    unsigned __int128 den = ((unsigned __int128)(uint64_t)K) << 32;
    return (uint64_t)(num / den);
}
int64_t oracle_lookup_g(const uint64_t* P, int64_t m, uint64_t sk) {
    int64_t j = 0; /* linear scan: the plain definition of g */
    while (j < m && !(P[j] > sk)) j++;
    return j;
}

/* O7 — uniform point in triangle via the square-root warp ([r10]). */
static f3 point_in_tri(const OScene* s, int64_t t, float u1, float u2) {
    const float* v = s->vert + 9 * t;
    f3 v0 = ld3(v), v1 = ld3(v + 3), v2 = ld3(v + 6);
    float su = sqrtf(u1);
    float b1 = 1.0f - su;
    float b2 = u2 * su;
    float b0 = (1.0f - b1) - b2;
    return add(add(scl(b1, v0), scl(b2, v1)), scl(b0, v2));
}
void oracle_point_in_tri(const OScene* s, int64_t t, float u1, float u2, float* p) {
    f3 r = point_in_tri(s, t, u1, u2);
    p[0] = r.x; p[1] = r.y; p[2] = r.z;
}

/* O8 — Eq. 2 for area lights (R1-R5): VPL flux =
 * rho/pi * D * sum_l L_l * A_l cos_p cos_l / r^2 * V, D = f(N)/K.          */
static void near_vpl(const OScene* s, const OParams* p, const int64_t* order, const uint64_t* P, int64_t m,
                     int64_t K, float D, int64_t k, OVpl* out) {
    uint64_t F = P[m - 1];
    uint64_t sk = oracle_stratum(p->seed, k, K, F);
    int64_t j = oracle_lookup_g(P, m, sk);
    int64_t t = order[j];
    float u1 = u01(oracle_draw(p->seed, STREAM_NEAR, (uint32_t)k, 1));
    float u2 = u01(oracle_draw(p->seed, STREAM_NEAR, (uint32_t)k, 2));
    f3 x = point_in_tri(s, t, u1, u2);
    f3 n = ld3(s->nrm + 3 * t);
    float E[3] = {0.0f, 0.0f, 0.0f};
    for (int l = 0; l < s->nL; l++) {
        const float* L = s->lights + 16 * l;
        float u3 = u01(oracle_draw(p->seed, STREAM_NEAR, (uint32_t)k, 3 + 2 * l));
        float u4 = u01(oracle_draw(p->seed, STREAM_NEAR, (uint32_t)k, 4 + 2 * l));
        f3 y = add(add(light_corner(L), scl(u3, light_eu(L))), scl(u4, light_ev(L)));
        f3 d = sub(y, x);
        float r2 = dot(d, d);
        float cp = dot(n, d);
        if (light_is_point(L)) { /* R27: Phi * cos(omega) / (4 pi r^2) * V */
            if (cp > 0.0f && !occluded(s, x, y)) {
                float g = point_g(cp, r2);
                for (int c = 0; c < 3; c++) E[c] += L[13 + c] * g;
            }
            continue;
        }
        float cl = -dot(light_n(L), d);
        if (cp > 0.0f && cl > 0.0f && !occluded(s, x, y)) {
            float g = ((L[12] * cp) * cl) / (r2 * r2);
            for (int c = 0; c < 3; c++) E[c] += L[13 + c] * g;
        }
    }
    const float INV_PI = (float)(1.0 / PI_D);
    out->pos[0] = x.x; out->pos[1] = x.y; out->pos[2] = x.z;
    out->nrm[0] = n.x; out->nrm[1] = n.y; out->nrm[2] = n.z;
    for (int c = 0; c < 3; c++) out->flux[c] = (s->alb[3 * t + c] * (D * E[c])) * INV_PI;
    out->tri = (int32_t)t; out->tag = 0; out->depth = 0; out->walk = (int32_t)k;
}

/* Malley cosine direction around unit n with the Duff et al. basis (O10). */
static f3 malley(const OScene* s, uint64_t seed, uint32_t w, uint32_t* j, f3 n) {
    (void)s;
    float a = 0.0f, b = 0.0f, q = 0.0f;
    int found = 0;
    for (int att = 0; att < 64; att++) {
        float ua = u01(oracle_draw(seed, STREAM_WALK, w, (*j)++));
        float ub = u01(oracle_draw(seed, STREAM_WALK, w, (*j)++));
        a = 2.0f * ua - 1.0f;
        b = 2.0f * ub - 1.0f;
        q = a * a + b * b;
        if (q < 1.0f) { found = 1; break; }
    }
    if (!found) { a = 0.0f; b = 0.0f; q = 0.0f; }
    float z = sqrtf(1.0f - q);
    float sg = copysignf(1.0f, n.z);
    float ia = -1.0f / (sg + n.z);
    float bb = (n.x * n.y) * ia;
    f3 t1 = mk(1.0f + sg * ((n.x * n.x) * ia), sg * bb, -sg * n.x);
    f3 t2 = mk(bb, sg + (n.y * n.y) * ia, -n.y);
    return mk((a * t1.x + b * t2.x) + z * n.x, (a * t1.y + b * t2.y) + z * n.y, (a * t1.z + b * t2.z) + z * n.z);
}

/* Uniform direction on the sphere for a point light's emission (R27), with
 * no transcendental: rejection in the cube, a,b,c = 2U - 1 until
 * 0 < a*a + b*b + c*c <= 1 (at most 64 attempts, else (0, 0, 1)); the
 * direction (a, b, c) is not normalised (MT and x = o + t*dir do not need it). */
static f3 sphere_dir(uint64_t seed, uint32_t w, uint32_t* j) {
    for (int att = 0; att < 64; att++) {
        float a = 2.0f * u01(oracle_draw(seed, STREAM_WALK, w, (*j)++)) - 1.0f;
        float b = 2.0f * u01(oracle_draw(seed, STREAM_WALK, w, (*j)++)) - 1.0f;
        float c = 2.0f * u01(oracle_draw(seed, STREAM_WALK, w, (*j)++)) - 1.0f;
        float q = (a * a + b * b) + c * c;
        if (q > 0.0f && q <= 1.0f) return mk(a, b, c);
    }
    return mk(0.0f, 0.0f, 1.0f);
}

/* O10 — one sparse-IR walk (P:15, P:35, P:46 step 3; R9-R11).  Writes up to
 * max_depth deposits (flux not yet divided by the walk count); returns count. */
static int walk(const OScene* s, const OParams* p, const uint8_t* labels, uint32_t w, OVpl* dep) {
    uint32_t j = 0;
    uint32_t x0 = oracle_draw(p->seed, STREAM_WALK, w, j++);
    int l = (int)(((uint64_t)x0 * (uint64_t)s->nL) >> 32);
    const float* L = s->lights + 16 * l;
    float beta[3];
    /* beta0 = power of light l x n_L: pi A L for an area light, Phi for a point light (R27) */
    for (int c = 0; c < 3; c++)
        beta[c] = light_is_point(L) ? (float)((double)L[13 + c] * (double)s->nL)
                                    : (float)(PI_D * (double)L[12] * (double)L[13 + c] * (double)s->nL);
    float u1 = u01(oracle_draw(p->seed, STREAM_WALK, w, j++));
    float u2 = u01(oracle_draw(p->seed, STREAM_WALK, w, j++));
    f3 o = add(add(light_corner(L), scl(u1, light_eu(L))), scl(u2, light_ev(L)));   /* point: e_u = e_v = 0 */
    f3 dir = light_is_point(L) ? sphere_dir(p->seed, w, &j) : malley(s, p->seed, w, &j, light_n(L));
    const float INV_PI = (float)(1.0 / PI_D);
    int cnt = 0;
    for (int d = 1; d <= p->max_depth; d++) {
        float t;
        int64_t h = closest_hit(s, o, dir, s->eps, INFINITY, &t);
        if (h < 0) break;
        f3 nh = ld3(s->nrm + 3 * h);
        if (dot(nh, dir) >= 0.0f) break; /* back face: absorbed */
        f3 x = add(o, scl(t, dir));
        const float* rho = s->alb + 3 * h;
        if (!labels[h]) { /* far patch: deposit (near deposits discarded) */
            OVpl* v = dep + cnt++;
            v->pos[0] = x.x; v->pos[1] = x.y; v->pos[2] = x.z;
            v->nrm[0] = nh.x; v->nrm[1] = nh.y; v->nrm[2] = nh.z;
            for (int c = 0; c < 3; c++) v->flux[c] = (rho[c] * beta[c]) * INV_PI;
            v->tri = (int32_t)h; v->tag = 1; v->depth = d; v->walk = (int32_t)w;
        }
        if (d == p->max_depth) break;
        if (p->rr) {
            float q = ((rho[0] + rho[1]) + rho[2]) / 3.0f;
            float xi = u01(oracle_draw(p->seed, STREAM_WALK, w, j++));
            if (!(xi < q)) break;
            for (int c = 0; c < 3; c++) beta[c] = (beta[c] * rho[c]) / q;
        } else {
            for (int c = 0; c < 3; c++) beta[c] = beta[c] * rho[c];
        }
        dir = malley(s, p->seed, w, &j, nh);
        o = x;
    }
    return cnt;
}

/* Full VPL generation (P:46 steps 1-3).  out must hold max_out records.
 * Returns the number written (n_out) or -1 if max_out is too small.        */
int64_t oracle_generate_vpls(const OScene* s, const uint8_t* labels, const OParams* p, OVpl* out,
                             int64_t max_out, OInfo* info) {
    memset(info, 0, sizeof(*info));
    int64_t n_near = 0, n_far = 0;
    for (int64_t i = 0; i < s->n; i++) {
        n_near += labels[i] != 0;
        n_far += labels[i] == 0;
    }
    info->n_near = n_near;
    info->n_far_tris = n_far;
    uint8_t* lit = (uint8_t*)malloc(s->n);
    int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (s->n + 1));
    uint64_t* P = (uint64_t*)malloc(sizeof(uint64_t) * (s->n + 1));
    int64_t m = 0;
    if (p->K_near > 0 && p->n_walks_fixed == 0) {
        oracle_lit(s, labels, lit);
        m = oracle_near_table(s, lit, order, P, NULL);
    }
    info->n_lit = m;
    int64_t K = p->K_near, Mf = p->M - p->K_near;
    if (p->n_walks_fixed > 0) { K = 0; }
    else if (m == 0) { K = 0; Mf = p->M; info->flags |= FLAG_EMPTY_NEAR; }
    else if (n_far == 0) { K = p->M; Mf = 0; info->flags |= FLAG_EMPTY_FAR; }
    if (K > max_out) { free(lit); free(order); free(P); return -1; }
    info->K = K;
    /* near part: K strata over [0, f(N)) */
    if (K > 0) {
        float D = (float)((double)P[m - 1] / (double)K / 1099511627776.0);
#pragma omp parallel for schedule(dynamic, 8)
        for (int64_t k = 0; k < K; k++) near_vpl(s, p, order, P, m, K, D, k, out + k);
    }
    /* far part: walks in index order, first-M_far-deposits rule (R11) */
    int64_t n_out = K;
    const int64_t B = 1024;
    OVpl* buf = (OVpl*)malloc(sizeof(OVpl) * B * (p->max_depth > 0 ? p->max_depth : 1));
    int* cnt = (int*)malloc(sizeof(int) * B);
    int64_t walks = 0;
    if (p->n_walks_fixed > 0) {
        for (int64_t w0 = 0; w0 < p->n_walks_fixed; w0 += B) {
            int64_t nb = p->n_walks_fixed - w0 < B ? p->n_walks_fixed - w0 : B;
#pragma omp parallel for schedule(dynamic, 1)
            for (int64_t i = 0; i < nb; i++) cnt[i] = walk(s, p, labels, (uint32_t)(w0 + i), buf + i * p->max_depth);
            for (int64_t i = 0; i < nb; i++)
                for (int c = 0; c < cnt[i]; c++) {
                    if (n_out >= max_out) { free(buf); free(cnt); free(lit); free(order); free(P); return -1; }
                    out[n_out++] = buf[i * p->max_depth + c];
                }
        }
        walks = p->n_walks_fixed;
    } else if (Mf > 0) {
        if (K + Mf > max_out) { free(buf); free(cnt); free(lit); free(order); free(P); return -1; }
        int64_t Wmax = 1024 * Mf, have = 0;
        int done = 0;
        for (int64_t w0 = 0; w0 < Wmax && !done; w0 += B) {
            int64_t nb = Wmax - w0 < B ? Wmax - w0 : B;
#pragma omp parallel for schedule(dynamic, 1)
            for (int64_t i = 0; i < nb; i++) cnt[i] = walk(s, p, labels, (uint32_t)(w0 + i), buf + i * p->max_depth);
            for (int64_t i = 0; i < nb && !done; i++) {
                walks = w0 + i + 1;
                for (int c = 0; c < cnt[i] && have < Mf; c++) { out[n_out++] = buf[i * p->max_depth + c]; have++; }
                if (have >= Mf) done = 1;
            }
        }
        if (!done) info->flags |= FLAG_WALK_BUDGET_UNMET;
    }
    /* divide walk fluxes by the number of walks used (R11) */
    if (walks > 0) {
        float fw = (float)walks;
        for (int64_t i = K; i < n_out; i++)
            for (int c = 0; c < 3; c++) out[i].flux[c] = out[i].flux[c] / fw;
    }
    info->M_far = n_out - K;
    info->n_walks = walks;
    info->n_out = n_out;
    free(buf); free(cnt); free(lit); free(order); free(P);
    return n_out;
}

/* ------------------------------------------------------------------------ */
/* O12 — G-buffer at the pixel centre (R16).  Output per pixel:     */
/* gb[12] = pos(3) nrm(3) alb(3) t, tri (as float bits), front (0/1).        */
/* ------------------------------------------------------------------------ */
typedef struct {
    float pos[3], nrm[3], alb[3], t;
    int32_t tri, front;
} OGbuf;

static void primary_dir(const OScene* s, int px, int py, f3* dir_out) {
    const float* c = s->cam;
    f3 fwd = ld3(c + 3), up = ld3(c + 6), right = ld3(c + 9);
    float tx = c[12], ty = c[13];
    float sx = ((2.0f * ((float)px + 0.5f)) / (float)s->W - 1.0f) * tx;
    float sy = (1.0f - (2.0f * ((float)py + 0.5f)) / (float)s->H) * ty;
    f3 d = add(add(fwd, scl(sx, right)), scl(sy, up));
    float len = sqrtf(dot(d, d));
    *dir_out = mk(d.x / len, d.y / len, d.z / len);
}

void oracle_gbuffer(const OScene* s, const int32_t* pix, int64_t n_pix, OGbuf* out) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t k = 0; k < n_pix; k++) {
        int32_t id = pix[k];
        int px = id % s->W, py = id / s->W;
        f3 dir;
        primary_dir(s, px, py, &dir);
        f3 o = ld3(s->cam);
        float t = 0.0f;
        int64_t h = closest_hit(s, o, dir, 0.0f, INFINITY, &t);
        OGbuf* g = out + k;
        memset(g, 0, sizeof(*g));
        g->tri = -1;
        if (h < 0) continue;
        f3 x = add(o, scl(t, dir));
        f3 n = ld3(s->nrm + 3 * h);
        g->pos[0] = x.x; g->pos[1] = x.y; g->pos[2] = x.z;
        g->nrm[0] = n.x; g->nrm[1] = n.y; g->nrm[2] = n.z;
        for (int c = 0; c < 3; c++) g->alb[c] = s->alb[3 * h + c];
        g->t = t;
        g->tri = (int32_t)h;
        g->front = dot(n, dir) < 0.0f;
    }
}

/* ------------------------------------------------------------------------ */
/* O13 — the gather, Eq. 1 indirect term, brute-force visibility:  */
/* L(x) = rho_x/pi * sum_i Phi_i cx ci / (r2 * max(r2, b^2)) * V(x, y_i),     */
/* cx = n_x.d, ci = -n_i.d, d = y_i - x; self-triangle excluded (R14);        */
/* accumulated in fp64 in VPL array order.                                    */
/* Optional per-pixel bitmaps (ceil(M/32) words each): traced (cull passed)  */
/* and visible.                                                               */
/* ------------------------------------------------------------------------ */
void oracle_gather(const OScene* s, const OGbuf* gb, int64_t n_pix, const OVpl* v, int64_t M, float* rgb,
                   double* rgb64, int64_t* traced_count, uint32_t* traced_bits, uint32_t* vis_bits) {
    int64_t words = (M + 31) / 32;
    int64_t total_traced = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : total_traced)
    for (int64_t k = 0; k < n_pix; k++) {
        const OGbuf* g = gb + k;
        double acc[3] = {0.0, 0.0, 0.0};
        if (traced_bits) memset(traced_bits + k * words, 0, sizeof(uint32_t) * words);
        if (vis_bits) memset(vis_bits + k * words, 0, sizeof(uint32_t) * words);
        if (g->tri >= 0 && g->front) {
            f3 x = ld3(g->pos), nx = ld3(g->nrm);
            for (int64_t i = 0; i < M; i++) {
                if (v[i].tri == g->tri) continue;
                f3 y = ld3(v[i].pos);
                f3 d = sub(y, x);
                float r2 = dot(d, d);
                f3 ni = ld3(v[i].nrm);               /* R26: the cosine terms as fused dots */
#if ORACLE_O0
                float cx = dot(nx, d);                /* O13 as written: plain dots */
                float ci = -dot(ni, d);
#else
                float cx = fmaf(nx.z, d.z, fmaf(nx.y, d.y, nx.x * d.x));
                float ci = -fmaf(ni.z, d.z, fmaf(ni.y, d.y, ni.x * d.x));
#endif
                if (!(cx > 0.0f && ci > 0.0f)) continue;
                total_traced++;
                if (traced_bits) traced_bits[k * words + i / 32] |= 1u << (i % 32);
                if (occluded(s, x, y)) continue;
                if (vis_bits) vis_bits[k * words + i / 32] |= 1u << (i % 32);
                double r2d = (double)r2, b2d = (double)s->b2;
                double G = ((double)cx * (double)ci) / (r2d * (r2d > b2d ? r2d : b2d));
                for (int c = 0; c < 3; c++) acc[c] += (double)v[i].flux[c] * G;
            }
        }
        for (int c = 0; c < 3; c++) {
            double val = acc[c] * (double)g->alb[c] / PI_D;
            if (!(g->tri >= 0 && g->front)) val = 0.0;
            rgb[3 * k + c] = (float)val;
            if (rgb64) rgb64[3 * k + c] = val;
        }
    }
    if (traced_count) *traced_count = total_traced;
}

/* ------------------------------------------------------------------------ */
/* O14 — the direct term L_e of Eq. 1 ("L_e(y) represents direct   */
/* illumination"; SPEC shade_direct S:327-335) for the area lights of BJ:7-11 */
/* (reading R21): per pixel, S uniform samples y on every light,            */
/*   E_c += L_l,c * ((A_l * cx) * cl) / (r2 * r2)  if cx > 0, cl > 0, V(x,y), */
/* d = y - x, cx = n_x.d, cl = -n_l.d (the same form as O8), draws 2(lS+s)  */
/* and 2(lS+s)+1 of Philox stream 4, item = pixel index; fp32 in this order. */
/* out_c = (rho_c * (E_c * inv_S + P_c)) * INV_PI; miss / back face -> 0.    */
/* A point light (R27) needs no samples: P_c += Phi_c * cx / ((r2 sqrt r2)  */
/* 4 pi) if cx > 0 and V(x, y) (the same term as O8's point form).          */
/* ------------------------------------------------------------------------ */
void oracle_direct(const OScene* s, const OGbuf* gb, const int32_t* pix, int64_t n_pix, int32_t S, uint64_t seed,
                   float inv_S, float* rgb) {
    const float INV_PI = (float)(1.0 / PI_D);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t k = 0; k < n_pix; k++) {
        const OGbuf* g = gb + k;
        float E[3] = {0.0f, 0.0f, 0.0f}, Pt[3] = {0.0f, 0.0f, 0.0f};
        int ok = g->tri >= 0 && g->front;
        if (ok) {
            f3 x = ld3(g->pos), nx = ld3(g->nrm);
            for (int l = 0; l < s->nL; l++) {
                const float* L = s->lights + 16 * l;
                if (light_is_point(L)) {
                    f3 y = light_corner(L);
                    f3 d = sub(y, x);
                    float r2 = dot(d, d);
                    float cx = dot(nx, d);
                    if (cx > 0.0f && !occluded(s, x, y)) {
                        float gg = point_g(cx, r2);
                        for (int c = 0; c < 3; c++) Pt[c] += L[13 + c] * gg;
                    }
                    continue;
                }
                for (int q = 0; q < S; q++) {
                    uint32_t j = 2u * (uint32_t)(l * S + q);
                    float u = u01(oracle_draw(seed, STREAM_DIRECT, (uint32_t)pix[k], j));
                    float v = u01(oracle_draw(seed, STREAM_DIRECT, (uint32_t)pix[k], j + 1));
                    f3 y = add(add(light_corner(L), scl(u, light_eu(L))), scl(v, light_ev(L)));
                    f3 d = sub(y, x);
                    float r2 = dot(d, d);
                    float cx = dot(nx, d);
                    float cl = -dot(light_n(L), d);
                    if (cx > 0.0f && cl > 0.0f && !occluded(s, x, y)) {
                        float gg = ((L[12] * cx) * cl) / (r2 * r2);
                        for (int c = 0; c < 3; c++) E[c] += L[13 + c] * gg;
                    }
                }
            }
        }
        for (int c = 0; c < 3; c++) rgb[3 * k + c] = ok ? (g->alb[c] * ((E[c] * inv_S) + Pt[c])) * INV_PI : 0.0f;
    }
}

/* ------------------------------------------------------------------------ */
/* O15 — the rejection-sampling comparator (P:29-32 [r3]: "reject those VPLs */
/* that contribute less than the average value to the resulting image";     */
/* SPEC generate_rejection_vpls S:252-260; reading R23).                     */
/* Probes: a 8 x 8 grid of image blocks, one pixel per block, offset        */
/* floor(U(draw 0 / 1 of Philox stream 5, item b) * block size).             */
/* ------------------------------------------------------------------------ */
void oracle_probe_pixels(int W, int H, uint64_t seed, int32_t* pix /* [64] */) {
    for (int b = 0; b < 64; b++) {
        int bx = b % 8, by = b / 8;
        int x0 = bx * W / 8, x1 = (bx + 1) * W / 8, y0 = by * H / 8, y1 = (by + 1) * H / 8;
        float u = u01(oracle_draw(seed, STREAM_PROBE, (uint32_t)b, 0));
        float v = u01(oracle_draw(seed, STREAM_PROBE, (uint32_t)b, 1));
        int px = x0 + (int)(u * (float)(x1 - x0));
        int py = y0 + (int)(v * (float)(y1 - y0));
        pix[b] = py * W + px;
    }
}

/* lum(c) = ((c.r + c.g) + c.b) / 3 */
static inline float lum3(const float* c) { return ((c[0] + c[1]) + c[2]) / 3.0f; }

/* probe scores of the pilot candidates (shared by O15 and O16) */
static void probe_scores(const OScene* s, const OGbuf* probes, int64_t nq, const OVpl* pilot, int64_t np_,
                         float* sc) {
#pragma omp parallel for schedule(dynamic, 8)
    for (int64_t i = 0; i < np_; i++) {
        float acc = 0.0f;
        float li = lum3(pilot[i].flux);
        f3 y = ld3(pilot[i].pos), ny = ld3(pilot[i].nrm);
        for (int64_t q = 0; q < nq; q++) {
            const OGbuf* g = probes + q;
            float t = 0.0f;
            if (g->tri >= 0 && g->front && g->tri != pilot[i].tri) {
                f3 x = ld3(g->pos), nx = ld3(g->nrm);
                f3 d = sub(y, x);
                float r2 = dot(d, d);
                float cx = dot(nx, d);
                float ci = -dot(ny, d);
                if (cx > 0.0f && ci > 0.0f && !occluded(s, x, y)) {
                    float w = (cx * ci) / (r2 * (r2 > s->b2 ? r2 : s->b2));
                    t = (w * li) * lum3(g->alb);
                }
            }
            acc += t;
        }
        sc[i] = acc;
    }
}

/* Score of candidate i: s_i = sum over probes q = 0..nq-1, in that order, in
 * fp32 of t_iq = ((cx*ci) / (r2 * max(r2, b^2)) * lum(Phi_i)) * lum(rho_q)
 * when the Eq. 1 term is traced (O13's cull and self-exclusion) and visible,
 * else 0 — the Eq. 1 summand of the VPL at the probe, as luminance.
 * mean = fp64 sum of the scores in index order / pilot.
 * Acceptance ([r3]'s rejection rule, made unbiased — reading R23):
 *   p_i = max(P_MIN, min(1, s_i / mean)) in fp64 (p_i = 1 when mean = 0),
 *   accept iff (double)U(draw 0 of Philox stream 6, item i) < p_i,
 * scanning in index order until `budget` are accepted (n_scanned = index of
 * the last one + 1, or pilot).  Kept flux = Phi * (float)((pilot / n_scanned)
 * / p_i): the scanned prefix stands for the whole pilot, 1/p_i undoes the
 * thinning.  Returns the number accepted (<= budget); out holds them. */
#define REJ_P_MIN 0.05
int64_t oracle_rejection(const OScene* s, const OGbuf* probes, int64_t nq, const OVpl* pilot, int64_t np_,
                         int64_t budget, uint64_t seed, OVpl* out, float* scores, double* mean_out,
                         int64_t* n_scanned_out) {
    float* sc = scores ? scores : (float*)malloc(sizeof(float) * (size_t)(np_ > 0 ? np_ : 1));
    probe_scores(s, probes, nq, pilot, np_, sc);
    double sum = 0.0;
    for (int64_t i = 0; i < np_; i++) sum += (double)sc[i];
    double mean = np_ > 0 ? sum / (double)np_ : 0.0;
    if (mean_out) *mean_out = mean;
    int64_t* acc_i = (int64_t*)malloc(sizeof(int64_t) * (size_t)(budget > 0 ? budget : 1));
    double* acc_p = (double*)malloc(sizeof(double) * (size_t)(budget > 0 ? budget : 1));
    int64_t o = 0, scanned = np_;
    for (int64_t i = 0; i < np_ && o < budget; i++) {
        double p = mean > 0.0 ? (double)sc[i] / mean : 1.0;
        if (p > 1.0) p = 1.0;
        if (p < REJ_P_MIN) p = REJ_P_MIN;
        double u = (double)u01(oracle_draw(seed, STREAM_REJECT, (uint32_t)i, 0));
        if (u < p) {
            acc_i[o] = i;
            acc_p[o] = p;
            o++;
            if (o == budget) scanned = i + 1;
        }
    }
    for (int64_t k = 0; k < o; k++) {
        float f = (float)(((double)np_ / (double)scanned) / acc_p[k]);
        out[k] = pilot[acc_i[k]];
        for (int c = 0; c < 3; c++) out[k].flux[c] = out[k].flux[c] * f;
    }
    free(acc_i); free(acc_p);
    if (!scores) free(sc);
    if (n_scanned_out) *n_scanned_out = scanned;
    return o;
}

/* ------------------------------------------------------------------------ */
/* O16 — the Metropolis comparator (P:31-32 [r2]: "distributes VPLs according */
/* to Metropolis-Hastings sampling"; reading R24).  The paper */
/* gives no mutation details; this is a Metropolis-Hastings sampler over the  */
/* pilot candidates laid out along their Morton curve (the O4 quantisation    */
/* over the pilot's position box, ties by index), target                      */
/* f_j = max(s_pool[j], 0.05 mean) (O15's probe scores), symmetric local      */
/* mutation j' = j + delta (mod pilot), delta uniform in [-R, R] \ {0}.      */
/* Chain c (Philox stream 7, item c, draws in sequence): start              */
/* j = (x0 * pilot) >> 32; each step k = (x * 2R) >> 32, delta = k - R (k < R) */
/* else k - R + 1, accept iff (double)U(next draw) < f_j' / f_j (fp64).      */
/* After `burn` steps every state is emitted; flux *= (float)((pilot / N) *  */
/* (mean_f / f_j)), mean_f = fp64 sum of f in pool order / pilot, N =       */
/* chains * per_chain: the 1/p importance weight of the stationary law.      */
/* Returns N; out[c * per_chain + t] is chain c's t-th emitted state.         */
/* ------------------------------------------------------------------------ */
#define MH_LARGE 0.3
int64_t oracle_metropolis(const OScene* s, const OGbuf* probes, int64_t nq, const OVpl* pilot, int64_t np_,
                          int64_t chains, int64_t per_chain, int64_t burn, int64_t R, uint64_t seed, OVpl* out,
                          float* scores, int64_t* pool_out, int64_t* accepted_out) {
    if (np_ < 2 || chains < 1 || per_chain < 0 || burn < 0 || R < 1) return 0;
    float* sc = scores ? scores : (float*)malloc(sizeof(float) * (size_t)np_);
    probe_scores(s, probes, nq, pilot, np_, sc);
    double sum = 0.0;
    for (int64_t i = 0; i < np_; i++) sum += (double)sc[i];
    double mean = sum / (double)np_;
    /* pool: Morton order of the pilot positions (O4 formula) */
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = 0; i < np_; i++)
        for (int a = 0; a < 3; a++) {
            if (pilot[i].pos[a] < lo[a]) lo[a] = pilot[i].pos[a];
            if (pilot[i].pos[a] > hi[a]) hi[a] = pilot[i].pos[a];
        }
    float scale[3];
    for (int a = 0; a < 3; a++) {
        float ext = hi[a] - lo[a];
        scale[a] = ext > 0.0f ? 1024.0f / ext : 0.0f;
    }
    MKey* keys = (MKey*)malloc(sizeof(MKey) * (size_t)np_);
    for (int64_t i = 0; i < np_; i++) {
        uint32_t q[3];
        for (int a = 0; a < 3; a++) {
            uint32_t qa = (uint32_t)((pilot[i].pos[a] - lo[a]) * scale[a]);
            q[a] = qa < 1023u ? qa : 1023u;
        }
        keys[i].code = oracle_morton3(q[0], q[1], q[2]);
        keys[i].idx = i;
    }
    qsort(keys, (size_t)np_, sizeof(MKey), mkey_cmp);
    double* f = (double*)malloc(sizeof(double) * (size_t)np_);
    double fsum = 0.0;
    for (int64_t j = 0; j < np_; j++) {
        double v = mean > 0.0 ? (double)sc[keys[j].idx] : 1.0;
        double fl = 0.05 * mean;
        f[j] = v > fl ? v : fl;
        if (pool_out) pool_out[j] = keys[j].idx;
        fsum += f[j];
    }
    double mean_f = fsum / (double)np_;
    int64_t N = chains * per_chain;
    int64_t acc_total = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : acc_total)
    for (int64_t c = 0; c < chains; c++) {
        uint32_t j = 0;
        uint32_t x0 = oracle_draw(seed, STREAM_MH, (uint32_t)c, j++);
        int64_t cur = (int64_t)(((uint64_t)x0 * (uint64_t)np_) >> 32);
        for (int64_t t = 0; t < burn + per_chain; t++) {
            double sel = (double)u01(oracle_draw(seed, STREAM_MH, (uint32_t)c, j++));
            uint32_t xk = oracle_draw(seed, STREAM_MH, (uint32_t)c, j++);
            int64_t nxt;
            if (sel < MH_LARGE) {                     /* large step: uniform over the pool */
                nxt = (int64_t)(((uint64_t)xk * (uint64_t)np_) >> 32);
            } else {                                  /* small step: local Morton neighbour */
                int64_t k = (int64_t)(((uint64_t)xk * (uint64_t)(2 * R)) >> 32);
                int64_t delta = k < R ? k - R : k - R + 1;
                nxt = ((cur + delta) % np_ + np_) % np_;
            }
            double u = (double)u01(oracle_draw(seed, STREAM_MH, (uint32_t)c, j++));
            if (u < f[nxt] / f[cur]) { cur = nxt; acc_total++; }
            if (t >= burn) {
                OVpl* o = out + c * per_chain + (t - burn);
                *o = pilot[keys[cur].idx];
                float w = (float)(((double)np_ / (double)N) * (mean_f / f[cur]));
                for (int a = 0; a < 3; a++) o->flux[a] = o->flux[a] * w;
            }
        }
    }
    if (accepted_out) *accepted_out = acc_total;
    free(keys); free(f);
    if (!scores) free(sc);
    return N;
}

/* visibility of explicit (point, VPL) pairs — for sampled-pair parity */
void oracle_pair_visibility(const OScene* s, const float* x, const float* y, int64_t n, uint8_t* vis) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < n; i++) vis[i] = (uint8_t)!occluded(s, ld3(x + 3 * i), ld3(y + 3 * i));
}

/* Sampled full-size checks: strata k0..k1-1 of the near part (same table as
 * oracle_generate_vpls builds; K = the final near count) and the raw
 * deposits of walks w0..w1-1 (flux not yet divided by the walk count). */
int64_t oracle_near_strata(const OScene* s, const uint8_t* labels, const OParams* p, int64_t K, int64_t k0, int64_t k1,
                           OVpl* out) {
    uint8_t* lit = (uint8_t*)malloc(s->n);
    int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (s->n + 1));
    uint64_t* P = (uint64_t*)malloc(sizeof(uint64_t) * (s->n + 1));
    oracle_lit(s, labels, lit);
    int64_t m = oracle_near_table(s, lit, order, P, NULL);
    if (m > 0 && K > 0) {
        float D = (float)((double)P[m - 1] / (double)K / 1099511627776.0);
#pragma omp parallel for schedule(dynamic, 8)
        for (int64_t k = k0; k < k1; k++) near_vpl(s, p, order, P, m, K, D, k, out + (k - k0));
    }
    free(lit); free(order); free(P);
    return m;
}

void oracle_walk_range(const OScene* s, const uint8_t* labels, const OParams* p, int64_t w0, int64_t w1, OVpl* dep,
                       int32_t* cnt) {
    int64_t md = p->max_depth > 0 ? p->max_depth : 1;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t w = w0; w < w1; w++) cnt[w - w0] = walk(s, p, labels, (uint32_t)w, dep + (w - w0) * md);
}

int oracle_abi(void) { return ORACLE_ABI; }
int oracle_variant(void) { return ORACLE_O0; }   /* 1: the frozen O0 build */
int oracle_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
