/* sdf.c — CPU ORACLE, NEXT-1: the paper's point-set SDF intersection.
 * TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * PAPER §II-B/§II-C, readings R40-R45 of DESIGN.md:
 *   R40 AABB primitives: the points are binned into cubic cells of edge a (the paper's
 *       voxel / (D_v D_sv), Table I: 0.5 m / (2 * 4)); a cell's AABB per axis is the extent of
 *       its points, or the cell's full extent on an axis where that extent exceeds a / 2.
 *   R41 SDF of an AABB at x: Eqs. 1-4 over the AABB's own points (the "points being evaluated",
 *       P:131), ascending id: w_i = E(-|p_i - x|^2 / (2 sigma^2)), sigma = xi r_s,
 *       pbar = sum w p / W, nbar = sum w n / W (Eq. 3 literally, not normalised),
 *       f = (x - pbar) . nbar; undefined ("fails") when W is not > 0.  FP32 throughout;
 *       E = the exp of sdf_expf below, written identically in the CUDA path (like R2's sincos).
 *       Summation order (the paper fixes none): the points in chunks of 32 consecutive ones
 *       (the last chunk padded with zero terms); each chunk summed by the pairwise tree that
 *       halves it in place (v[i] += v[i + s], s = 16, 8, 4, 2, 1); the chunk sums added in
 *       ascending chunk order (R41b).
 *   R42 march: for an AABB the ray enters (slab test, t_far >= 0), a segment of length
 *       L = a sqrt(3) (the AABB cell's diameter, l_d / (D_v D_sv)) centred on the projection of
 *       the AABB's centre on the ray; from its near end (clamped to t >= 0) march by |f| (r_s
 *       where f fails) until the far end; a hit where |f(s_i)| < t_sdf, or where
 *       sign f(s_i) != sign f(s_i+1): then at the linear zero between the two samples.
 *   R43 the segment's hit is the lexicographic min (t, cell index) over every AABB; departure:
 *       the cell of the previous hit is skipped, and so is every AABB whose SDF at the ray
 *       origin is defined with |f| <= tau and a unit normal within theta_ex of a departure
 *       normal (the R8 sheet rule with the SDF in place of the disk).
 *   R44 at a hit x*: the reflection normal is nbar(x*) / |nbar(x*)|; label and id of the
 *       coarse record are those of the AABB's point nearest to x* (lowest id on ties).
 * This is tier 0 for the SDF mode: every AABB of the scene is tested for every segment.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

typedef struct {      /* tier 1 (optional): a uniform grid over the AABBs, see or_sdf_grid_build */
    double org[3], v, pad;
    int64_t dims[3];
    int64_t* start;     /* [ncell + 1] CSR offsets */
    int64_t* aabb;      /* AABB indices registered per cell, ascending */
    int64_t* stamp;     /* [n_aabb] last query that tested the AABB */
    int64_t query;
} sdf_tgrid;

struct or_sdf {
    float org[3];       /* cell origin: the points' minimum */
    float a;            /* cell edge */
    int64_t dims[3];
    int64_t n_aabb;
    int64_t* cell;      /* [n_aabb] linear cell index, ascending */
    int64_t* start;     /* [n_aabb + 1] into ids */
    int64_t* ids;       /* point ids per AABB, ascending */
    float* lo;          /* [3 n_aabb] AABB bounds */
    float* hi;
    sdf_tgrid* tg;      /* tier 1 when set */
};

/* R41: exp(x) for x <= 0 in FP32, fixed operation order (Cody-Waite ln2 split + degree-7
 * Taylor polynomial in Horner form, every multiply-add a single-rounding fmaf, then 2^k by the
 * exponent bits); 0 below -87 (FP32 exp underflow). */
float or_sdf_expf(float x) {
    if (x < -87.0f) return 0.0f;
    float kf = floorf(fmaf(x, 1.44269504f, 0.5f));
    float r = fmaf(kf, -0.693359375f, x);
    r = fmaf(kf, 2.12194440e-4f, r);
    float p = 1.98412698e-4f;
    p = fmaf(p, r, 1.38888889e-3f);
    p = fmaf(p, r, 8.33333333e-3f);
    p = fmaf(p, r, 4.16666667e-2f);
    p = fmaf(p, r, 1.66666667e-1f);
    p = fmaf(p, r, 0.5f);
    p = fmaf(p, r, 1.0f);
    p = fmaf(p, r, 1.0f);
    int k = (int)kf;
    union {
        int i;
        float f;
    } s;
    s.i = (k + 127) << 23;
    return p * s.f;
}

static float dot3f(const float a[3], const float b[3]) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }

static int cmp_key(const void* A, const void* B) {
    const int64_t* a = (const int64_t*)A;
    const int64_t* b = (const int64_t*)B;
    if (a[0] != b[0]) return a[0] < b[0] ? -1 : 1;
    return a[1] < b[1] ? -1 : a[1] > b[1];
}

or_sdf* or_sdf_build(const or_scene* S, float a) {
    if (S->n <= 0 || !(a > 0.0f)) return NULL;
    or_sdf* G = (or_sdf*)calloc(1, sizeof(or_sdf));
    G->a = a;
    float mx[3];
    for (int k = 0; k < 3; ++k) G->org[k] = mx[k] = S->p[k];
    for (int64_t i = 0; i < S->n; ++i)
        for (int k = 0; k < 3; ++k) {
            if (S->p[3 * i + k] < G->org[k]) G->org[k] = S->p[3 * i + k];
            if (S->p[3 * i + k] > mx[k]) mx[k] = S->p[3 * i + k];
        }
    for (int k = 0; k < 3; ++k) G->dims[k] = (int64_t)floorf((mx[k] - G->org[k]) / a) + 1;
    /* (cell, id) pairs sorted: cells ascending, ids ascending within a cell */
    int64_t* kv = (int64_t*)malloc(sizeof(int64_t) * 2 * (size_t)S->n);
    for (int64_t i = 0; i < S->n; ++i) {
        int64_t c[3];
        for (int k = 0; k < 3; ++k) {
            c[k] = (int64_t)floorf((S->p[3 * i + k] - G->org[k]) / a);
            if (c[k] < 0) c[k] = 0;
            if (c[k] > G->dims[k] - 1) c[k] = G->dims[k] - 1;
        }
        kv[2 * i] = c[0] + G->dims[0] * (c[1] + G->dims[1] * c[2]);
        kv[2 * i + 1] = i;
    }
    qsort(kv, (size_t)S->n, 2 * sizeof(int64_t), cmp_key);
    int64_t na = 0;
    for (int64_t i = 0; i < S->n; ++i)
        if (i == 0 || kv[2 * i] != kv[2 * i - 2]) na++;
    G->n_aabb = na;
    G->cell = (int64_t*)malloc(sizeof(int64_t) * (size_t)na);
    G->start = (int64_t*)malloc(sizeof(int64_t) * (size_t)(na + 1));
    G->ids = (int64_t*)malloc(sizeof(int64_t) * (size_t)S->n);
    G->lo = (float*)malloc(sizeof(float) * 3 * (size_t)na);
    G->hi = (float*)malloc(sizeof(float) * 3 * (size_t)na);
    int64_t q = -1;
    for (int64_t i = 0; i < S->n; ++i) {
        if (i == 0 || kv[2 * i] != kv[2 * i - 2]) {
            ++q;
            G->cell[q] = kv[2 * i];
            G->start[q] = i;
        }
        G->ids[i] = kv[2 * i + 1];
    }
    G->start[na] = S->n;
    free(kv);
    /* R40: AABB = points' extent per axis, the cell's full extent where that exceeds a / 2 */
    for (int64_t j = 0; j < na; ++j) {
        int64_t c = G->cell[j];
        int64_t ci[3] = {c % G->dims[0], (c / G->dims[0]) % G->dims[1], c / (G->dims[0] * G->dims[1])};
        for (int k = 0; k < 3; ++k) {
            float lo = INFINITY, hi = -INFINITY;
            for (int64_t t = G->start[j]; t < G->start[j + 1]; ++t) {
                float v = S->p[3 * G->ids[t] + k];
                if (v < lo) lo = v;
                if (v > hi) hi = v;
            }
            if (hi - lo > 0.5f * a) {
                lo = G->org[k] + (float)ci[k] * a;
                hi = G->org[k] + (float)(ci[k] + 1) * a;
            }
            G->lo[3 * j + k] = lo;
            G->hi[3 * j + k] = hi;
        }
    }
    return G;
}

void or_sdf_free(or_sdf* G) {
    if (!G) return;
    if (G->tg) {
        free(G->tg->start);
        free(G->tg->aabb);
        free(G->tg->stamp);
        free(G->tg);
    }
    free(G->cell);
    free(G->start);
    free(G->ids);
    free(G->lo);
    free(G->hi);
    free(G);
}

int64_t or_sdf_count(const or_sdf* G) { return G ? G->n_aabb : 0; }

void or_sdf_aabb(const or_sdf* G, int64_t j, float lo[3], float hi[3], int64_t* cell, int64_t* n_pts) {
    for (int k = 0; k < 3; ++k) {
        lo[k] = G->lo[3 * j + k];
        hi[k] = G->hi[3 * j + k];
    }
    *cell = G->cell[j];
    *n_pts = G->start[j + 1] - G->start[j];
}

/* R41b: the pairwise tree sum of one chunk of 32 terms (halved in place) */
static float chunk_sum(float v[32]) {
    for (int s = 16; s >= 1; s >>= 1)
        for (int i = 0; i < s; ++i) v[i] = v[i] + v[i + s];
    return v[0];
}

/* R41: f of AABB j at x (and nbar, unnormalised); 0 where it fails */
int or_sdf_eval(const or_scene* S, const or_sdf* G, int64_t j, const float x[3], float sigma, float* f,
                float nbar[3]) {
    const float inv = 1.0f / (2.0f * sigma * sigma);
    /* sums[0] = W, sums[1..3] = sum w p, sums[4..6] = sum w n */
    float sums[7] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
    for (int64_t c0 = G->start[j]; c0 < G->start[j + 1]; c0 += 32) {
        float v[7][32];
        for (int i = 0; i < 32; ++i) {
            const int64_t t = c0 + i;
            for (int q = 0; q < 7; ++q) v[q][i] = 0.0f;
            if (t >= G->start[j + 1]) continue;  /* zero padding of the last chunk */
            const float* p = S->p + 3 * G->ids[t];
            const float* n = S->nrm + 3 * G->ids[t];
            float d[3] = {p[0] - x[0], p[1] - x[1], p[2] - x[2]};
            float q = fmaf(d[2], d[2], fmaf(d[1], d[1], d[0] * d[0]));  /* R41: |p - x|^2 */
            float w = or_sdf_expf(-(q * inv));
            v[0][i] = w;
            for (int k = 0; k < 3; ++k) {
                v[1 + k][i] = w * p[k];
                v[4 + k][i] = w * n[k];
            }
        }
        for (int q = 0; q < 7; ++q) sums[q] = sums[q] + chunk_sum(v[q]);
    }
    const float W = sums[0], P[3] = {sums[1], sums[2], sums[3]}, N[3] = {sums[4], sums[5], sums[6]};
    if (!(W > 0.0f)) return 0;
    float pb[3], e[3];
    for (int k = 0; k < 3; ++k) {
        pb[k] = P[k] / W;
        nbar[k] = N[k] / W;
        e[k] = x[0 + k] - pb[k];
    }
    *f = dot3f(e, nbar);
    return 1;
}

/* R42: march of AABB j along (o, d) from t >= 0; 1 and *t on a hit */
static int march(const or_scene* S, const or_sdf* G, int64_t j, const float o[3], const float d[3],
                 const or_sdf_params* Q, float* t_hit) {
    float c[3], tn = 0.0f, tf = INFINITY;
    for (int k = 0; k < 3; ++k) {
        const float lo = G->lo[3 * j + k], hi = G->hi[3 * j + k];
        c[k] = 0.5f * (lo + hi);
        if (d[k] != 0.0f) {
            float ta = (lo - o[k]) / d[k], tb = (hi - o[k]) / d[k];
            if (ta > tb) {
                float s = ta;
                ta = tb;
                tb = s;
            }
            if (ta > tn) tn = ta;
            if (tb < tf) tf = tb;
        } else if (o[k] < lo || o[k] > hi) {
            return 0;
        }
    }
    if (!(tn <= tf)) return 0;  /* the ray misses the AABB (or it lies behind the origin) */
    const float half = 0.5f * (Q->cell * 1.7320508f);
    float w[3] = {c[0] - o[0], c[1] - o[1], c[2] - o[2]};
    const float tc = dot3f(w, d);
    float t = tc - half;
    const float te = tc + half;
    if (t < 0.0f) t = 0.0f;
    const float sigma = Q->xi * Q->r_s;
    float x[3] = {o[0] + t * d[0], o[1] + t * d[1], o[2] + t * d[2]};
    float f0, nb[3];
    int ok0 = or_sdf_eval(S, G, j, x, sigma, &f0, nb);
    for (int it = 0; it < 4096; ++it) {
        if (ok0 && fabsf(f0) < Q->t_sdf) {
            *t_hit = t;
            return 1;
        }
        const float step = ok0 ? fabsf(f0) : Q->r_s;
        const float t1 = t + step;
        if (t1 > te) return 0;
        float x1[3] = {o[0] + t1 * d[0], o[1] + t1 * d[1], o[2] + t1 * d[2]};
        float f1;
        const int ok1 = or_sdf_eval(S, G, j, x1, sigma, &f1, nb);
        if (ok0 && ok1 && ((f0 < 0.0f) != (f1 < 0.0f))) {
            *t_hit = t + step * (f0 / (f0 - f1));
            return 1;
        }
        t = t1;
        f0 = f1;
        ok0 = ok1;
    }
    return 0;
}

/* R43 departure sheet: AABB j is transparent to a ray leaving o with departure normals lam */
static int excluded(const or_scene* S, const or_sdf* G, int64_t j, const float o[3], const float* lam,
                    int n_lam, const or_sdf_params* Q, float tau, float cos_ex) {
    if (n_lam == 0) return 0;
    float f, nb[3];
    if (!or_sdf_eval(S, G, j, o, Q->xi * Q->r_s, &f, nb)) return 0;
    if (!(fabsf(f) <= tau)) return 0;
    const float l = sqrtf(dot3f(nb, nb));
    if (!(l > 0.0f)) return 0;
    const float u[3] = {nb[0] / l, nb[1] / l, nb[2] / l};
    for (int k = 0; k < n_lam; ++k)
        if (fabsf(dot3f(u, lam + 3 * k)) >= cos_ex) return 1;
    return 0;
}

/* tier 1: the same argmin over the AABBs a FP64 walk of the tier-1 grid reaches.  AABB j is
 * registered in every cell its box inflated by pad overlaps; a march of j can only start once
 * the ray is in its box (slab test) and only at t >= tn - L (L = the march segment: its centre
 * projection lies within half a diagonal of the box), so once best_t < t_exit - pad - L no
 * untested AABB can win.  Candidates are compared lexicographically (t, index), so the visiting
 * order does not matter: the result is tier 0's. */
static int64_t nearest_t1(const or_scene* S, const or_sdf* G, const or_sdf_params* Q, const float o[3],
                          const float d[3], const float* lam, int n_lam, int64_t prev_cell, float tau,
                          float cos_ex, float* bt_out) {
    sdf_tgrid* T = G->tg;
    const int64_t qid = ++T->query;
    float bt = INFINITY;
    int64_t bj = -1;
    const double L = 2.0 * (double)(0.5f * (Q->cell * 1.7320508f));
    double od[3] = {o[0], o[1], o[2]}, dd[3] = {d[0], d[1], d[2]};
    double t0 = 0.0, t1 = INFINITY;
    for (int a = 0; a < 3; ++a) {
        double lo = T->org[a], hi = T->org[a] + (double)T->dims[a] * T->v;
        if (dd[a] != 0.0) {
            double ta = (lo - od[a]) / dd[a], tb = (hi - od[a]) / dd[a];
            t0 = fmax(t0, fmin(ta, tb));
            t1 = fmin(t1, fmax(ta, tb));
        } else if (od[a] < lo || od[a] > hi) {
            t1 = -1.0;
        }
    }
    if (t0 > t1) {
        *bt_out = bt;
        return -1;
    }
    int64_t c[3];
    double tm[3];
    for (int a = 0; a < 3; ++a) {
        double x = od[a] + t0 * dd[a];
        c[a] = (int64_t)floor((x - T->org[a]) / T->v);
        if (c[a] < 0) c[a] = 0;
        if (c[a] > T->dims[a] - 1) c[a] = T->dims[a] - 1;
        tm[a] = dd[a] != 0.0 ? (T->org[a] + (double)(c[a] + (dd[a] > 0.0)) * T->v - od[a]) / dd[a] : INFINITY;
    }
    for (;;) {
        const int64_t cell = c[0] + T->dims[0] * (c[1] + T->dims[1] * c[2]);
        for (int64_t k = T->start[cell]; k < T->start[cell + 1]; ++k) {
            const int64_t j = T->aabb[k];
            if (T->stamp[j] == qid) continue;
            T->stamp[j] = qid;
            if (G->cell[j] == prev_cell) continue;
            float t;
            if (!march(S, G, j, o, d, Q, &t)) continue;
            if (!(t < bt || (t == bt && j < bj))) continue;
            if (excluded(S, G, j, o, lam, n_lam, Q, tau, cos_ex)) continue;
            bt = t;
            bj = j;
        }
        int ax = 0;
        if (tm[1] < tm[ax]) ax = 1;
        if (tm[2] < tm[ax]) ax = 2;
        if ((double)bt < tm[ax] - T->pad - L) break;
        c[ax] += dd[ax] > 0.0 ? 1 : -1;
        if (c[ax] < 0 || c[ax] >= T->dims[ax]) break;
        tm[ax] = (T->org[ax] + (double)(c[ax] + (dd[ax] > 0.0)) * T->v - od[ax]) / dd[ax];
    }
    *bt_out = bt;
    return bj;
}

/* tier 1 for the SDF: register every AABB in the cells (edge voxel, origin = the AABB grid's
 * minus one voxel) its box inflated by 1e-4 m + 1e-6 x extent overlaps */
void or_sdf_grid_build(or_sdf* G, double voxel) {
    if (!G || G->n_aabb == 0) return;
    sdf_tgrid* T = (sdf_tgrid*)calloc(1, sizeof(sdf_tgrid));
    double lo[3], hi[3], ext = 0.0;
    for (int k = 0; k < 3; ++k) {
        lo[k] = INFINITY;
        hi[k] = -INFINITY;
    }
    for (int64_t j = 0; j < G->n_aabb; ++j)
        for (int k = 0; k < 3; ++k) {
            if (G->lo[3 * j + k] < lo[k]) lo[k] = G->lo[3 * j + k];
            if (G->hi[3 * j + k] > hi[k]) hi[k] = G->hi[3 * j + k];
        }
    for (int k = 0; k < 3; ++k) ext = fmax(ext, fmax(fabs(lo[k]), fabs(hi[k])));
    T->v = voxel;
    T->pad = 1e-4 + 1e-6 * ext;
    int64_t nc = 1;
    for (int k = 0; k < 3; ++k) {
        T->org[k] = lo[k] - voxel;
        T->dims[k] = (int64_t)ceil((hi[k] + voxel - T->org[k]) / voxel) + 1;
        nc *= T->dims[k];
    }
    int64_t* cnt = (int64_t*)calloc((size_t)nc + 1, sizeof(int64_t));
    for (int pass = 0; pass < 2; ++pass) {
        for (int64_t j = 0; j < G->n_aabb; ++j) {
            int64_t a0[3], a1[3];
            for (int k = 0; k < 3; ++k) {
                a0[k] = (int64_t)floor(((double)G->lo[3 * j + k] - T->pad - T->org[k]) / voxel);
                a1[k] = (int64_t)floor(((double)G->hi[3 * j + k] + T->pad - T->org[k]) / voxel);
                if (a0[k] < 0) a0[k] = 0;
                if (a1[k] > T->dims[k] - 1) a1[k] = T->dims[k] - 1;
            }
            for (int64_t z = a0[2]; z <= a1[2]; ++z)
                for (int64_t y = a0[1]; y <= a1[1]; ++y)
                    for (int64_t x = a0[0]; x <= a1[0]; ++x) {
                        const int64_t cell = x + T->dims[0] * (y + T->dims[1] * z);
                        if (pass == 0) cnt[cell + 1]++;
                        else T->aabb[T->start[cell] + cnt[cell]++] = j;
                    }
        }
        if (pass == 0) {
            T->start = (int64_t*)malloc(sizeof(int64_t) * ((size_t)nc + 1));
            T->start[0] = 0;
            for (int64_t c = 0; c < nc; ++c) T->start[c + 1] = T->start[c] + cnt[c + 1];
            T->aabb = (int64_t*)malloc(sizeof(int64_t) * (size_t)(T->start[nc] > 0 ? T->start[nc] : 1));
            memset(cnt, 0, sizeof(int64_t) * ((size_t)nc + 1));
        }
    }
    free(cnt);
    T->stamp = (int64_t*)calloc((size_t)G->n_aabb, sizeof(int64_t));
    G->tg = T;
}

/* R43-R44: the segment's nearest SDF hit over every AABB (tier 0; tier 1 when G->tg is set) */
int64_t or_sdf_nearest(const or_scene* S, const or_sdf* G, const or_sdf_params* Q, const float o[3],
                       const float d[3], const float* lam, int n_lam, int64_t prev_cell, float tau,
                       float cos_ex, float* t_out, int64_t* cell_out, float n_out[3]) {
    float bt = INFINITY;
    int64_t bj = -1;
    if (G->tg) {
        bj = nearest_t1(S, G, Q, o, d, lam, n_lam, prev_cell, tau, cos_ex, &bt);
    } else {
        for (int64_t j = 0; j < G->n_aabb; ++j) {
            if (G->cell[j] == prev_cell) continue;
            float t;
            if (!march(S, G, j, o, d, Q, &t)) continue;
            if (!(t < bt)) continue;  /* cells ascend: equal t keeps the lower cell */
            if (excluded(S, G, j, o, lam, n_lam, Q, tau, cos_ex)) continue;
            bt = t;
            bj = j;
        }
    }
    *t_out = bt;
    if (bj < 0) {
        *cell_out = -1;
        return -1;
    }
    *cell_out = G->cell[bj];
    float x[3] = {o[0] + bt * d[0], o[1] + bt * d[1], o[2] + bt * d[2]};
    float f, nb[3];
    n_out[0] = n_out[1] = n_out[2] = 0.0f;
    if (or_sdf_eval(S, G, bj, x, Q->xi * Q->r_s, &f, nb)) {
        const float l = sqrtf(dot3f(nb, nb));
        if (l > 0.0f)
            for (int k = 0; k < 3; ++k) n_out[k] = nb[k] / l;
    }
    /* the AABB's point nearest to the hit point: the record's label and id */
    int64_t best = -1;
    float bq = INFINITY;
    for (int64_t t = G->start[bj]; t < G->start[bj + 1]; ++t) {
        const float* p = S->p + 3 * G->ids[t];
        float e[3] = {p[0] - x[0], p[1] - x[1], p[2] - x[2]};
        float q = dot3f(e, e);
        if (q < bq) {
            bq = q;
            best = G->ids[t];
        }
    }
    return best;
}

/* ---- NEXT-4 helpers (gd.c) ------------------------------------------------------------ */
/* the AABB-grid cell of point id (R40 binning) */
int64_t or_sdf_cell_of(const or_scene* S, const or_sdf* G, int64_t id) {
    int64_t c[3];
    for (int k = 0; k < 3; ++k) {
        c[k] = (int64_t)floorf((S->p[3 * id + k] - G->org[k]) / G->a);
        if (c[k] < 0) c[k] = 0;
        if (c[k] > G->dims[k] - 1) c[k] = G->dims[k] - 1;
    }
    return c[0] + G->dims[0] * (c[1] + G->dims[1] * c[2]);
}

static int64_t aabb_of_cell(const or_sdf* G, int64_t cell) {
    int64_t lo = 0, hi = G->n_aabb - 1;
    while (lo <= hi) {
        int64_t mid = (lo + hi) / 2;
        if (G->cell[mid] == cell) return mid;
        if (G->cell[mid] < cell) lo = mid + 1;
        else hi = mid - 1;
    }
    return -1;
}

/* R53: the unit normal of Eq. 3 at x over the points of the AABBs in the 3x3x3 cells around
 * `cell` ("additionally evaluating the points in the neighboring AABB primitives").
 * Rows (dz, dy) ascending; a row = the points of its cells x-1..x+1 in (cell, id) order; each
 * row summed in chunks of 32 by the R41b tree, rows and chunks added in order.  0 if W <= 0. */
int or_sdf_normal27(const or_scene* S, const or_sdf* G, int64_t cell, const float x[3], float sigma,
                    float n_out[3]) {
    const float inv = 1.0f / (2.0f * sigma * sigma);
    const int64_t cx = cell % G->dims[0], cy = (cell / G->dims[0]) % G->dims[1],
                  cz = cell / (G->dims[0] * G->dims[1]);
    float sums[4] = {0.0f, 0.0f, 0.0f, 0.0f}; /* W, N */
    for (int64_t dz = -1; dz <= 1; ++dz)
        for (int64_t dy = -1; dy <= 1; ++dy) {
            const int64_t y = cy + dy, z = cz + dz;
            if (y < 0 || y >= G->dims[1] || z < 0 || z >= G->dims[2]) continue;
            /* the row's point list: cells x-1..x+1 (inside the grid), ascending; the AABBs of
             * consecutive cells are consecutive, so the list is ids[first .. last) */
            int64_t first = -1, last = -1;
            for (int64_t dx = -1; dx <= 1; ++dx) {
                const int64_t xx = cx + dx;
                if (xx < 0 || xx >= G->dims[0]) continue;
                const int64_t j = aabb_of_cell(G, xx + G->dims[0] * (y + G->dims[1] * z));
                if (j < 0) continue;
                if (first < 0) first = G->start[j];
                last = G->start[j + 1];
            }
            if (first < 0) continue;
            const int64_t* ids = G->ids + first;
            const int64_t m = last - first;
            for (int64_t c0 = 0; c0 < m; c0 += 32) {
                float v[4][32];
                for (int i = 0; i < 32; ++i) {
                    for (int q = 0; q < 4; ++q) v[q][i] = 0.0f;
                    if (c0 + i >= m) continue;
                    const float* p = S->p + 3 * ids[c0 + i];
                    const float* nn = S->nrm + 3 * ids[c0 + i];
                    float d[3] = {p[0] - x[0], p[1] - x[1], p[2] - x[2]};
                    float q = fmaf(d[2], d[2], fmaf(d[1], d[1], d[0] * d[0]));
                    float w = or_sdf_expf(-(q * inv));
                    v[0][i] = w;
                    for (int k = 0; k < 3; ++k) v[1 + k][i] = w * nn[k];
                }
                for (int q = 0; q < 4; ++q) sums[q] = sums[q] + chunk_sum(v[q]);
            }
        }
    if (!(sums[0] > 0.0f)) return 0;
    float nb[3] = {sums[1] / sums[0], sums[2] / sums[0], sums[3] / sums[0]};
    const float l = sqrtf(dot3f(nb, nb));
    if (!(l > 0.0f)) return 0;
    for (int k = 0; k < 3; ++k) n_out[k] = nb[k] / l;
    return 1;
}

/* NEXT-2 helper (env.c): the AABB grid's geometry */
void or_sdf_geometry(const or_sdf* G, float org[3], float* a, int64_t dims[3]) {
    for (int k = 0; k < 3; ++k) {
        org[k] = G->org[k];
        dims[k] = G->dims[k];
    }
    *a = G->a;
}
