/* coarse.c — CPU ORACLE, coarse path tracing.  TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Plain, slow, single-threaded definition of the north_star coarse path:
 * every segment's hit is the brute-force global argmin over all surfels (no grid).
 * FP32 throughout the traced geometry, fixed operation order (R3), compiled without
 * FMA contraction.  Transcendentals only through or_sincos (R2), in FP64.
 *
 * Citations: P:n = /root/reference/PAPER.md line n; R<k> = DESIGN.md reading k.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------ */
/* R2: FP64 sincos — pi/2 Cody-Waite reduction (2 parts) + fdlibm kernel polynomials.     */
/* Evaluated in a fixed order, no FMA; used for ray generation (A2) and fan angles (A7). */
/* ------------------------------------------------------------------------------------ */
static const double OR_PIO2_1 = 1.57079632673412561417e+00;  /* first 33 bits of pi/2 */
static const double OR_PIO2_1T = 6.07710050650619224932e-11; /* pi/2 - PIO2_1 */
static const double OR_INVPIO2 = 6.36619772367581382433e-01; /* 2/pi */
static const double OR_PI = 3.14159265358979311600e+00;

static double or_ksin(double x) {
    const double S1 = -1.66666666666666324348e-01, S2 = 8.33333333332248946124e-03,
                 S3 = -1.98412698298579493134e-04, S4 = 2.75573137070700676789e-06,
                 S5 = -2.50507602534068634195e-08, S6 = 1.58969099521155010221e-10;
    double z = x * x;
    double v = z * x;
    double r = S2 + z * (S3 + z * (S4 + z * (S5 + z * S6)));
    return x + v * (S1 + z * r);
}

static double or_kcos(double x) {
    const double C1 = 4.16666666666666019037e-02, C2 = -1.38888888888741095749e-03,
                 C3 = 2.48015872894767294178e-05, C4 = -2.75573143513906633035e-07,
                 C5 = 2.08757232129817482790e-09, C6 = -1.13596475577881948265e-11;
    double z = x * x;
    double r = z * (C1 + z * (C2 + z * (C3 + z * (C4 + z * (C5 + z * C6)))));
    return 1.0 - (0.5 * z - z * r);
}

void or_sincos(double x, double* s, double* c) {
    double kf = floor(x * OR_INVPIO2 + 0.5);
    double y = (x - kf * OR_PIO2_1) - kf * OR_PIO2_1T;
    long k = (long)kf;
    double sy = or_ksin(y), cy = or_kcos(y);
    switch (k & 3) {
        case 0: *s = sy; *c = cy; break;
        case 1: *s = cy; *c = -sy; break;
        case 2: *s = -sy; *c = -cy; break;
        default: *s = -cy; *c = sy; break;
    }
}

/* R1 / A2: spherical Fibonacci direction of lattice index i out of n (P:146 uniform
 * launching; BJ "rays from the TX over a Fibonacci sphere"). */
void or_fib_dir(uint64_t i, uint64_t n, float d[3]) {
    const double g = 0.3819660112501051; /* (3 - sqrt 5) / 2 */
    double z = 1.0 - (2.0 * (double)i + 1.0) / (double)n;
    double x = (double)i * g;
    double fr = x - floor(x);
    double phi = (2.0 * OR_PI) * fr;
    double s, c;
    or_sincos(phi, &s, &c);
    double rr = sqrt(1.0 - z * z);
    d[0] = (float)(rr * c);
    d[1] = (float)(rr * s);
    d[2] = (float)z;
}

float or_cos_ex(float theta_ex_deg) {
    double s, c;
    or_sincos((double)theta_ex_deg * (OR_PI / 180.0), &s, &c);
    return (float)c;
}

/* R12: c_R * omega, omega = sqrt(4 pi / N) */
float or_cRw(float c_R, int64_t n_rays) {
    return (float)((double)c_R * sqrt(4.0 * OR_PI / (double)n_rays));
}

/* R3: dot = (x*x' + y*y') + z*z' */
static float dot3(const float a[3], const float b[3]) {
    return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
}

/* R7-R8: HIT predicate of one surfel, disk (p, n, r). */
static inline int hit_impl(const float o[3], const float d[3], const float p[3], const float n[3],
                           float r, const float* lam, int n_lam, float tau, float cos_ex, float* t) {
    float w[3] = {o[0] - p[0], o[1] - p[1], o[2] - p[2]};
    float f0 = dot3(w, n);
    float dn = dot3(d, n);
    if (!(f0 * dn < 0.0f)) return 0;         /* origin must approach the surfel plane */
    if (fabsf(f0) <= tau) {                   /* departure-sheet exclusion (R8) */
        for (int k = 0; k < n_lam; ++k) {
            float c = dot3(n, lam + 3 * k);
            if (fabsf(c) >= cos_ex) return 0;
        }
    }
    float tt = (-f0) / dn;
    float h[3] = {o[0] + tt * d[0], o[1] + tt * d[1], o[2] + tt * d[2]};
    float q[3] = {h[0] - p[0], h[1] - p[1], h[2] - p[2]};
    float qq = dot3(q, q);
    float r2 = r * r;
    if (!(qq <= r2)) return 0;
    *t = tt;
    return 1;
}

int or_hit(const float o[3], const float d[3], const float p[3], const float n[3], float r,
           const float* lam, int n_lam, float tau, float cos_ex, float* t) {
    return hit_impl(o, d, p, n, r, lam, n_lam, tau, cos_ex, t);
}

/* A4: d' = d - (2 (d.n)) n, then d' / sqrt(d'.d') */
void or_reflect(const float d[3], const float n[3], float out[3]) {
    float k = 2.0f * dot3(d, n);
    float x[3] = {d[0] - k * n[0], d[1] - k * n[1], d[2] - k * n[2]};
    float l = sqrtf(dot3(x, x));
    out[0] = x[0] / l;
    out[1] = x[1] / l;
    out[2] = x[2] / l;
}

/* C.1 step 2(a): global lexicographic argmin over all surfels of (t, id) (R9).  Tier 0 is
 * this loop; with S->grid set the tier-1 grid (grid.c) computes the same minimum. */
int64_t or_nearest(const or_scene* S, const float o[3], const float d[3], const float* lam,
                   int n_lam, int64_t prev, float tau, float cos_ex, float* t_hit) {
    if (S->grid) return or_grid_nearest(S, S->grid, o, d, lam, n_lam, prev, tau, cos_ex, t_hit);
    int64_t best = -1;
    float bt = INFINITY;
    for (int64_t i = 0; i < S->n; ++i) {
        if (i == prev) continue;
        float t;
        if (!hit_impl(o, d, S->p + 3 * i, S->nrm + 3 * i, S->r[i], lam, n_lam, tau, cos_ex, &t))
            continue;
        if (t < bt) { /* ids ascend, so equal t keeps the lower id */
            bt = t;
            best = i;
        }
    }
    *t_hit = bt;
    return best;
}

/* ------------------------------------------------------------------------------------ */
/* ray state, records and events                                                        */
/* ------------------------------------------------------------------------------------ */
typedef or_hist hist_t;
typedef or_event event_t;

typedef struct {
    or_coarse* raw;
    int64_t cap, n;
    event_t* ev;
    int64_t ev_cap, n_ev;
    uint64_t bounces;
    int64_t* hit_ids; /* optional per-segment hits of the current ray */
} sink_t;

static void emit_record(sink_t* K, const hist_t* h, uint32_t rx, float L, uint64_t ray_id) {
    if (K->n < K->cap) {
        or_coarse* c = &K->raw[K->n];
        memset(c, 0, sizeof(*c));
        c->rx = rx;
        c->n_int = (uint8_t)h->n;
        c->n_diff = (uint8_t)h->n_diff;
        c->kinds = h->kinds;
        for (int k = 0; k < h->n; ++k) {
            c->label[k] = h->label[k];
            c->prim[k] = h->prim[k];
            c->v[k][0] = h->v[k][0];
            c->v[k][1] = h->v[k][1];
            c->v[k][2] = h->v[k][2];
        }
        c->s_edge = h->s_edge;
        c->L = L;
        c->ray_id = ray_id;
    }
    K->n++;
}

typedef struct {
    float e[3];
    float len;
} edge_geo_t;

/* per-edge unit direction and length: ev = b - a, len = sqrt(ev.ev), e = ev / len */
static void edge_geo(const or_edge* E, edge_geo_t* g) {
    float ev[3] = {E->b[0] - E->a[0], E->b[1] - E->a[1], E->b[2] - E->a[2]};
    g->len = sqrtf(dot3(ev, ev));
    g->e[0] = ev[0] / g->len;
    g->e[1] = ev[1] / g->len;
    g->e[2] = ev[2] / g->len;
}

typedef struct {
    const or_scene* S;
    const or_launch_params* P;
    float cos_ex;
    float cRw;
    float b_e;        /* edge occlusion bias r_max + tau (R13) */
    edge_geo_t* eg;
} ctx_t;

/* RX captures of one segment (R12).  R(s) = kR * s + R0 where s is the capture distance
 * argument: for primary rays s = L + t_j, kR = c_R*omega, R0 = 0; after a diffraction
 * s = s' + t_j (distance since the edge), kR = c_R*(n pi/M)|sin theta|, R0 = edge_bin/2. */
static void rx_captures(const ctx_t* C, sink_t* K, const hist_t* h, const float o[3],
                        const float d[3], float t_hit, float L, float Ls, float kR, float R0,
                        int after_diff, uint64_t ray_id) {
    const or_launch_params* P = C->P;
    for (int j = 0; j < P->n_rx; ++j) {
        const float* x = P->rx + 3 * j;
        float w[3] = {x[0] - o[0], x[1] - o[1], x[2] - o[2]};
        float tj = dot3(w, d);
        if (!(tj > 0.0f && tj < t_hit)) continue;
        float pr[3] = {w[0] - tj * d[0], w[1] - tj * d[1], w[2] - tj * d[2]};
        float pp = dot3(pr, pr);
        float R;
        if (after_diff) R = kR * (Ls + tj) + R0;
        else R = kR * (L + tj);
        if (!(pp <= R * R)) continue;
        emit_record(K, h, (uint32_t)j, L + tj, ray_id);
    }
}

/* R13: edge captures of one segment -> diffraction events */
static void edge_captures(const ctx_t* C, sink_t* K, const hist_t* h, const float o[3],
                          const float d[3], float t_hit, float L, uint64_t ray_id) {
    const or_scene* S = C->S;
    for (int j = 0; j < S->n_edges; ++j) {
        const or_edge* E = &S->edges[j];
        const edge_geo_t* g = &C->eg[j];
        float b = dot3(d, g->e);
        float w0[3] = {o[0] - E->a[0], o[1] - E->a[1], o[2] - E->a[2]};
        float den = 1.0f - b * b;
        if (!(den > 1e-12f)) continue;
        float de = dot3(g->e, w0);
        float dd = dot3(d, w0);
        float te = (b * de - dd) / den;
        float s = (de - b * dd) / den;
        if (!(s >= 0.0f && s <= g->len)) continue;
        if (!(te > 0.0f && te < t_hit + C->b_e)) continue;
        float pc[3] = {o[0] + te * d[0], o[1] + te * d[1], o[2] + te * d[2]};
        float pe[3] = {E->a[0] + s * g->e[0], E->a[1] + s * g->e[1], E->a[2] + s * g->e[2]};
        float dv[3] = {pc[0] - pe[0], pc[1] - pe[1], pc[2] - pe[2]};
        float dist2 = dot3(dv, dv);
        float R = C->cRw * (L + te);
        if (!(dist2 <= R * R)) continue;
        if (K->n_ev < K->ev_cap) {
            event_t* ev = &K->ev[K->n_ev];
            memset(ev, 0, sizeof(*ev));
            ev->h = *h;
            ev->edge = (uint32_t)j;
            ev->s = s;
            ev->sbin = (int32_t)floorf(s / C->P->edge_bin);
            ev->d[0] = d[0];
            ev->d[1] = d[1];
            ev->d[2] = d[2];
            ev->L = L + te;
            ev->dist2 = dist2;
            ev->ray_id = ray_id;
        }
        K->n_ev++;
    }
}

/* C.1 step 2: trace one ray (primary or fan) */
static void trace(const ctx_t* C, sink_t* K, hist_t h, const float o0[3], const float d0[3],
                  float L0, int refl_budget, int allow_edges, const float* lam0, int n_lam0,
                  int after_diff, float kR, float R0, uint64_t ray_id) {
    const or_launch_params* P = C->P;
    const or_scene* S = C->S;
    float o[3] = {o0[0], o0[1], o0[2]};
    float d[3] = {d0[0], d0[1], d0[2]};
    float lam[6];
    int n_lam = n_lam0;
    for (int k = 0; k < 3 * n_lam0; ++k) lam[k] = lam0[k];
    float L = L0, Ls = 0.0f;
    int64_t prev = -1;
    const int sdf = P->sdf.cell > 0.0f && S->sdf;  /* NEXT-1: point-set SDF intersection */
    for (int seg = 0; seg <= refl_budget; ++seg) {
        float th, nsdf[3] = {0.0f, 0.0f, 0.0f};
        int64_t cell = -1;
        int64_t s = sdf ? or_sdf_nearest(S, S->sdf, &P->sdf, o, d, lam, n_lam, prev, P->tau, C->cos_ex,
                                         &th, &cell, nsdf)
                        : or_nearest(S, o, d, lam, n_lam, prev, P->tau, C->cos_ex, &th);
        K->bounces++;
        if (K->hit_ids) K->hit_ids[seg] = s;
        rx_captures(C, K, &h, o, d, th, L, Ls, kR, R0, after_diff, ray_id);
        if (allow_edges && h.n_diff < P->max_diff && h.n < OR_MAX_INT)
            edge_captures(C, K, &h, o, d, th, L, ray_id);
        if (s < 0 || seg == refl_budget) break;
        /* A4: reflect at the hit surfel (SDF mode: at the SDF hit, its MLS normal, R44) */
        float hp[3] = {o[0] + th * d[0], o[1] + th * d[1], o[2] + th * d[2]};
        const float* n = sdf ? nsdf : S->nrm + 3 * s;
        h.label[h.n] = S->label[s];
        h.prim[h.n] = (uint32_t)s;
        h.v[h.n][0] = hp[0];
        h.v[h.n][1] = hp[1];
        h.v[h.n][2] = hp[2];
        h.n++;
        float dr[3];
        or_reflect(d, n, dr);
        d[0] = dr[0];
        d[1] = dr[1];
        d[2] = dr[2];
        o[0] = hp[0];
        o[1] = hp[1];
        o[2] = hp[2];
        L = L + th;
        Ls = Ls + th;
        lam[0] = n[0];
        lam[1] = n[1];
        lam[2] = n[2];
        n_lam = 1;
        prev = sdf ? cell : s;
    }
}

/* ---- R17 record order: (rx, n_int, kinds, label[0..7]) then L then ray id ---- */
static int key_cmp(const or_coarse* a, const or_coarse* b) {
    if (a->rx != b->rx) return a->rx < b->rx ? -1 : 1;
    if (a->n_int != b->n_int) return a->n_int < b->n_int ? -1 : 1;
    if (a->kinds != b->kinds) return a->kinds < b->kinds ? -1 : 1;
    for (int k = 0; k < OR_MAX_INT; ++k)
        if (a->label[k] != b->label[k]) return a->label[k] < b->label[k] ? -1 : 1;
    return 0;
}

static int rec_cmp(const void* pa, const void* pb) {
    const or_coarse* a = (const or_coarse*)pa;
    const or_coarse* b = (const or_coarse*)pb;
    int c = key_cmp(a, b);
    if (c) return c;
    if (a->L != b->L) return a->L < b->L ? -1 : 1;
    if (a->ray_id != b->ray_id) return a->ray_id < b->ray_id ? -1 : 1;
    return 0;
}

int64_t or_dedupe(or_coarse* recs, int64_t n, int32_t kappa) {
    if (n <= 0) return 0;
    qsort(recs, (size_t)n, sizeof(or_coarse), rec_cmp);
    int64_t m = 0, run = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (i > 0 && key_cmp(&recs[i], &recs[i - 1]) == 0) run++;
        else run = 0;
        if (run < kappa) recs[m++] = recs[i];
    }
    return m;
}

/* ---- R14 event order: (history key, edge, sbin) then dist2 then ray id ---- */
static int ev_key_cmp(const event_t* a, const event_t* b) {
    if (a->h.n != b->h.n) return a->h.n < b->h.n ? -1 : 1;
    if (a->h.kinds != b->h.kinds) return a->h.kinds < b->h.kinds ? -1 : 1;
    for (int k = 0; k < OR_MAX_INT; ++k) {
        int32_t la = k < a->h.n ? a->h.label[k] : 0, lb = k < b->h.n ? b->h.label[k] : 0;
        if (la != lb) return la < lb ? -1 : 1;
    }
    if (a->edge != b->edge) return a->edge < b->edge ? -1 : 1;
    if (a->sbin != b->sbin) return a->sbin < b->sbin ? -1 : 1;
    return 0;
}

static int ev_cmp(const void* pa, const void* pb) {
    const event_t* a = (const event_t*)pa;
    const event_t* b = (const event_t*)pb;
    int c = ev_key_cmp(a, b);
    if (c) return c;
    if (a->dist2 != b->dist2) return a->dist2 < b->dist2 ? -1 : 1;
    if (a->ray_id != b->ray_id) return a->ray_id < b->ray_id ? -1 : 1;
    return 0;
}

static void ctx_init(ctx_t* C, const or_scene* S, const or_launch_params* P) {
    C->S = S;
    C->P = P;
    C->cos_ex = or_cos_ex(P->theta_ex_deg);
    C->cRw = or_cRw(P->c_R, P->n_rays);
    float rmax = 0.0f;
    for (int64_t i = 0; i < S->n; ++i)
        if (S->r[i] > rmax) rmax = S->r[i];
    C->b_e = rmax + P->tau;
    C->eg = (edge_geo_t*)calloc((size_t)(S->n_edges > 0 ? S->n_edges : 1), sizeof(edge_geo_t));
    for (int j = 0; j < S->n_edges; ++j) edge_geo(&S->edges[j], &C->eg[j]);
}

/* R15-R16: Keller fan of one (deduped) event; rank = its position in event-key order */
static void fan(const ctx_t* C, sink_t* K, const event_t* ev, uint64_t rank) {
    const or_launch_params* P = C->P;
    const or_edge* E = &C->S->edges[ev->edge];
    const edge_geo_t* g = &C->eg[ev->edge];
    double ct = (double)dot3(ev->d, g->e);
    double st = sqrt(fmax(0.0, 1.0 - ct * ct));
    if (st < 1e-6) return;
    int M0 = (int)ceil((double)E->n_exp * 180.0 / (double)P->dphi_deg);
    int M = (int)ceil((double)M0 * st);
    if (M < 1) M = 1;
    double wedge = (double)E->n_exp * OR_PI;
    float kR = (float)((double)P->c_R * (wedge / (double)M) * st);
    float R0 = 0.5f * P->edge_bin;
    float o[3] = {E->a[0] + ev->s * g->e[0], E->a[1] + ev->s * g->e[1], E->a[2] + ev->s * g->e[2]};
    hist_t h = ev->h;
    h.label[h.n] = E->label;
    h.prim[h.n] = ev->edge;
    h.v[h.n][0] = o[0];
    h.v[h.n][1] = o[1];
    h.v[h.n][2] = o[2];
    h.kinds = (uint16_t)(h.kinds | (1u << h.n));
    h.n++;
    h.n_diff++;
    h.s_edge = ev->s;
    int n_refl = 0;
    for (int k = 0; k < ev->h.n; ++k)
        if (!((ev->h.kinds >> k) & 1u)) n_refl++;
    int budget = P->max_refl - n_refl;
    if (budget < 0) return;
    if (h.n + budget > OR_MAX_INT) budget = OR_MAX_INT - h.n;
    float lam[6] = {E->n0[0], E->n0[1], E->n0[2], E->n1[0], E->n1[1], E->n1[2]};
    for (int m = 0; m < M; ++m) {
        double phi = (((double)m + 0.5) * wedge) / (double)M;
        double sp, cp;
        or_sincos(phi, &sp, &cp);
        float dir[3];
        for (int k = 0; k < 3; ++k) {
            double x2 = cp * (double)E->t0[k] + sp * (double)E->n0[k];
            dir[k] = (float)(x2 * st + (double)g->e[k] * ct);
        }
        uint64_t rid = (1ull << 63) | (rank << 8) | (uint64_t)m;
        trace(C, K, h, o, dir, ev->L, budget, 0, lam, 2, 1, kR, R0, rid);
    }
}

static void free_ctx(ctx_t* C) { free(C->eg); }

int or_trace_primary(const or_scene* S, const or_launch_params* P, or_coarse* raw,
                     int64_t raw_cap, int64_t* n_raw, or_event* ev, int64_t ev_cap,
                     int64_t* n_ev, uint64_t* n_bounces) {
    ctx_t C;
    ctx_init(&C, S, P);
    sink_t K;
    memset(&K, 0, sizeof(K));
    K.raw = raw;
    K.cap = raw_cap;
    K.ev = ev;
    K.ev_cap = ev_cap;
    hist_t h0;
    memset(&h0, 0, sizeof(h0));
    int edges_on = S->n_edges > 0 && P->max_diff > 0;
    for (uint64_t i = (uint64_t)P->rank; i < (uint64_t)P->n_rays; i += (uint64_t)P->world) {
        float d[3];
        or_fib_dir(i, (uint64_t)P->n_rays, d);
        trace(&C, &K, h0, P->tx, d, 0.0f, P->max_refl, edges_on, NULL, 0, 0, C.cRw, 0.0f, i);
    }
    free_ctx(&C);
    *n_raw = K.n;
    *n_ev = K.n_ev;
    *n_bounces = K.bounces;
    return (K.n > raw_cap || K.n_ev > ev_cap) ? 4 : 0;
}

int64_t or_event_dedupe(or_event* ev, int64_t n) {
    if (n <= 0) return 0;
    qsort(ev, (size_t)n, sizeof(event_t), ev_cmp);
    int64_t m = 0;
    for (int64_t i = 0; i < n; ++i)
        if (i == 0 || ev_key_cmp(&ev[i], &ev[i - 1]) != 0) ev[m++] = ev[i];
    return m;
}

int or_trace_fans(const or_scene* S, const or_launch_params* P, const or_event* ev, int64_t n_ev,
                  int32_t part, int32_t parts, or_coarse* raw, int64_t raw_cap, int64_t* n_raw,
                  uint64_t* n_bounces) {
    ctx_t C;
    ctx_init(&C, S, P);
    sink_t K;
    memset(&K, 0, sizeof(K));
    K.raw = raw;
    K.cap = raw_cap;
    for (int64_t r = part; r < n_ev; r += parts) fan(&C, &K, &ev[r], (uint64_t)r);
    free_ctx(&C);
    *n_raw = K.n;
    *n_bounces = K.bounces;
    return K.n > raw_cap ? 4 : 0;
}

int or_launch(const or_scene* S, const or_launch_params* P0, or_coarse* raw, int64_t raw_cap,
              int64_t* n_raw, or_coarse* out, int64_t out_cap, int64_t* n_out,
              uint64_t* n_bounces) {
    /* the oracle computes the GLOBAL set: every lattice index, whatever rank/world say */
    or_launch_params P = *P0;
    P.rank = 0;
    P.world = 1;
    int64_t ev_cap = 1 << 16, nr = 0, ne = 0, nf = 0;
    uint64_t b1 = 0, b2 = 0;
    or_event* ev = NULL;
    for (;;) {
        ev = (or_event*)malloc(sizeof(or_event) * (size_t)ev_cap);
        or_trace_primary(S, &P, raw, raw_cap, &nr, ev, ev_cap, &ne, &b1);
        if (ne <= ev_cap) break;
        free(ev);
        ev_cap = ne;
    }
    ne = or_event_dedupe(ev, ne);
    int64_t cap2 = raw_cap > nr ? raw_cap - nr : 0;
    or_trace_fans(S, &P, ev, ne, 0, 1, raw + (nr < raw_cap ? nr : raw_cap), cap2, &nf, &b2);
    free(ev);
    *n_raw = nr + nf;
    *n_bounces = b1 + b2;
    if (nr + nf > raw_cap) {
        *n_out = 0;
        return 4;
    }
    int64_t m = or_dedupe(raw, nr + nf, P.kappa);
    *n_out = m;
    if (m > out_cap) return 4;
    memcpy(out, raw, sizeof(or_coarse) * (size_t)m);
    return 0;
}

int or_trace_rays(const or_scene* S, const or_launch_params* P, const uint64_t* ray_ids,
                  int64_t n, or_coarse* raw, int64_t raw_cap, int64_t* n_raw, int64_t* hit_ids,
                  uint64_t* n_bounces) {
    ctx_t C;
    ctx_init(&C, S, P);
    sink_t K;
    memset(&K, 0, sizeof(K));
    K.raw = raw;
    K.cap = raw_cap;
    hist_t h0;
    memset(&h0, 0, sizeof(h0));
    int nseg = P->max_refl + 1;
    for (int64_t q = 0; q < n; ++q) {
        float d[3];
        or_fib_dir(ray_ids[q], (uint64_t)P->n_rays, d);
        if (hit_ids) {
            for (int k = 0; k < nseg; ++k) hit_ids[q * nseg + k] = -2;
            K.hit_ids = hit_ids + q * nseg;
        }
        trace(&C, &K, h0, P->tx, d, 0.0f, P->max_refl, 0, NULL, 0, 0, C.cRw, 0.0f, ray_ids[q]);
    }
    free(C.eg);
    *n_raw = K.n;
    *n_bounces = K.bounces;
    return K.n > raw_cap ? 4 : 0;
}

/* ---- pin helpers (same arithmetic as edge_captures / fan, exposed for tests) ---- */
int or_edge_closest(const float o[3], const float d[3], const or_edge* E, float* te, float* s,
                    float* dist2) {
    edge_geo_t g;
    edge_geo(E, &g);
    float b = dot3(d, g.e);
    float w0[3] = {o[0] - E->a[0], o[1] - E->a[1], o[2] - E->a[2]};
    float den = 1.0f - b * b;
    if (!(den > 1e-12f)) return 0;
    float de = dot3(g.e, w0);
    float dd = dot3(d, w0);
    *te = (b * de - dd) / den;
    *s = (de - b * dd) / den;
    float pc[3] = {o[0] + *te * d[0], o[1] + *te * d[1], o[2] + *te * d[2]};
    float pe[3] = {E->a[0] + *s * g.e[0], E->a[1] + *s * g.e[1], E->a[2] + *s * g.e[2]};
    float dv[3] = {pc[0] - pe[0], pc[1] - pe[1], pc[2] - pe[2]};
    *dist2 = dot3(dv, dv);
    return 1;
}

int or_fan_dirs(const or_edge* E, const float d[3], float dphi_deg, float* out, int cap) {
    edge_geo_t g;
    edge_geo(E, &g);
    double ct = (double)dot3(d, g.e);
    double st = sqrt(fmax(0.0, 1.0 - ct * ct));
    if (st < 1e-6) return 0;
    int M0 = (int)ceil((double)E->n_exp * 180.0 / (double)dphi_deg);
    int M = (int)ceil((double)M0 * st);
    if (M < 1) M = 1;
    double wedge = (double)E->n_exp * OR_PI;
    for (int m = 0; m < M && m < cap; ++m) {
        double phi = (((double)m + 0.5) * wedge) / (double)M;
        double sp, cp;
        or_sincos(phi, &sp, &cp);
        for (int k = 0; k < 3; ++k) {
            double x2 = cp * (double)E->t0[k] + sp * (double)E->n0[k];
            out[3 * m + k] = (float)(x2 * st + (double)g.e[k] * ct);
        }
    }
    return M;
}
