/* post.c — CPU ORACLE, refined-path post-processing (§II-E,
 * P:234-242).  TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
 * CPU legs may call it; it shares no code with the CUDA library.
 *
 * FP64, single-threaded, plain, in the paper's order (readings R33-R36):
 *   1. exact label ("the label of the closest point to the intersection point"): every
 *      reflection vertex x takes the label of the surfel i minimising |p_i - x| (lowest id on
 *      ties) among all surfels with |p_i - x| <= 2 r_s; none -> the coarse label stays (R33);
 *   2. shortest path per (rx, interaction chain, labels) (R28 with the exact labels);
 *   3. order by propagation delay ("sorted based on propagation time delay"), ties in
 *      key order (R35);
 *   4. greedy first-Fresnel-zone dedupe (Eq. 13): walking that order, a path is a
 *      duplicate of an already accepted path with the same rx and interaction chain when every
 *      one of its interaction points lies within the accepted path's first Fresnel radius
 *      psi_k = sqrt(lambda s1 s2 / (s1 + s2)) at that interaction (s1, s2 = the accepted
 *      path's distances to its neighbouring points) AND the angle between every pair of k-th
 *      rays is below the threshold (R36).  Only non-duplicates are kept.
 * Only status-OK records take part.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

static double dot3(const double a[3], const double b[3]) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }

static int key_cmp(const or_refined* a, const or_refined* b) {
    if (a->rx != b->rx) return a->rx < b->rx ? -1 : 1;
    if (a->n_int != b->n_int) return a->n_int < b->n_int ? -1 : 1;
    if (a->kinds != b->kinds) return a->kinds < b->kinds ? -1 : 1;
    for (int k = 0; k < OR_MAX_INT; ++k)
        if (a->label[k] != b->label[k]) return a->label[k] < b->label[k] ? -1 : 1;
    return 0;
}

static int shortest_cmp(const void* pa, const void* pb) { /* (key, L, ray id) */
    const or_refined *a = (const or_refined*)pa, *b = (const or_refined*)pb;
    int c = key_cmp(a, b);
    if (c) return c;
    if (a->L != b->L) return a->L < b->L ? -1 : 1;
    if (a->ray_id != b->ray_id) return a->ray_id < b->ray_id ? -1 : 1;
    return 0;
}

typedef struct {
    double delay;
    int64_t pos; /* position in key order */
} dkey;

static int delay_cmp(const void* pa, const void* pb) {
    const dkey *a = (const dkey*)pa, *b = (const dkey*)pb;
    if (a->delay != b->delay) return a->delay < b->delay ? -1 : 1;
    return a->pos < b->pos ? -1 : a->pos > b->pos ? 1 : 0;
}

static void points(const or_post_params* Q, const or_refined* r, double I[OR_MAX_INT + 2][3]) {
    for (int a = 0; a < 3; ++a) {
        I[0][a] = Q->tx[a];
        I[r->n_int + 1][a] = Q->rx[3 * (int64_t)r->rx + a];
    }
    for (int k = 0; k < r->n_int; ++k)
        for (int a = 0; a < 3; ++a) I[k + 1][a] = r->v[k][a];
}

/* is b a duplicate of the accepted path a (same rx and chain checked by the caller) */
int or_fresnel_dup(const or_post_params* Q, double cos_max, const or_refined* a, const or_refined* b) {
    double A[OR_MAX_INT + 2][3], B[OR_MAX_INT + 2][3];
    points(Q, a, A);
    points(Q, b, B);
    const int n = a->n_int;
    for (int k = 1; k <= n; ++k) {
        double u1[3] = {A[k - 1][0] - A[k][0], A[k - 1][1] - A[k][1], A[k - 1][2] - A[k][2]};
        double u2[3] = {A[k + 1][0] - A[k][0], A[k + 1][1] - A[k][1], A[k + 1][2] - A[k][2]};
        double s1 = sqrt(dot3(u1, u1)), s2 = sqrt(dot3(u2, u2));
        double psi2 = Q->lambda_m * s1 * s2 / (s1 + s2); /* Eq. 13 squared */
        double d[3] = {B[k][0] - A[k][0], B[k][1] - A[k][1], B[k][2] - A[k][2]};
        if (!(dot3(d, d) <= psi2)) return 0;
    }
    for (int k = 0; k <= n; ++k) {
        double u[3] = {A[k + 1][0] - A[k][0], A[k + 1][1] - A[k][1], A[k + 1][2] - A[k][2]};
        double w[3] = {B[k + 1][0] - B[k][0], B[k + 1][1] - B[k][1], B[k + 1][2] - B[k][2]};
        double c = dot3(u, w) / (sqrt(dot3(u, u)) * sqrt(dot3(w, w)));
        if (!(c > cos_max)) return 0;
    }
    return 1;
}

int64_t or_postprocess(const or_scene* S, const or_post_params* Q, const or_refined* in, int64_t n,
                       or_refined* out) {
    or_refined* w = (or_refined*)malloc(sizeof(or_refined) * (size_t)(n > 0 ? n : 1));
    int64_t m = 0;
    for (int64_t i = 0; i < n; ++i)
        if (in[i].status == NRT_OR_OK) w[m++] = in[i];
    /* 1. exact labels (brute force over every surfel) */
    const double lim2 = (2.0 * Q->r_s) * (2.0 * Q->r_s);
    for (int64_t q = 0; q < m; ++q)
        for (int k = 0; k < w[q].n_int; ++k) {
            if ((w[q].kinds >> k) & 1u) continue;
            const double* x = w[q].v[k];
            int64_t best = -1;
            double bd = 0.0;
            for (int64_t i = 0; i < S->n; ++i) {
                double d[3] = {(double)S->p[3 * i] - x[0], (double)S->p[3 * i + 1] - x[1],
                               (double)S->p[3 * i + 2] - x[2]};
                double d2 = dot3(d, d);
                if (d2 <= lim2 && (best < 0 || d2 < bd)) {
                    best = i;
                    bd = d2;
                }
            }
            if (best >= 0) w[q].label[k] = S->label[best];
        }
    /* 2. shortest per key */
    qsort(w, (size_t)m, sizeof(or_refined), shortest_cmp);
    int64_t u = 0;
    for (int64_t i = 0; i < m; ++i)
        if (u == 0 || key_cmp(&w[u - 1], &w[i]) != 0) w[u++] = w[i];
    /* 3. delay order */
    dkey* dk = (dkey*)malloc(sizeof(dkey) * (size_t)(u > 0 ? u : 1));
    for (int64_t i = 0; i < u; ++i) {
        dk[i].delay = w[i].delay;
        dk[i].pos = i;
    }
    qsort(dk, (size_t)u, sizeof(dkey), delay_cmp);
    /* 4. greedy first-Fresnel-zone dedupe */
    double sn, cos_max;
    or_sincos(Q->angle_deg * (3.14159265358979311600e+00 / 180.0), &sn, &cos_max);
    int64_t n_out = 0;
    for (int64_t j = 0; j < u; ++j) {
        const or_refined* b = &w[dk[j].pos];
        int dup = 0;
        for (int64_t i = 0; i < n_out && !dup; ++i) {
            const or_refined* a = &out[i];
            if (a->rx == b->rx && a->n_int == b->n_int && a->kinds == b->kinds)
                dup = or_fresnel_dup(Q, cos_max, a, b);
        }
        if (!dup) out[n_out++] = *b;
    }
    free(dk);
    free(w);
    return n_out;
}
