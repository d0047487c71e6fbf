/* gd.c — CPU ORACLE, NEXT-4: the paper's own path refinement.
 * TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * PAPER §II-E, Table I (rho = 2000, delta = 1e-4, alpha = beta = 0.4), Table II
 * (refinement r_s / t_sdf), Table III (t_d, t_a); readings R50-R56 of DESIGN.md.  FP32
 * throughout (the coarse tracer's precision), every operation in the order written here.
 *   R50 start: I_k = the coarse vertex; a reflection's AABB cell = the cell of its record point
 *       (R40 binning), its normal n = R53 at I_k, (u, v) = R54 basis of n; a diffraction moves
 *       along its edge's unit direction w (Eq. 8).
 *   R51 one iteration visits k = 1..N in order (Gauss-Seidel: I_{k-1} is already this
 *       iteration's): g = (I_k - I_{k+1})/|.| + (I_k - I_{k-1})/|.| (Eqs. fkr-fkt), the
 *       gradient (g.u, g.v) or g.w, Delta = -gradient, backtracking from gamma = 1: while
 *       f_k(x + gamma Delta) > f_k(x) + alpha gamma grad.Delta, gamma *= beta (Eq. 12; at most
 *       64 shrinks, then the point stays).
 *   R52 a diffraction's new point must lie on its edge (0 <= s <= len) else OFF_EDGE.
 *   R55 a reflection's new point is the SDF hit (R42-R44 with the refinement's r_s, t_sdf) of
 *       the ray from I_{k-1} toward the descended position, with the departure rule of vertex
 *       k-1 (its cell skipped, its normal / the edge's face normals as departure normals); no
 *       hit ends the path (NO_SUPPORT).  The new normal n' = R53 at the hit; the basis is kept
 *       when |(x' - x).n| < t_d and n.n' > cos t_a, else n = n', (u, v) = R54(n').
 *   R53 normal: Eq. 3 over the points of the hit AABB's 3x3x3 cell neighbourhood (sdf.c).
 *   R54 basis: u = (n x a)/|n x a|, a = the axis of least |n_i| (x < y < z on ties), v = n x u.
 *   R56 after rho iterations: ||grad f||^2 = sum of the squared gradient components at the
 *       final points < delta, else NO_CONVERGE; then each segment I_j -> I_{j+1} is traced
 *       (departure rule of j) and OCCLUDED if a hit lies before |I_{j+1} - I_j| - 2 xi r_s.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

#define C_LIGHT 299792458.0
#define PI_D 3.14159265358979323846

int64_t or_sdf_cell_of(const or_scene* S, const or_sdf* G, int64_t id);
int or_sdf_normal27(const or_scene* S, const or_sdf* G, int64_t cell, const float x[3], float sigma,
                    float n_out[3]);

static float dot3(const float a[3], const float b[3]) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }

/* |y - Q| + |y - P| (f_k, Eq. fk) */
static float fk(const float y[3], const float P[3], const float Q[3]) {
    float e1[3] = {y[0] - Q[0], y[1] - Q[1], y[2] - Q[2]};
    float e2[3] = {y[0] - P[0], y[1] - P[1], y[2] - P[2]};
    return sqrtf(dot3(e1, e1)) + sqrtf(dot3(e2, e2));
}

/* g = (x - Q)/|x - Q| + (x - P)/|x - P| and f_k(x) */
static float grad_vec(const float x[3], const float P[3], const float Q[3], float g[3]) {
    float e1[3] = {x[0] - Q[0], x[1] - Q[1], x[2] - Q[2]};
    float e2[3] = {x[0] - P[0], x[1] - P[1], x[2] - P[2]};
    const float l1 = sqrtf(dot3(e1, e1)), l2 = sqrtf(dot3(e2, e2));
    for (int i = 0; i < 3; ++i) g[i] = e1[i] / l1 + e2[i] / l2;
    return l1 + l2;
}

/* R54 */
void or_gd_basis(const float n[3], float u[3], float v[3]) {
    int ax = 0;
    if (fabsf(n[1]) < fabsf(n[ax])) ax = 1;
    if (fabsf(n[2]) < fabsf(n[ax])) ax = 2;
    float a[3] = {0.0f, 0.0f, 0.0f};
    a[ax] = 1.0f;
    float c[3] = {n[1] * a[2] - n[2] * a[1], n[2] * a[0] - n[0] * a[2], n[0] * a[1] - n[1] * a[0]};
    const float l = sqrtf(dot3(c, c));
    for (int i = 0; i < 3; ++i) u[i] = c[i] / l;
    v[0] = n[1] * u[2] - n[2] * u[1];
    v[1] = n[2] * u[0] - n[0] * u[2];
    v[2] = n[0] * u[1] - n[1] * u[0];
}

typedef struct {
    int kind;          /* 0 reflection, 1 diffraction */
    float x[3];
    float n[3], u[3], v[3];
    int64_t cell;      /* reflection: the AABB cell of the current point */
    int64_t pid;       /* reflection: the record point (nearest point of the hit AABB) */
    const or_edge* E;  /* diffraction */
    float w[3], len;
} gvert;

/* trace from vertex j (0 = TX) of the path toward `to`: departure rule of vertex j */
static int64_t trace_from(const or_scene* S, const or_gd_params* Q, const gvert* V, int j, const float* o,
                          const float d[3], float cos_ex, float* t, int64_t* cell, float nh[3]) {
    float lam[6];
    int n_lam = 0;
    int64_t prev = -1;
    if (j > 0) {
        const gvert* A = &V[j - 1];
        if (A->kind == 0) {
            for (int i = 0; i < 3; ++i) lam[i] = A->n[i];
            n_lam = 1;
            prev = A->cell;
        } else {
            for (int i = 0; i < 3; ++i) {
                lam[i] = A->E->n0[i];
                lam[3 + i] = A->E->n1[i];
            }
            n_lam = 2;
        }
    }
    return or_sdf_nearest(S, S->sdf, &Q->sdf, o, d, lam, n_lam, prev, Q->tau, cos_ex, t, cell, nh);
}

static void refine_gd_one(const or_scene* S, const or_gd_params* Q, const or_coarse* c, or_refined* out) {
    memset(out, 0, sizeof(*out));
    out->rx = c->rx;
    out->n_int = c->n_int;
    out->n_diff = c->n_diff;
    out->kinds = c->kinds;
    out->ray_id = c->ray_id;
    const int N = c->n_int;
    const float sigma = Q->sdf.xi * Q->sdf.r_s;
    const float cos_ex = or_cos_ex(Q->theta_ex_deg);
    const float cos_ta = or_cos_ex(Q->t_a_deg);  /* the same FP64 sincos, rounded to FP32 */
    float TX[3] = {Q->tx[0], Q->tx[1], Q->tx[2]};
    float RX[3] = {Q->rx[3 * c->rx], Q->rx[3 * c->rx + 1], Q->rx[3 * c->rx + 2]};
    gvert V[OR_MAX_INT];
    int status = NRT_OR_OK;
    /* R50 */
    for (int k = 0; k < N; ++k) {
        gvert* A = &V[k];
        memset(A, 0, sizeof(*A));
        for (int i = 0; i < 3; ++i) A->x[i] = c->v[k][i];
        out->label[k] = c->label[k];
        out->prim[k] = c->prim[k];
        if ((c->kinds >> k) & 1) {
            A->kind = 1;
            A->E = &S->edges[c->prim[k]];
            float ev[3] = {A->E->b[0] - A->E->a[0], A->E->b[1] - A->E->a[1], A->E->b[2] - A->E->a[2]};
            A->len = sqrtf(dot3(ev, ev));
            for (int i = 0; i < 3; ++i) A->w[i] = ev[i] / A->len;
        } else {
            A->kind = 0;
            A->pid = c->prim[k];
            A->cell = or_sdf_cell_of(S, S->sdf, A->pid);
            if (!or_sdf_normal27(S, S->sdf, A->cell, A->x, sigma, A->n)) status = NRT_OR_NO_SUPPORT;
            else or_gd_basis(A->n, A->u, A->v);
        }
    }
    int it = 0;
    for (; it < Q->rho && status == NRT_OR_OK; ++it) {
        for (int k = 0; k < N && status == NRT_OR_OK; ++k) {  /* R51 */
            gvert* A = &V[k];
            const float* P = k == 0 ? TX : V[k - 1].x;
            const float* R = k == N - 1 ? RX : V[k + 1].x;
            float g[3];
            const float f0 = grad_vec(A->x, P, R, g);
            float y[3];
            if (A->kind == 0) {
                const float gu = dot3(g, A->u), gv = dot3(g, A->v);
                const float slope = -(gu * gu + gv * gv);
                float gam = 1.0f;
                int ok = 0;
                for (int s = 0; s < 64; ++s) {
                    const float du = -gu * gam, dv = -gv * gam;
                    for (int i = 0; i < 3; ++i) y[i] = (A->x[i] + du * A->u[i]) + dv * A->v[i];
                    if (!(fk(y, P, R) > f0 + (Q->alpha * gam) * slope)) {
                        ok = 1;
                        break;
                    }
                    gam = Q->beta * gam;
                }
                if (!ok)
                    for (int i = 0; i < 3; ++i) y[i] = A->x[i];
                /* R55: reproject by tracing from I_{k-1} toward y */
                float d[3] = {y[0] - P[0], y[1] - P[1], y[2] - P[2]};
                const float ld = sqrtf(dot3(d, d));
                for (int i = 0; i < 3; ++i) d[i] = d[i] / ld;
                float t, nh[3];
                int64_t cell;
                const int64_t pid = trace_from(S, Q, V, k, P, d, cos_ex, &t, &cell, nh);
                if (pid < 0) {
                    status = NRT_OR_NO_SUPPORT;
                    break;
                }
                float xn[3] = {P[0] + t * d[0], P[1] + t * d[1], P[2] + t * d[2]};
                float nn[3];
                if (or_sdf_normal27(S, S->sdf, cell, xn, sigma, nn)) {
                    float dx[3] = {xn[0] - A->x[0], xn[1] - A->x[1], xn[2] - A->x[2]};
                    const float dist = fabsf(dot3(dx, A->n));
                    const float ca = dot3(A->n, nn);
                    if (!(dist < Q->t_d && ca > cos_ta)) {
                        for (int i = 0; i < 3; ++i) A->n[i] = nn[i];
                        or_gd_basis(A->n, A->u, A->v);
                    }
                }
                for (int i = 0; i < 3; ++i) A->x[i] = xn[i];
                A->cell = cell;
                A->pid = pid;
            } else {
                const float gw = dot3(g, A->w);
                const float slope = -(gw * gw);
                float gam = 1.0f;
                int ok = 0;
                for (int s = 0; s < 64; ++s) {
                    const float dw = -gw * gam;
                    for (int i = 0; i < 3; ++i) y[i] = A->x[i] + dw * A->w[i];
                    if (!(fk(y, P, R) > f0 + (Q->alpha * gam) * slope)) {
                        ok = 1;
                        break;
                    }
                    gam = Q->beta * gam;
                }
                if (!ok)
                    for (int i = 0; i < 3; ++i) y[i] = A->x[i];
                /* R52: still on the edge */
                float ya[3] = {y[0] - A->E->a[0], y[1] - A->E->a[1], y[2] - A->E->a[2]};
                const float s = dot3(ya, A->w);
                if (!(s >= 0.0f && s <= A->len)) {
                    status = NRT_OR_OFF_EDGE;
                    break;
                }
                for (int i = 0; i < 3; ++i) A->x[i] = y[i];
            }
        }
    }
    out->iters = it;
    /* R56: gradient norm at the final points */
    float gs = 0.0f;
    for (int k = 0; k < N; ++k) {
        const float* P = k == 0 ? TX : V[k - 1].x;
        const float* R = k == N - 1 ? RX : V[k + 1].x;
        float g[3];
        grad_vec(V[k].x, P, R, g);
        if (V[k].kind == 0) {
            const float gu = dot3(g, V[k].u), gv = dot3(g, V[k].v);
            gs = gs + (gu * gu + gv * gv);
        } else {
            const float gw = dot3(g, V[k].w);
            gs = gs + gw * gw;
        }
    }
    out->gradsq = gs;
    if (status == NRT_OR_OK && !(gs < Q->delta)) status = NRT_OR_NO_CONVERGE;
    if (status == NRT_OR_OK) {
        const float m = 2.0f * sigma;
        for (int j = 0; j <= N && status == NRT_OR_OK; ++j) {
            const float* o = j == 0 ? TX : V[j - 1].x;
            const float* to = j == N ? RX : V[j].x;
            float d[3] = {to[0] - o[0], to[1] - o[1], to[2] - o[2]};
            const float L = sqrtf(dot3(d, d));
            for (int i = 0; i < 3; ++i) d[i] = d[i] / L;
            float t, nh[3];
            int64_t cell;
            if (trace_from(S, Q, V, j, o, d, cos_ex, &t, &cell, nh) >= 0 && t < L - m) status = NRT_OR_OCCLUDED;
        }
    }
    out->status = status;
    /* outputs (FP64 from the FP32 points): vertices, L, delay, angles (R26, R27), labels (R44) */
    double I[OR_MAX_INT + 2][3];
    for (int i = 0; i < 3; ++i) {
        I[0][i] = TX[i];
        I[N + 1][i] = RX[i];
    }
    for (int k = 0; k < N; ++k) {
        for (int i = 0; i < 3; ++i) I[k + 1][i] = V[k].x[i];
        for (int i = 0; i < 3; ++i) out->v[k][i] = V[k].x[i];
        if (V[k].kind == 0) {
            out->prim[k] = (uint32_t)V[k].pid;
            out->label[k] = S->label[V[k].pid];
        }
    }
    double L = 0.0;
    for (int j = 0; j <= N; ++j) {
        double s[3] = {I[j + 1][0] - I[j][0], I[j + 1][1] - I[j][1], I[j + 1][2] - I[j][2]};
        L += sqrt(s[0] * s[0] + s[1] * s[1] + s[2] * s[2]);
    }
    out->L = L;
    out->delay = L / C_LIGHT;
    double d0[3] = {I[1][0] - I[0][0], I[1][1] - I[0][1], I[1][2] - I[0][2]};
    double l0 = sqrt(d0[0] * d0[0] + d0[1] * d0[1] + d0[2] * d0[2]);
    double dl[3] = {I[N][0] - I[N + 1][0], I[N][1] - I[N + 1][1], I[N][2] - I[N + 1][2]};
    double ll = sqrt(dl[0] * dl[0] + dl[1] * dl[1] + dl[2] * dl[2]);
    out->aod_az = (float)(atan2(d0[1], d0[0]) * 180.0 / PI_D);
    out->aod_el = (float)(asin(fmax(-1.0, fmin(1.0, d0[2] / l0))) * 180.0 / PI_D);
    out->aoa_az = (float)(atan2(dl[1], dl[0]) * 180.0 / PI_D);
    out->aoa_el = (float)(asin(fmax(-1.0, fmin(1.0, dl[2] / ll))) * 180.0 / PI_D);
    for (int k = 0; k < N; ++k) {
        double din[3] = {I[k + 1][0] - I[k][0], I[k + 1][1] - I[k][1], I[k + 1][2] - I[k][2]};
        double l = sqrt(din[0] * din[0] + din[1] * din[1] + din[2] * din[2]);
        const float* ax = V[k].kind == 0 ? V[k].n : V[k].w;
        double c2 = (din[0] * ax[0] + din[1] * ax[1] + din[2] * ax[2]) / l;
        if (V[k].kind == 0) c2 = fabs(c2);
        out->inc[k] = (float)(acos(fmax(-1.0, fmin(1.0, c2))) * 180.0 / PI_D);
    }
}

int or_refine_gd(const or_scene* S, const or_gd_params* Q, const or_coarse* in, int64_t n, or_refined* out) {
    if (!S->sdf) return 2;
    for (int64_t q = 0; q < n; ++q) refine_gd_one(S, Q, &in[q], &out[q]);
    return 0;
}

/* pin helper: one line search of vertex k of a path at points x (3N floats), as R51 (no
 * reprojection): writes the accepted gamma and the descended point */
float or_gd_line_search(const float x[3], const float P[3], const float Q3[3], const float u[3],
                        const float v[3], int diffraction, float alpha, float beta, float y[3]) {
    float g[3];
    const float f0 = grad_vec(x, P, Q3, g);
    const float gu = dot3(g, u), gv = diffraction ? 0.0f : dot3(g, v);
    const float slope = diffraction ? -(gu * gu) : -(gu * gu + gv * gv);
    float gam = 1.0f;
    for (int s = 0; s < 64; ++s) {
        const float du = -gu * gam, dv = -gv * gam;
        for (int i = 0; i < 3; ++i)
            y[i] = diffraction ? x[i] + du * u[i] : (x[i] + du * u[i]) + dv * v[i];
        if (!(fk(y, P, Q3) > f0 + (alpha * gam) * slope)) return gam;
        gam = beta * gam;
    }
    for (int i = 0; i < 3; ++i) y[i] = x[i];
    return 0.0f;
}
