/* refine.c — CPU ORACLE, path refinement (rows A9-A10).  TEST INFRASTRUCTURE ONLY.
 *
 * FP64, single-threaded, plain.  For a coarse path with interaction points I_1..I_n
 * (I_0 = TX, I_{n+1} = RX) the refined path is the root z* of the residual r(z)
 * reached by damped Gauss-Newton from the coarse seed (readings R18-R28):
 *
 *   reflection k (unknown x_k in R^3):
 *     N_k  = { i : label_i = label_k, |p_i - x_k| <= 4 sigma },   sigma = xi * r_s
 *     w_i  = exp(-|p_i - x_k|^2 / (2 sigma^2))                                      (Eq. 4)
 *     p(x) = sum w p / sum w                                                        (Eq. 2)
 *     n(x) = normalize(sum w sgn(n_i . n_seed) n_i / sum w)                         (Eq. 3, R20)
 *     f    = (x_k - p(x)) . n(x)                                                    (Eq. 1)
 *     g_k  = (I_k - I_{k-1})/|.| + (I_k - I_{k+1})/|.|                       (Eqs. 9-10 vector)
 *     (u, v) = basis of n(x): u = normalize(n x a), a = axis with least |n.a|, v = n x u
 *     r_k  = [ g_k . u, g_k . v, f ]
 *   diffraction k (unknown t_k, I_k = a + t_k e, Eq. 8):   r_k = g_k . e            (Eq. 11)
 *
 * Jacobian: central differences, h = 1e-7 m.  Step D = -(J^T J + lam I)^-1 J^T r,
 * lam = 1e-12 tr(J^T J)/dim.  Backtracking (Eq. 12 in its Armijo form, R24):
 * gamma <- beta*gamma while |r(z + gamma D)|^2 > (1 - 2 alpha gamma) |r(z)|^2.
 * Converged when |D|_inf < tol.  Stalled (NO_CONVERGE, reading R23b) when the accepted step
 * moved the iterate by less than tol, |gamma D|_inf < tol, while |D|_inf >= tol: the iterate
 * is then frozen at a non-root (a residual minimum with r != 0), and every further iteration
 * repeats the same step.  Then validity (R25): on-edge, same side, support,
 * visibility (FP64 shadow rays with sheet exclusions); delay = L / c (R26); angles (R27).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

#define NV OR_MAX_INT
#define MAXDIM (3 * OR_MAX_INT)

static const double C_LIGHT = 299792458.0;
static const double PI_D = 3.14159265358979311600e+00;

typedef struct {
    const or_scene* S;
    const or_refine_params* R;
    /* same-label index lists (label -> surfel ids) */
    int64_t* lab_start; /* [4097] */
    int64_t* lab_ids;   /* [n] */
    double sigma, rad2, tx[3], rx[3];
    /* optional neighbourhood index (or_refine on large clouds): cells of edge 4 sigma, ids
     * ascending per cell.  It only finds the candidates; the MLS sums run over exactly the
     * label-list ids within 4 sigma, in the same ascending order (bitwise the same sums). */
    int64_t* nb_start;  /* [ncell + 1] or NULL */
    int64_t* nb_ids;
    double nb_org[3], nb_cell;
    int64_t nb_dims[3];
    int64_t* scratch;   /* candidate ids of one query */
    int64_t scratch_cap;
} rctx_t;

static int or_refine_use_grid = 1; /* pin tests switch it off to compare with the plain loop */
void or_refine_set_grid(int on) { or_refine_use_grid = on; }

static int cmp_i64(const void* a, const void* b) {
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return x < y ? -1 : x > y;
}

/* the ids q of `label` with |p_q - x|^2 <= rad2, ascending (grid query); returns the count */
static int64_t nb_query(rctx_t* C, int32_t label, const double x[3]) {
    const or_scene* S = C->S;
    int64_t c[3], m = 0;
    for (int a = 0; a < 3; ++a) c[a] = (int64_t)floor((x[a] - C->nb_org[a]) / C->nb_cell);
    for (int64_t z = c[2] - 1; z <= c[2] + 1; ++z)
        for (int64_t y = c[1] - 1; y <= c[1] + 1; ++y)
            for (int64_t xx = c[0] - 1; xx <= c[0] + 1; ++xx) {
                if (xx < 0 || y < 0 || z < 0 || xx >= C->nb_dims[0] || y >= C->nb_dims[1] ||
                    z >= C->nb_dims[2])
                    continue;
                int64_t cell = xx + C->nb_dims[0] * (y + C->nb_dims[1] * z);
                for (int64_t k = C->nb_start[cell]; k < C->nb_start[cell + 1]; ++k) {
                    int64_t i = C->nb_ids[k];
                    if (S->label[i] != label) continue;
                    double dd[3] = {S->p[3 * i] - x[0], S->p[3 * i + 1] - x[1], S->p[3 * i + 2] - x[2]};
                    if ((dd[0] * dd[0] + dd[1] * dd[1]) + dd[2] * dd[2] > C->rad2) continue;
                    if (m == C->scratch_cap) {
                        C->scratch_cap = C->scratch_cap ? 2 * C->scratch_cap : 1024;
                        C->scratch = (int64_t*)realloc(C->scratch, sizeof(int64_t) * (size_t)C->scratch_cap);
                    }
                    C->scratch[m++] = i;
                }
            }
    qsort(C->scratch, (size_t)m, sizeof(int64_t), cmp_i64);
    return m;
}

static void nb_build(rctx_t* C) {
    const or_scene* S = C->S;
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = 0; i < S->n; ++i)
        for (int a = 0; a < 3; ++a) {
            lo[a] = fmin(lo[a], S->p[3 * i + a]);
            hi[a] = fmax(hi[a], S->p[3 * i + a]);
        }
    C->nb_cell = 4.0 * C->sigma;
    for (int a = 0; a < 3; ++a) {
        C->nb_org[a] = lo[a] - C->nb_cell;
        C->nb_dims[a] = (int64_t)ceil((hi[a] - C->nb_org[a]) / C->nb_cell) + 2;
    }
    int64_t nc = C->nb_dims[0] * C->nb_dims[1] * C->nb_dims[2];
    C->nb_start = (int64_t*)calloc((size_t)nc + 1, sizeof(int64_t));
    C->nb_ids = (int64_t*)malloc(sizeof(int64_t) * (size_t)(S->n > 0 ? S->n : 1));
    int64_t* cellof = (int64_t*)malloc(sizeof(int64_t) * (size_t)(S->n > 0 ? S->n : 1));
    for (int64_t i = 0; i < S->n; ++i) {
        int64_t c[3];
        for (int a = 0; a < 3; ++a) c[a] = (int64_t)floor((S->p[3 * i + a] - C->nb_org[a]) / C->nb_cell);
        cellof[i] = c[0] + C->nb_dims[0] * (c[1] + C->nb_dims[1] * c[2]);
        C->nb_start[cellof[i] + 1]++;
    }
    for (int64_t c = 0; c < nc; ++c) C->nb_start[c + 1] += C->nb_start[c];
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)nc);
    memcpy(fill, C->nb_start, sizeof(int64_t) * (size_t)nc);
    for (int64_t i = 0; i < S->n; ++i) C->nb_ids[fill[cellof[i]]++] = i;
    free(fill);
    free(cellof);
}

static double dot(const double a[3], const double b[3]) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }
static double norm(const double a[3]) { return sqrt(dot(a, a)); }
static void cross(const double a[3], const double b[3], double o[3]) {
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
}

/* MLS at x over the same-label neighbourhood (Eqs. 1-4). Returns 0 if empty/degenerate. */
static int mls(const rctx_t* C, int32_t label, const double nseed[3], const double x[3],
               double pbar[3], double nbar[3]) {
    const or_scene* S = C->S;
    double W = 0, P[3] = {0, 0, 0}, Nn[3] = {0, 0, 0};
    const int64_t* ids = C->lab_ids + C->lab_start[label];
    int64_t cnt = C->lab_start[label + 1] - C->lab_start[label];
    if (C->nb_start) {
        cnt = nb_query((rctx_t*)C, label, x);
        ids = C->scratch;
    }
    for (int64_t q = 0; q < cnt; ++q) {
        int64_t i = ids[q];
        double p[3] = {S->p[3 * i], S->p[3 * i + 1], S->p[3 * i + 2]};
        double dd[3] = {p[0] - x[0], p[1] - x[1], p[2] - x[2]};
        double d2 = dot(dd, dd);
        if (d2 > C->rad2) continue;
        double w = exp(-d2 / (2.0 * C->sigma * C->sigma));
        double n[3] = {S->nrm[3 * i], S->nrm[3 * i + 1], S->nrm[3 * i + 2]};
        double sg = dot(n, nseed) < 0.0 ? -1.0 : 1.0;
        W += w;
        for (int a = 0; a < 3; ++a) {
            P[a] += w * p[a];
            Nn[a] += w * sg * n[a];
        }
    }
    if (!(W > 0.0)) return 0;
    for (int a = 0; a < 3; ++a) {
        pbar[a] = P[a] / W;
        nbar[a] = Nn[a] / W;
    }
    double l = norm(nbar);
    if (!(l > 0.0)) return 0;
    for (int a = 0; a < 3; ++a) nbar[a] /= l;
    return 1;
}

/* MLS at x with the derivatives of pbar(x) and nbar(x) (analytic Jacobian, reading R37):
 *   w_i = exp(-|d_i|^2 / 2 s^2), d_i = p_i - x, dw_i/dx = w_i d_i / s^2;
 *   pbar = x + sum w d / W,  dpbar/dx = (sum w d d^T / s^2 - (pbar - x) dW^T) / W,
 *     dW = sum w d / s^2;
 *   nbar = N / |N|, N = sum w sgn(n_i . n_seed) n_i,
 *   dnbar/dx = (I - nbar nbar^T) (sum w sgn n_i d^T / s^2) / |N|.
 * The same neighbourhood (same-label surfels within 4 sigma) and id order as mls().
 * Returns 0 where mls() does. */
static int mls_d(const rctx_t* C, int32_t label, const double nseed[3], const double x[3],
                 double dP[3][3], double dN[3][3], double nbar[3], double pbar[3]) {
    const or_scene* S = C->S;
    const double s2 = C->sigma * C->sigma;
    double W = 0, Dv[3] = {0, 0, 0}, Sdd[3][3] = {{0}}, Nn[3] = {0, 0, 0}, Snd[3][3] = {{0}};
    const int64_t* ids = C->lab_ids + C->lab_start[label];
    int64_t cnt = C->lab_start[label + 1] - C->lab_start[label];
    if (C->nb_start) {
        cnt = nb_query((rctx_t*)C, label, x);
        ids = C->scratch;
    }
    for (int64_t q = 0; q < cnt; ++q) {
        int64_t i = ids[q];
        double p[3] = {S->p[3 * i], S->p[3 * i + 1], S->p[3 * i + 2]};
        double dd[3] = {p[0] - x[0], p[1] - x[1], p[2] - x[2]};
        double d2 = dot(dd, dd);
        if (d2 > C->rad2) continue;
        double w = exp(-d2 / (2.0 * C->sigma * C->sigma));
        double n[3] = {S->nrm[3 * i], S->nrm[3 * i + 1], S->nrm[3 * i + 2]};
        double sg = dot(n, nseed) < 0.0 ? -1.0 : 1.0;
        W += w;
        for (int a = 0; a < 3; ++a) {
            Dv[a] += w * dd[a];
            Nn[a] += w * sg * n[a];
            for (int b = 0; b < 3; ++b) {
                Sdd[a][b] += w * dd[a] * dd[b];
                Snd[a][b] += w * sg * n[a] * dd[b];
            }
        }
    }
    if (!(W > 0.0)) return 0;
    double ln = norm(Nn);
    if (!(ln > 0.0)) return 0;
    double dW[3], q[3];
    for (int a = 0; a < 3; ++a) {
        dW[a] = Dv[a] / s2;
        q[a] = Dv[a] / W;          /* pbar - x */
        pbar[a] = x[a] + q[a];
        nbar[a] = Nn[a] / ln;
    }
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) dP[a][b] = (Sdd[a][b] / s2 - q[a] * dW[b]) / W;
    double M[3][3];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) M[a][b] = Snd[a][b] / s2;
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
            double t = M[a][b];
            for (int c = 0; c < 3; ++c) t -= nbar[a] * nbar[c] * M[c][b];
            dN[a][b] = t / ln;
        }
    return 1;
}

static void basis(const double n[3], double u[3], double v[3]) {
    double ax[3] = {0, 0, 0};
    double m0 = fabs(n[0]), m1 = fabs(n[1]), m2 = fabs(n[2]);
    int k = 0;
    if (m1 < m0) k = 1;
    if (m2 < (k == 0 ? m0 : m1)) k = 2;
    ax[k] = 1.0;
    cross(n, ax, u);
    double l = norm(u);
    for (int a = 0; a < 3; ++a) u[a] /= l;
    cross(n, u, v);
}

typedef struct {
    int n;                 /* interactions */
    int dim;
    int kind[NV];          /* 0 reflection, 1 diffraction */
    int32_t label[NV];
    uint32_t prim[NV];
    double nseed[NV][3];   /* reflection: normal of the coarse hit surfel */
    double ea[NV][3], ee[NV][3], elen[NV]; /* diffraction: edge origin, unit dir, length */
    int col[NV];           /* first unknown index */
} pathdef_t;

/* unknown vector z -> interaction points I[0..n+1] */
static void points(const rctx_t* C, const pathdef_t* D, const double* z, double I[NV + 2][3]) {
    for (int a = 0; a < 3; ++a) {
        I[0][a] = C->tx[a];
        I[D->n + 1][a] = C->rx[a];
    }
    for (int k = 0; k < D->n; ++k) {
        const double* zk = z + D->col[k];
        if (D->kind[k] == 0)
            for (int a = 0; a < 3; ++a) I[k + 1][a] = zk[a];
        else
            for (int a = 0; a < 3; ++a) I[k + 1][a] = D->ea[k][a] + zk[0] * D->ee[k][a];
    }
}

/* residual r(z); also the per-vertex MLS normals. returns 0 if undefined (no support) */
static int residual(const rctx_t* C, const pathdef_t* D, const double* z, double* r,
                    double nbar_out[NV][3], double* gradsq) {
    double I[NV + 2][3];
    points(C, D, z, I);
    double gs = 0.0;
    for (int k = 0; k < D->n; ++k) {
        const double* x = I[k + 1];
        double a[3] = {x[0] - I[k][0], x[1] - I[k][1], x[2] - I[k][2]};
        double b[3] = {x[0] - I[k + 2][0], x[1] - I[k + 2][1], x[2] - I[k + 2][2]};
        double la = norm(a), lb = norm(b);
        if (!(la > 0.0 && lb > 0.0)) return 0;
        double g[3] = {a[0] / la + b[0] / lb, a[1] / la + b[1] / lb, a[2] / la + b[2] / lb};
        double* rk = r + D->col[k];
        if (D->kind[k] == 0) {
            double pb[3], nb[3], u[3], v[3];
            if (!mls(C, D->label[k], D->nseed[k], x, pb, nb)) return 0;
            basis(nb, u, v);
            double xp[3] = {x[0] - pb[0], x[1] - pb[1], x[2] - pb[2]};
            rk[0] = dot(g, u);
            rk[1] = dot(g, v);
            rk[2] = dot(xp, nb);
            gs += rk[0] * rk[0] + rk[1] * rk[1];
            if (nbar_out)
                for (int q = 0; q < 3; ++q) nbar_out[k][q] = nb[q];
        } else {
            rk[0] = dot(g, D->ee[k]);
            gs += rk[0] * rk[0];
        }
    }
    if (gradsq) *gradsq = gs;
    return 1;
}

/* Analytic Jacobian of the residual of residual() (reading R37): chain rule through
 * g_k = (x_k - x_{k-1})/|.| + (x_k - x_{k+1})/|.| (d(h/|h|)/dh = (I - h h^T/|h|^2)/|h|),
 * the MLS point and normal (mls_d), the basis u = normalize(nbar x a) (a fixed per evaluation:
 * du/dnbar = (I - u u^T)/|nbar x a| (-[a]x)), v = nbar x u (dv/dnbar = -[u]x + [nbar]x du/dnbar)
 * and x_k = a_k + t_k e_k for diffractions.  J[i*m + j] = dr_i/dz_j.  0 where the residual is
 * undefined. */
static void cross_mat(const double a[3], double Mx[3][3]) { /* Mx v = a x v */
    Mx[0][0] = 0; Mx[0][1] = -a[2]; Mx[0][2] = a[1];
    Mx[1][0] = a[2]; Mx[1][1] = 0; Mx[1][2] = -a[0];
    Mx[2][0] = -a[1]; Mx[2][1] = a[0]; Mx[2][2] = 0;
}

static int jacobian(const rctx_t* C, const pathdef_t* D, const double* z, double* J) {
    const int m = D->dim;
    double I[NV + 2][3];
    points(C, D, z, I);
    memset(J, 0, sizeof(double) * m * m);
    for (int k = 0; k < D->n; ++k) {
        const double* x = I[k + 1];
        double a[3] = {x[0] - I[k][0], x[1] - I[k][1], x[2] - I[k][2]};
        double b[3] = {x[0] - I[k + 2][0], x[1] - I[k + 2][1], x[2] - I[k + 2][2]};
        double la = norm(a), lb = norm(b);
        if (!(la > 0.0 && lb > 0.0)) return 0;
        double ha[3], hb[3], g[3];
        for (int q = 0; q < 3; ++q) {
            ha[q] = a[q] / la;
            hb[q] = b[q] / lb;
            g[q] = ha[q] + hb[q];
        }
        double Ma[3][3], Mb[3][3];
        for (int p = 0; p < 3; ++p)
            for (int q = 0; q < 3; ++q) {
                Ma[p][q] = ((p == q ? 1.0 : 0.0) - ha[p] * ha[q]) / la;
                Mb[p][q] = ((p == q ? 1.0 : 0.0) - hb[p] * hb[q]) / lb;
            }
        /* rows of vertex k: derivative rows w.r.t. x_{k-1}, x_k, x_{k+1} (R[row][nbr][coord]) */
        int nrow = D->kind[k] == 0 ? 3 : 1;
        double R[3][3][3];
        memset(R, 0, sizeof(R));
        if (D->kind[k] == 0) {
            double dP[3][3], dN[3][3], nb[3], pb[3];
            if (!mls_d(C, D->label[k], D->nseed[k], x, dP, dN, nb, pb)) return 0;
            /* the residual's own MLS point (P/W, as residual()) for (x - pbar) */
            double pbr[3], nbr[3];
            if (!mls(C, D->label[k], D->nseed[k], x, pbr, nbr)) return 0;
            double u[3], v[3];
            basis(nbr, u, v);
            double m0 = fabs(nbr[0]), m1 = fabs(nbr[1]), m2 = fabs(nbr[2]);
            int ax = 0;
            if (m1 < m0) ax = 1;
            if (m2 < (ax == 0 ? m0 : m1)) ax = 2;
            double av[3] = {0, 0, 0};
            av[ax] = 1.0;
            double c[3];
            cross(nbr, av, c);
            double lc = norm(c), Ax[3][3], Ux[3][3], Nx[3][3], dU[3][3], dV[3][3];
            cross_mat(av, Ax);
            cross_mat(u, Ux);
            cross_mat(nbr, Nx);
            for (int p = 0; p < 3; ++p)
                for (int q = 0; q < 3; ++q) {
                    double t = 0;
                    for (int r = 0; r < 3; ++r) t += ((p == r ? 1.0 : 0.0) - u[p] * u[r]) * (-Ax[r][q]);
                    dU[p][q] = t / lc;
                }
            for (int p = 0; p < 3; ++p)
                for (int q = 0; q < 3; ++q) {
                    double t = -Ux[p][q];
                    for (int r = 0; r < 3; ++r) t += Nx[p][r] * dU[r][q];
                    dV[p][q] = t;
                }
            double xp[3] = {x[0] - pbr[0], x[1] - pbr[1], x[2] - pbr[2]};
            for (int q = 0; q < 3; ++q) {
                double gu = 0, gv = 0, uM = 0, vM = 0, up = 0, vp = 0, un = 0, vn = 0, fx = 0;
                for (int p = 0; p < 3; ++p) {
                    /* g^T dU dN[:, q] and g^T dV dN[:, q] */
                    double dun = 0, dvn = 0;
                    for (int r = 0; r < 3; ++r) {
                        dun += dU[p][r] * dN[r][q];
                        dvn += dV[p][r] * dN[r][q];
                    }
                    gu += g[p] * dun;
                    gv += g[p] * dvn;
                    uM += u[p] * (Ma[p][q] + Mb[p][q]);
                    vM += v[p] * (Ma[p][q] + Mb[p][q]);
                    up += u[p] * Ma[p][q];
                    vp += v[p] * Ma[p][q];
                    un += u[p] * Mb[p][q];
                    vn += v[p] * Mb[p][q];
                    fx += nbr[p] * ((p == q ? 1.0 : 0.0) - dP[p][q]) + xp[p] * dN[p][q];
                }
                R[0][1][q] = uM + gu;
                R[1][1][q] = vM + gv;
                R[2][1][q] = fx;
                R[0][0][q] = -up;
                R[1][0][q] = -vp;
                R[0][2][q] = -un;
                R[1][2][q] = -vn;
            }
        } else {
            const double* e = D->ee[k];
            for (int q = 0; q < 3; ++q) {
                double t1 = 0, t0 = 0, t2 = 0;
                for (int p = 0; p < 3; ++p) {
                    t1 += e[p] * (Ma[p][q] + Mb[p][q]);
                    t0 += e[p] * Ma[p][q];
                    t2 += e[p] * Mb[p][q];
                }
                R[0][1][q] = t1;
                R[0][0][q] = -t0;
                R[0][2][q] = -t2;
            }
        }
        /* scatter into J: neighbour j = k-1, k, k+1 (unknown vertices only) */
        for (int nb_ = 0; nb_ < 3; ++nb_) {
            int j = k - 1 + nb_;
            if (j < 0 || j >= D->n) continue;
            for (int row = 0; row < nrow; ++row) {
                double* Jr = J + (D->col[k] + row) * m;
                if (D->kind[j] == 0) {
                    for (int q = 0; q < 3; ++q) Jr[D->col[j] + q] += R[row][nb_][q];
                } else {
                    double t = 0;
                    for (int q = 0; q < 3; ++q) t += R[row][nb_][q] * D->ee[j][q];
                    Jr[D->col[j]] += t;
                }
            }
        }
    }
    return 1;
}

static double sq(const double* r, int m) {
    double s = 0;
    for (int i = 0; i < m; ++i) s += r[i] * r[i];
    return s;
}

/* solve (A) x = b for SPD A (dim <= MAXDIM) by Cholesky; 0 on failure */
static int chol_solve(double* A, double* b, int m) {
    for (int j = 0; j < m; ++j) {
        double d = A[j * m + j];
        for (int k = 0; k < j; ++k) d -= A[j * m + k] * A[j * m + k];
        if (!(d > 0.0)) return 0;
        d = sqrt(d);
        A[j * m + j] = d;
        for (int i = j + 1; i < m; ++i) {
            double s = A[i * m + j];
            for (int k = 0; k < j; ++k) s -= A[i * m + k] * A[j * m + k];
            A[i * m + j] = s / d;
        }
    }
    for (int i = 0; i < m; ++i) {
        double s = b[i];
        for (int k = 0; k < i; ++k) s -= A[i * m + k] * b[k];
        b[i] = s / A[i * m + i];
    }
    for (int i = m - 1; i >= 0; --i) {
        double s = b[i];
        for (int k = i + 1; k < m; ++k) s -= A[k * m + i] * b[k];
        b[i] = s / A[i * m + i];
    }
    return 1;
}

/* FP64 segment occlusion test with departure/arrival sheet exclusions (R25 d) */
static int occluded(const rctx_t* C, const double x0[3], const double x1[3], const double* lam0,
                    int n0, const double* lam1, int n1) {
    const or_scene* S = C->S;
    const double tau = C->R->tau;
    double s, ce;
    or_sincos(C->R->theta_ex_deg * (PI_D / 180.0), &s, &ce);
    double dv[3] = {x1[0] - x0[0], x1[1] - x0[1], x1[2] - x0[2]};
    double len = norm(dv);
    double d[3] = {dv[0] / len, dv[1] / len, dv[2] / len};
    for (int64_t i = 0; i < S->n; ++i) {
        double p[3] = {S->p[3 * i], S->p[3 * i + 1], S->p[3 * i + 2]};
        double n[3] = {S->nrm[3 * i], S->nrm[3 * i + 1], S->nrm[3 * i + 2]};
        double r = S->r[i];
        double w[3] = {x0[0] - p[0], x0[1] - p[1], x0[2] - p[2]};
        double f0 = dot(w, n), dn = dot(d, n);
        if (!(f0 * dn < 0.0)) continue;
        double t = -f0 / dn;
        if (!(t < len)) continue;
        double h[3] = {x0[0] + t * d[0] - p[0], x0[1] + t * d[1] - p[1], x0[2] + t * d[2] - p[2]};
        if (!(dot(h, h) <= r * r)) continue;
        int ex = 0;
        if (fabs(f0) <= tau)
            for (int k = 0; k < n0; ++k)
                if (fabs(dot(n, lam0 + 3 * k)) >= ce) ex = 1;
        double w1[3] = {x1[0] - p[0], x1[1] - p[1], x1[2] - p[2]};
        double f1 = dot(w1, n);
        if (!ex && fabs(f1) <= tau)
            for (int k = 0; k < n1; ++k)
                if (fabs(dot(n, lam1 + 3 * k)) >= ce) ex = 1;
        if (!ex) return 1;
    }
    return 0;
}

static int supported(const rctx_t* C, int32_t label, const double x[3]) {
    const or_scene* S = C->S;
    const double tau = C->R->tau;
    for (int64_t q = C->lab_start[label]; q < C->lab_start[label + 1]; ++q) {
        int64_t i = C->lab_ids[q];
        double p[3] = {S->p[3 * i], S->p[3 * i + 1], S->p[3 * i + 2]};
        double n[3] = {S->nrm[3 * i], S->nrm[3 * i + 1], S->nrm[3 * i + 2]};
        double r = S->r[i];
        double w[3] = {x[0] - p[0], x[1] - p[1], x[2] - p[2]};
        if (fabs(dot(w, n)) <= tau && dot(w, w) <= r * r + tau * tau) return 1;
    }
    return 0;
}

static void refine_one(const rctx_t* C, const or_coarse* c, or_refined* out) {
    const or_scene* S = C->S;
    const or_refine_params* R = C->R;
    memset(out, 0, sizeof(*out));
    out->rx = c->rx;
    out->n_int = c->n_int;
    out->n_diff = c->n_diff;
    out->kinds = c->kinds;
    for (int k = 0; k < NV; ++k) {
        out->label[k] = c->label[k];
        out->prim[k] = c->prim[k];
    }
    out->ray_id = c->ray_id;
    pathdef_t D;
    memset(&D, 0, sizeof(D));
    D.n = c->n_int;
    double z[MAXDIM];
    int m = 0;
    for (int k = 0; k < D.n; ++k) {
        D.kind[k] = (c->kinds >> k) & 1u;
        D.label[k] = c->label[k];
        D.prim[k] = c->prim[k];
        D.col[k] = m;
        if (D.kind[k] == 0) {
            for (int a = 0; a < 3; ++a) {
                D.nseed[k][a] = S->nrm[3 * (int64_t)c->prim[k] + a];
                z[m + a] = c->v[k][a];
            }
            m += 3;
        } else {
            const or_edge* E = &S->edges[c->prim[k]];
            double ev[3] = {(double)E->b[0] - E->a[0], (double)E->b[1] - E->a[1], (double)E->b[2] - E->a[2]};
            double l = norm(ev);
            for (int a = 0; a < 3; ++a) {
                D.ea[k][a] = E->a[a];
                D.ee[k][a] = ev[a] / l;
            }
            D.elen[k] = l;
            double w[3] = {c->v[k][0] - D.ea[k][0], c->v[k][1] - D.ea[k][1], c->v[k][2] - D.ea[k][2]};
            z[m] = dot(w, D.ee[k]);
            m += 1;
        }
    }
    D.dim = m;
    const double h = 1e-7;
    double r[MAXDIM], rp[MAXDIM], rm[MAXDIM], J[MAXDIM * MAXDIM], A[MAXDIM * MAXDIM], b[MAXDIM];
    int status = NRT_OR_NO_CONVERGE, it = 0;
    if (m == 0) status = NRT_OR_OK; /* LOS */
    else if (!residual(C, &D, z, r, NULL, NULL)) status = NRT_OR_NO_SUPPORT;
    else {
        for (it = 1; it <= R->max_iter; ++it) {
            int ok = 1;
            if (R->jac_fd) { /* Jacobian by central differences */
                for (int j = 0; j < m && ok; ++j) {
                    double zj = z[j];
                    z[j] = zj + h;
                    ok &= residual(C, &D, z, rp, NULL, NULL);
                    z[j] = zj - h;
                    ok &= residual(C, &D, z, rm, NULL, NULL);
                    z[j] = zj;
                    for (int i = 0; i < m; ++i) J[i * m + j] = (rp[i] - rm[i]) / (2.0 * h);
                }
            } else { /* analytic Jacobian (R37) */
                ok = jacobian(C, &D, z, J);
            }
            if (!ok) {
                status = NRT_OR_NO_SUPPORT;
                break;
            }
            double tr = 0;
            for (int i = 0; i < m; ++i) {
                for (int j = 0; j < m; ++j) {
                    double s = 0;
                    for (int q = 0; q < m; ++q) s += J[q * m + i] * J[q * m + j];
                    A[i * m + j] = s;
                }
                tr += A[i * m + i];
                double s = 0;
                for (int q = 0; q < m; ++q) s += J[q * m + i] * r[q];
                b[i] = -s;
            }
            double lam = 1e-12 * tr / m;
            for (int i = 0; i < m; ++i) A[i * m + i] += lam;
            if (!chol_solve(A, b, m)) {
                status = NRT_OR_DEGENERATE;
                break;
            }
            double dmax = 0;
            for (int i = 0; i < m; ++i) dmax = fmax(dmax, fabs(b[i]));
            if (dmax < R->tol_m) { /* converged: take the (tiny) full step */
                double zt[MAXDIM] = {0};
                for (int i = 0; i < m; ++i) zt[i] = z[i] + b[i];
                if (residual(C, &D, zt, rp, NULL, NULL)) {
                    for (int i = 0; i < m; ++i) z[i] = zt[i];
                    memcpy(r, rp, sizeof(double) * m);
                }
                status = NRT_OR_OK;
                break;
            }
            double f0 = sq(r, m), gam = 1.0;
            int acc = 0;
            while (gam > 1e-12) {
                double zt[MAXDIM];
                for (int i = 0; i < m; ++i) zt[i] = z[i] + gam * b[i];
                if (residual(C, &D, zt, rp, NULL, NULL) &&
                    sq(rp, m) <= (1.0 - 2.0 * R->alpha * gam) * f0) {
                    for (int i = 0; i < m; ++i) z[i] = zt[i];
                    memcpy(r, rp, sizeof(double) * m);
                    acc = 1;
                    break;
                }
                gam *= R->beta;
            }
            if (!acc) {
                status = NRT_OR_NO_CONVERGE;
                break;
            }
            if (gam * dmax < R->tol_m) { /* R23b: stalled at a non-root */
                status = NRT_OR_NO_CONVERGE;
                break;
            }
        }
        if (it > R->max_iter) it = R->max_iter;
    }
    out->iters = it;
    double I[NV + 2][3], nb[NV][3];
    memset(nb, 0, sizeof(nb));
    points(C, &D, z, I);
    double gsq = 0;
    if (status == NRT_OR_OK && m > 0) {
        if (!residual(C, &D, z, r, nb, &gsq)) status = NRT_OR_NO_SUPPORT;
    }
    out->gradsq = gsq;
    double rmax = 0;
    for (int i = 0; i < m; ++i) rmax = fmax(rmax, fabs(r[i]));
    out->resid = m ? rmax : 0.0;
    /* validity (R25) in order */
    if (status == NRT_OR_OK)
        for (int k = 0; k < D.n; ++k)
            if (D.kind[k] == 1) {
                double t = z[D.col[k]];
                if (!(t >= 0.0 && t <= D.elen[k])) status = NRT_OR_OFF_EDGE;
            }
    if (status == NRT_OR_OK)
        for (int k = 0; k < D.n; ++k)
            if (D.kind[k] == 0) {
                double a[3] = {I[k][0] - I[k + 1][0], I[k][1] - I[k + 1][1], I[k][2] - I[k + 1][2]};
                double bb[3] = {I[k + 2][0] - I[k + 1][0], I[k + 2][1] - I[k + 1][1], I[k + 2][2] - I[k + 1][2]};
                double sa = dot(a, nb[k]), sb = dot(bb, nb[k]);
                if (!((sa > 0 && sb > 0) || (sa < 0 && sb < 0))) status = NRT_OR_WRONG_SIDE;
            }
    if (status == NRT_OR_OK)
        for (int k = 0; k < D.n; ++k)
            if (D.kind[k] == 0 && !supported(C, D.label[k], I[k + 1])) status = NRT_OR_NO_SUPPORT;
    if (status == NRT_OR_OK) {
        for (int j = 0; j <= D.n && status == NRT_OR_OK; ++j) {
            double l0[6], l1[6];
            int n0 = 0, n1 = 0;
            if (j >= 1) { /* departure vertex j */
                int k = j - 1;
                if (D.kind[k] == 0) {
                    memcpy(l0, nb[k], sizeof(double) * 3);
                    n0 = 1;
                } else {
                    const or_edge* E = &S->edges[D.prim[k]];
                    for (int a = 0; a < 3; ++a) {
                        l0[a] = E->n0[a];
                        l0[3 + a] = E->n1[a];
                    }
                    n0 = 2;
                }
            }
            if (j + 1 <= D.n) { /* arrival vertex j+1 */
                int k = j;
                if (D.kind[k] == 0) {
                    memcpy(l1, nb[k], sizeof(double) * 3);
                    n1 = 1;
                } else {
                    const or_edge* E = &S->edges[D.prim[k]];
                    for (int a = 0; a < 3; ++a) {
                        l1[a] = E->n0[a];
                        l1[3 + a] = E->n1[a];
                    }
                    n1 = 2;
                }
            }
            if (occluded(C, I[j], I[j + 1], l0, n0, l1, n1)) status = NRT_OR_OCCLUDED;
        }
    }
    out->status = status;
    double L = 0;
    for (int j = 0; j <= D.n; ++j) {
        double s[3] = {I[j + 1][0] - I[j][0], I[j + 1][1] - I[j][1], I[j + 1][2] - I[j][2]};
        L += norm(s);
    }
    out->L = L;
    out->delay = L / C_LIGHT;
    for (int k = 0; k < D.n; ++k)
        for (int a = 0; a < 3; ++a) out->v[k][a] = I[k + 1][a];
    /* angles (R27): AoD along the first segment, AoA from the RX toward the last vertex */
    double d0[3] = {I[1][0] - I[0][0], I[1][1] - I[0][1], I[1][2] - I[0][2]};
    double l0 = norm(d0);
    double dl[3] = {I[D.n][0] - I[D.n + 1][0], I[D.n][1] - I[D.n + 1][1], I[D.n][2] - I[D.n + 1][2]};
    double ll = norm(dl);
    out->aod_az = (float)(atan2(d0[1], d0[0]) * 180.0 / PI_D);
    out->aod_el = (float)(asin(fmax(-1.0, fmin(1.0, d0[2] / l0))) * 180.0 / PI_D);
    out->aoa_az = (float)(atan2(dl[1], dl[0]) * 180.0 / PI_D);
    out->aoa_el = (float)(asin(fmax(-1.0, fmin(1.0, dl[2] / ll))) * 180.0 / PI_D);
    for (int k = 0; k < D.n; ++k) {
        double din[3] = {I[k + 1][0] - I[k][0], I[k + 1][1] - I[k][1], I[k + 1][2] - I[k][2]};
        double l = norm(din);
        double c2 = D.kind[k] == 0 ? fabs(dot(din, nb[k])) / l : dot(din, D.ee[k]) / l;
        out->inc[k] = (float)(acos(fmax(-1.0, fmin(1.0, c2))) * 180.0 / PI_D);
    }
}

int or_refine(const or_scene* S, const or_refine_params* R, const or_coarse* in, int64_t n,
              or_refined* out) {
    rctx_t C;
    memset(&C, 0, sizeof(C));
    C.S = S;
    C.R = R;
    C.sigma = R->xi * R->r_s;
    C.rad2 = (4.0 * C.sigma) * (4.0 * C.sigma);
    for (int a = 0; a < 3; ++a) {
        C.tx[a] = R->tx[a];
        C.rx[a] = 0;
    }
    C.lab_start = (int64_t*)calloc(4097 + 1, sizeof(int64_t));
    C.lab_ids = (int64_t*)malloc(sizeof(int64_t) * (size_t)(S->n > 0 ? S->n : 1));
    for (int64_t i = 0; i < S->n; ++i) C.lab_start[S->label[i] + 1]++;
    for (int l = 0; l < 4097; ++l) C.lab_start[l + 1] += C.lab_start[l];
    int64_t* fill = (int64_t*)calloc(4097, sizeof(int64_t));
    for (int64_t i = 0; i < S->n; ++i) {
        int l = S->label[i];
        C.lab_ids[C.lab_start[l] + fill[l]++] = i;
    }
    free(fill);
    if (or_refine_use_grid && n > 0 && S->n > 0) nb_build(&C);
    for (int64_t q = 0; q < n; ++q) {
        for (int a = 0; a < 3; ++a) C.rx[a] = R->rx[3 * (int64_t)in[q].rx + a];
        refine_one(&C, &in[q], &out[q]);
    }
    free(C.lab_start);
    free(C.lab_ids);
    free(C.nb_start);
    free(C.nb_ids);
    free(C.scratch);
    return 0;
}

/* pin helper: residual r(z) of coarse record c at its seed (z == NULL) or at z; returns dim
 * (or -1 if undefined); z_out (optional) receives the seed unknowns */
int or_path_residual(const or_scene* S, const or_refine_params* R, const or_coarse* c,
                     const double* z_in, double* r_out, double* z_out) {
    rctx_t C;
    memset(&C, 0, sizeof(C));
    C.S = S;
    C.R = R;
    C.sigma = R->xi * R->r_s;
    C.rad2 = (4.0 * C.sigma) * (4.0 * C.sigma);
    for (int a = 0; a < 3; ++a) {
        C.tx[a] = R->tx[a];
        C.rx[a] = R->rx[3 * (int64_t)c->rx + a];
    }
    C.lab_start = (int64_t*)calloc(4098, sizeof(int64_t));
    C.lab_ids = (int64_t*)malloc(sizeof(int64_t) * (size_t)(S->n > 0 ? S->n : 1));
    for (int64_t i = 0; i < S->n; ++i) C.lab_start[S->label[i] + 1]++;
    for (int l = 0; l < 4097; ++l) C.lab_start[l + 1] += C.lab_start[l];
    int64_t* fill = (int64_t*)calloc(4097, sizeof(int64_t));
    for (int64_t i = 0; i < S->n; ++i) C.lab_ids[C.lab_start[S->label[i]] + fill[S->label[i]]++] = i;
    free(fill);
    pathdef_t D;
    memset(&D, 0, sizeof(D));
    D.n = c->n_int;
    double z[MAXDIM];
    int m = 0;
    for (int k = 0; k < D.n; ++k) {
        D.kind[k] = (c->kinds >> k) & 1u;
        D.label[k] = c->label[k];
        D.prim[k] = c->prim[k];
        D.col[k] = m;
        if (D.kind[k] == 0) {
            for (int a = 0; a < 3; ++a) {
                D.nseed[k][a] = S->nrm[3 * (int64_t)c->prim[k] + a];
                z[m + a] = c->v[k][a];
            }
            m += 3;
        } else {
            const or_edge* E = &S->edges[c->prim[k]];
            double ev[3] = {(double)E->b[0] - E->a[0], (double)E->b[1] - E->a[1], (double)E->b[2] - E->a[2]};
            double l = norm(ev);
            for (int a = 0; a < 3; ++a) {
                D.ea[k][a] = E->a[a];
                D.ee[k][a] = ev[a] / l;
            }
            D.elen[k] = l;
            double w[3] = {c->v[k][0] - D.ea[k][0], c->v[k][1] - D.ea[k][1], c->v[k][2] - D.ea[k][2]};
            z[m] = dot(w, D.ee[k]);
            m += 1;
        }
    }
    D.dim = m;
    if (z_out) memcpy(z_out, z, sizeof(double) * m);
    if (z_in) memcpy(z, z_in, sizeof(double) * m);
    int ok = m == 0 ? 1 : residual(&C, &D, z, r_out, NULL, NULL);
    free(C.lab_start);
    free(C.lab_ids);
    return ok ? m : -1;
}

/* pin helper: the Jacobian of or_path_residual's residual (analytic or central differences) */
int or_path_jacobian(const or_scene* S, const or_refine_params* R, const or_coarse* c,
                     const double* z_in, int fd, double h, double* J_out) {
    rctx_t C;
    memset(&C, 0, sizeof(C));
    C.S = S;
    C.R = R;
    C.sigma = R->xi * R->r_s;
    C.rad2 = (4.0 * C.sigma) * (4.0 * C.sigma);
    for (int a = 0; a < 3; ++a) {
        C.tx[a] = R->tx[a];
        C.rx[a] = R->rx[3 * (int64_t)c->rx + a];
    }
    C.lab_start = (int64_t*)calloc(4098, sizeof(int64_t));
    C.lab_ids = (int64_t*)malloc(sizeof(int64_t) * (size_t)(S->n > 0 ? S->n : 1));
    for (int64_t i = 0; i < S->n; ++i) C.lab_start[S->label[i] + 1]++;
    for (int l = 0; l < 4097; ++l) C.lab_start[l + 1] += C.lab_start[l];
    int64_t* fill = (int64_t*)calloc(4097, sizeof(int64_t));
    for (int64_t i = 0; i < S->n; ++i) C.lab_ids[C.lab_start[S->label[i]] + fill[S->label[i]]++] = i;
    free(fill);
    pathdef_t D;
    memset(&D, 0, sizeof(D));
    D.n = c->n_int;
    double z[MAXDIM];
    int m = 0;
    for (int k = 0; k < D.n; ++k) {
        D.kind[k] = (c->kinds >> k) & 1u;
        D.label[k] = c->label[k];
        D.prim[k] = c->prim[k];
        D.col[k] = m;
        if (D.kind[k] == 0) {
            for (int a = 0; a < 3; ++a) {
                D.nseed[k][a] = S->nrm[3 * (int64_t)c->prim[k] + a];
                z[m + a] = c->v[k][a];
            }
            m += 3;
        } else {
            const or_edge* E = &S->edges[c->prim[k]];
            double ev[3] = {(double)E->b[0] - E->a[0], (double)E->b[1] - E->a[1], (double)E->b[2] - E->a[2]};
            double l = norm(ev);
            for (int a = 0; a < 3; ++a) {
                D.ea[k][a] = E->a[a];
                D.ee[k][a] = ev[a] / l;
            }
            D.elen[k] = l;
            double w[3] = {c->v[k][0] - D.ea[k][0], c->v[k][1] - D.ea[k][1], c->v[k][2] - D.ea[k][2]};
            z[m] = dot(w, D.ee[k]);
            m += 1;
        }
    }
    D.dim = m;
    if (z_in) memcpy(z, z_in, sizeof(double) * m);
    int ok = 1;
    if (m > 0 && !fd) ok = jacobian(&C, &D, z, J_out);
    if (m > 0 && fd) {
        double rp[MAXDIM], rm[MAXDIM];
        for (int jj = 0; jj < m && ok; ++jj) {
            double zj = z[jj];
            z[jj] = zj + h;
            ok &= residual(&C, &D, z, rp, NULL, NULL);
            z[jj] = zj - h;
            ok &= residual(&C, &D, z, rm, NULL, NULL);
            z[jj] = zj;
            for (int i = 0; i < m; ++i) J_out[i * m + jj] = (rp[i] - rm[i]) / (2.0 * h);
        }
    }
    free(C.lab_start);
    free(C.lab_ids);
    return ok ? m : -1;
}

/* pin helpers */
int or_mls(const or_scene* S, const or_refine_params* R, int32_t label, const double nseed[3],
           const double x[3], double pbar[3], double nbar[3], double* f) {
    rctx_t C;
    memset(&C, 0, sizeof(C));
    C.S = S;
    C.R = R;
    C.sigma = R->xi * R->r_s;
    C.rad2 = (4.0 * C.sigma) * (4.0 * C.sigma);
    C.lab_start = (int64_t*)calloc(4098, sizeof(int64_t));
    C.lab_ids = (int64_t*)malloc(sizeof(int64_t) * (size_t)(S->n > 0 ? S->n : 1));
    int64_t m = 0;
    for (int64_t i = 0; i < S->n; ++i)
        if (S->label[i] == label) C.lab_ids[m++] = i;
    C.lab_start[label] = 0;
    C.lab_start[label + 1] = m;
    int ok = mls(&C, label, nseed, x, pbar, nbar);
    if (ok) {
        double xp[3] = {x[0] - pbar[0], x[1] - pbar[1], x[2] - pbar[2]};
        *f = dot(xp, nbar);
    }
    free(C.lab_start);
    free(C.lab_ids);
    return ok;
}
