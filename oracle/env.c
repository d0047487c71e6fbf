/* env.c — CPU ORACLE, NEXT-2: the paper's coarse tracer — environment-driven launch and voxel
 * cone tracing.  TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * PAPER §II-B (IEs), §II-D, §III (Alg. 1), Table I;
 * readings R60-R69 of DESIGN.md.  FP32 geometry in the order written here; the SDF
 * intersection (sdf.c, R40-R44) validates every candidate.
 *   R60 voxels of V = 8a and subvoxels of S = 4a from the AABB grid's origin (D_v = 2,
 *       D_sv = 4: a voxel = 2^3 subvoxels = 8^3 AABB cells); IEs: a PCIE per non-empty
 *       subvoxel (reception point = the mean of its points, FP64 sums in id order; label = the
 *       label of the point nearest the subvoxel centre), a DEIE per piece of an edge cut by the
 *       subvoxel planes (reception point = the piece midpoint), an RXIE per RX.  IE order:
 *       PCIEs by subvoxel, DEIEs by (edge, piece), RXIEs by RX.
 *   R61 each voxel lists its IEs; its march distance = the Chebyshev distance (voxels) to the
 *       nearest voxel with IEs, at least 1.  Cone half-angle theta: tan theta = V / D, D = the
 *       diagonal of the points' bounding box.
 *   R62 cone-sphere test: v = c - o, t = v.d; pass iff t >= -r and |v - t d| <= t tan + r sec.
 *   R63 transmission: from the TX toward every IE's reception point, validated (R66).
 *   R64 propagation: march the cone ray's voxels with Alg. 1 from o; where the
 *       voxel holds IEs or its march distance is 1, evaluate its 3x3x3 neighbourhood (z, y, x
 *       ascending) except voxels in the ray's history ring (64 entries): voxel sphere
 *       (centre, V sqrt3/2) vs the cone, then each IE (ascending, not the ray's source IE):
 *       subvoxel sphere (S sqrt3/2) vs the cone and the separation test (reflection: in front
 *       of the reflecting surface; fan ray m: between its two separation planes), except RXIEs
 *       while the path has <= 2 interactions (the voxel test suffices); a candidate is
 *       validated by R66 and, if valid, handled by R65.
 *   R65 valid PCIE -> a reflection at the SDF hit point (label = the PCIE's, id = the hit's
 *       nearest point), a reflected cone ray (if max_refl allows); valid DEIE -> a diffraction
 *       at its reception point and a Keller fan of cone rays (R15 directions, bins between
 *       separation planes, if max_diff allows); valid RXIE -> a path record.
 *   R66 validation: the SDF trace from the source toward the reception point (departure rule
 *       of the source): a PCIE is valid iff the first hit lies in one of its AABBs; a DEIE iff
 *       no hit before its distance - a/2 ("reduce the maximum length by a small bias");
 *       an RXIE iff no hit before its distance.  A PCIE / DEIE the interaction caps would not
 *       let the path take is not validated (no ray is traced for it).
 *   R67 records: key as R17, L = the unfolded length, ray id = FNV-1a of the IE sequence; the
 *       kappa shortest per key (Table I: kappa = 100).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

void or_sdf_geometry(const or_sdf* G, float org[3], float* a, int64_t dims[3]);

enum { IE_PC = 0, IE_DE = 1, IE_RX = 2 };

typedef struct {
    float p[3];
    int32_t kind, label, ref;  /* PCIE: subvoxel index; DEIE: edge; RXIE: rx */
    int64_t sub[3];
    float s_edge;
} ie_t;

struct or_env {
    float org[3], a, V, S, tan_c, sec_c;
    int64_t sd[3], sv[3], vd[3];
    ie_t* ie;
    int64_t n_ie, n_pc;
    int64_t* pc_of_sub;   /* subvoxel -> PCIE index or -1 */
    int64_t* vstart;      /* [n_vox + 1] */
    int64_t* vids;        /* IE indices per voxel, ascending */
    int32_t* march;       /* per voxel, >= 1 */
};

static float dot3(const float a[3], const float b[3]) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }

static int cmp_f(const void* A, const void* B) {
    const float a = *(const float*)A, b = *(const float*)B;
    return a < b ? -1 : a > b;
}

/* R60 + R61 */
or_env* or_env_build(const or_scene* S, const float* rx, int32_t n_rx) {
    const or_sdf* G = S->sdf;
    if (!G) return NULL;
    or_env* E = (or_env*)calloc(1, sizeof(or_env));
    or_sdf_geometry(G, E->org, &E->a, E->sd);
    E->V = 8.0f * E->a;
    E->S = 4.0f * E->a;
    for (int k = 0; k < 3; ++k) {
        E->sv[k] = (E->sd[k] + 3) / 4;
        E->vd[k] = (E->sd[k] + 7) / 8;
    }
    const int64_t nsub = E->sv[0] * E->sv[1] * E->sv[2];
    double* sum = (double*)calloc((size_t)nsub * 3, sizeof(double));
    int64_t* cnt = (int64_t*)calloc((size_t)nsub, sizeof(int64_t));
    float* bq = (float*)malloc(sizeof(float) * (size_t)nsub);
    int32_t* blab = (int32_t*)malloc(sizeof(int32_t) * (size_t)nsub);
    for (int64_t s = 0; s < nsub; ++s) bq[s] = INFINITY;
    float bmin[3], bmax[3];
    for (int k = 0; k < 3; ++k) bmin[k] = bmax[k] = S->p[k];
    for (int64_t i = 0; i < S->n; ++i) {
        const float* p = S->p + 3 * i;
        int64_t sub[3];
        for (int k = 0; k < 3; ++k) {
            int64_t c = (int64_t)floorf((p[k] - E->org[k]) / E->a);
            if (c < 0) c = 0;
            if (c > E->sd[k] - 1) c = E->sd[k] - 1;
            sub[k] = c / 4;
            if (p[k] < bmin[k]) bmin[k] = p[k];
            if (p[k] > bmax[k]) bmax[k] = p[k];
        }
        const int64_t s = sub[0] + E->sv[0] * (sub[1] + E->sv[1] * sub[2]);
        for (int k = 0; k < 3; ++k) sum[3 * s + k] += (double)p[k];
        cnt[s]++;
        float d[3];
        for (int k = 0; k < 3; ++k) d[k] = p[k] - (E->org[k] + ((float)sub[k] + 0.5f) * E->S);
        const float q = dot3(d, d);
        if (q < bq[s]) {
            bq[s] = q;
            blab[s] = S->label[i];
        }
    }
    /* edges: pieces between the subvoxel planes */
    int64_t n_de = 0, cap_de = 64;
    ie_t* de = (ie_t*)malloc(sizeof(ie_t) * (size_t)cap_de);
    for (int32_t j = 0; j < S->n_edges; ++j) {
        const or_edge* Ed = &S->edges[j];
        float ev[3] = {Ed->b[0] - Ed->a[0], Ed->b[1] - Ed->a[1], Ed->b[2] - Ed->a[2]};
        const float len = sqrtf(dot3(ev, ev));
        float ts[4096];
        int nt = 0;
        ts[nt++] = 0.0f;
        for (int k = 0; k < 3; ++k) {
            if (ev[k] == 0.0f) continue;
            const float lo = fminf(Ed->a[k], Ed->b[k]), hi = fmaxf(Ed->a[k], Ed->b[k]);
            const int64_t m0 = (int64_t)floorf((lo - E->org[k]) / E->S), m1 = (int64_t)floorf((hi - E->org[k]) / E->S) + 1;
            for (int64_t m = m0; m <= m1 && nt < 4094; ++m) {
                const float t = ((E->org[k] + (float)m * E->S) - Ed->a[k]) / ev[k];
                if (t > 0.0f && t < 1.0f) ts[nt++] = t;
            }
        }
        ts[nt++] = 1.0f;
        qsort(ts, (size_t)nt, sizeof(float), cmp_f);
        for (int q = 0; q + 1 < nt; ++q) {
            if (!(ts[q + 1] > ts[q])) continue;
            const float tm = 0.5f * (ts[q] + ts[q + 1]);
            ie_t I;
            memset(&I, 0, sizeof(I));
            for (int k = 0; k < 3; ++k) I.p[k] = Ed->a[k] + tm * ev[k];
            I.kind = IE_DE;
            I.label = Ed->label;
            I.ref = j;
            I.s_edge = tm * len;
            if (n_de == cap_de) {
                cap_de *= 2;
                de = (ie_t*)realloc(de, sizeof(ie_t) * (size_t)cap_de);
            }
            de[n_de++] = I;
        }
    }
    int64_t n_pc = 0;
    for (int64_t s = 0; s < nsub; ++s) n_pc += cnt[s] > 0;
    E->n_pc = n_pc;
    E->n_ie = n_pc + n_de + n_rx;
    E->ie = (ie_t*)calloc((size_t)(E->n_ie > 0 ? E->n_ie : 1), sizeof(ie_t));
    E->pc_of_sub = (int64_t*)malloc(sizeof(int64_t) * (size_t)nsub);
    int64_t q = 0;
    for (int64_t s = 0; s < nsub; ++s) {
        E->pc_of_sub[s] = -1;
        if (!cnt[s]) continue;
        ie_t* I = &E->ie[q];
        for (int k = 0; k < 3; ++k) I->p[k] = (float)(sum[3 * s + k] / (double)cnt[s]);
        I->kind = IE_PC;
        I->label = blab[s];
        I->ref = (int32_t)s;
        I->sub[0] = s % E->sv[0];
        I->sub[1] = (s / E->sv[0]) % E->sv[1];
        I->sub[2] = s / (E->sv[0] * E->sv[1]);
        E->pc_of_sub[s] = q++;
    }
    for (int64_t j = 0; j < n_de; ++j) E->ie[q++] = de[j];
    for (int32_t j = 0; j < n_rx; ++j) {
        ie_t* I = &E->ie[q++];
        for (int k = 0; k < 3; ++k) I->p[k] = rx[3 * j + k];
        I->kind = IE_RX;
        I->label = j;
        I->ref = j;
    }
    for (int64_t i = n_pc; i < E->n_ie; ++i) /* DEIE / RXIE subvoxels */
        for (int k = 0; k < 3; ++k) {
            int64_t c = (int64_t)floorf((E->ie[i].p[k] - E->org[k]) / E->S);
            if (c < 0) c = 0;
            if (c > E->sv[k] - 1) c = E->sv[k] - 1;
            E->ie[i].sub[k] = c;
        }
    free(sum);
    free(cnt);
    free(bq);
    free(blab);
    free(de);
    /* R61: voxel lists, march distances, cone */
    const int64_t nv = E->vd[0] * E->vd[1] * E->vd[2];
    E->vstart = (int64_t*)calloc((size_t)nv + 1, sizeof(int64_t));
    E->vids = (int64_t*)malloc(sizeof(int64_t) * (size_t)(E->n_ie > 0 ? E->n_ie : 1));
    int64_t* vox = (int64_t*)malloc(sizeof(int64_t) * (size_t)(E->n_ie > 0 ? E->n_ie : 1));
    for (int64_t i = 0; i < E->n_ie; ++i) {
        int64_t v3[3];
        for (int k = 0; k < 3; ++k) {
            v3[k] = E->ie[i].sub[k] / 2;
            if (v3[k] > E->vd[k] - 1) v3[k] = E->vd[k] - 1;
        }
        vox[i] = v3[0] + E->vd[0] * (v3[1] + E->vd[1] * v3[2]);
        E->vstart[vox[i] + 1]++;
    }
    for (int64_t v = 0; v < nv; ++v) E->vstart[v + 1] += E->vstart[v];
    int64_t* fill = (int64_t*)calloc((size_t)nv, sizeof(int64_t));
    for (int64_t i = 0; i < E->n_ie; ++i) E->vids[E->vstart[vox[i]] + fill[vox[i]]++] = i;
    free(fill);
    free(vox);
    E->march = (int32_t*)malloc(sizeof(int32_t) * (size_t)nv);
    for (int64_t v = 0; v < nv; ++v) {
        const int64_t x = v % E->vd[0], y = (v / E->vd[0]) % E->vd[1], z = v / (E->vd[0] * E->vd[1]);
        int64_t best = 1 << 20;
        for (int64_t u = 0; u < nv; ++u) {
            if (E->vstart[u + 1] == E->vstart[u]) continue;
            const int64_t ux = u % E->vd[0], uy = (u / E->vd[0]) % E->vd[1], uz = u / (E->vd[0] * E->vd[1]);
            int64_t dd = llabs(ux - x);
            if (llabs(uy - y) > dd) dd = llabs(uy - y);
            if (llabs(uz - z) > dd) dd = llabs(uz - z);
            if (dd < best) best = dd;
        }
        E->march[v] = (int32_t)(best < 1 ? 1 : best);
    }
    float dg[3] = {bmax[0] - bmin[0], bmax[1] - bmin[1], bmax[2] - bmin[2]};
    const float D = sqrtf(dot3(dg, dg));
    E->tan_c = E->V / D;
    E->sec_c = sqrtf(1.0f + E->tan_c * E->tan_c);
    return E;
}

void or_env_free(or_env* E) {
    if (!E) return;
    free(E->ie);
    free(E->pc_of_sub);
    free(E->vstart);
    free(E->vids);
    free(E->march);
    free(E);
}

/* pin helpers */
int64_t or_env_count(const or_env* E, int64_t* n_pc) {
    *n_pc = E->n_pc;
    return E->n_ie;
}
void or_env_ie(const or_env* E, int64_t i, float p[3], int32_t* kind, int32_t* label, int64_t* voxel) {
    for (int k = 0; k < 3; ++k) p[k] = E->ie[i].p[k];
    *kind = E->ie[i].kind;
    *label = E->ie[i].label;
    int64_t v3[3];
    for (int k = 0; k < 3; ++k) {
        v3[k] = E->ie[i].sub[k] / 2;
        if (v3[k] > E->vd[k] - 1) v3[k] = E->vd[k] - 1;
    }
    *voxel = v3[0] + E->vd[0] * (v3[1] + E->vd[1] * v3[2]);
}
void or_env_grid(const or_env* E, int64_t vd[3], float* V, float* tan_c, const int32_t** march) {
    for (int k = 0; k < 3; ++k) vd[k] = E->vd[k];
    *V = E->V;
    *tan_c = E->tan_c;
    *march = E->march;
}

/* Alg. 1: one march of a_dist voxels from vpos along dir (voxel space) */
void or_env_march(const float vpos[3], const float dir[3], int32_t a_dist, float out[3]) {
    float T[3];
    for (int k = 0; k < 3; ++k) {
        const float C = floorf(vpos[k]);
        const float L = dir[k] >= 0.0f ? 1.0f : 0.0f;
        const float su = 1.0f / fmaxf(fabsf(dir[k]), 1e-16f);
        const float dn = fabsf(L - (vpos[k] - C));
        T[k] = dn * su + su * (float)(a_dist - 1);
    }
    float st;
    if (T[0] <= T[1] && T[0] <= T[2]) st = T[0];
    else if (T[1] < T[0] && T[1] <= T[2]) st = T[1];
    else st = T[2];
    st = st + 1e-2f;
    for (int k = 0; k < 3; ++k) out[k] = vpos[k] + dir[k] * st;
}

/* R62 */
int or_env_cone_sphere(const float o[3], const float d[3], float tan_c, float sec_c, const float c[3], float r) {
    float v[3] = {c[0] - o[0], c[1] - o[1], c[2] - o[2]};
    const float t = dot3(v, d);
    if (t < -r) return 0;
    float w[3] = {v[0] - t * d[0], v[1] - t * d[1], v[2] - t * d[2]};
    return sqrtf(dot3(w, w)) <= t * tan_c + r * sec_c;
}

/* ------------------------------------------------------------------------------------ */
typedef struct {
    const or_scene* S;
    const or_launch_params* P;
    const or_env* E;
    float cos_ex;
    or_coarse* raw;
    int64_t cap, n;
    uint64_t rays;
} ectx;

typedef struct {
    int32_t n, n_diff, n_refl;
    uint16_t kinds;
    int32_t label[OR_MAX_INT];
    uint32_t prim[OR_MAX_INT];
    float v[OR_MAX_INT][3];
    float s_edge;
    uint64_t hash;
} ehist;

typedef struct {
    float o[3], d[3];
    int kind;            /* 0 reflection, 1 fan ray */
    float nf[3];         /* reflection: the surface normal oriented to the reflected side */
    float nlo[3], nhi[3];/* fan ray: inward normals of its separation planes */
    float lam[6];
    int n_lam;
    int64_t prev_cell;
    int64_t src;         /* the IE the ray leaves */
    float L;
} cray;

static uint64_t mix(uint64_t h, uint64_t v) { return (h ^ v) * 1099511628211ull; }

static void emit(ectx* C, const ehist* h, int32_t rx, float L) {
    if (C->n < C->cap) {
        or_coarse* c = &C->raw[C->n];
        memset(c, 0, sizeof(*c));
        c->rx = (uint32_t)rx;
        c->n_int = (uint8_t)h->n;
        c->n_diff = (uint8_t)h->n_diff;
        c->kinds = h->kinds;
        for (int k = 0; k < h->n; ++k) {
            c->label[k] = h->label[k];
            c->prim[k] = h->prim[k];
            for (int a = 0; a < 3; ++a) c->v[k][a] = h->v[k][a];
        }
        c->s_edge = h->s_edge;
        c->L = L;
        c->ray_id = mix(h->hash, (1ull << 62) | (uint64_t)rx) & ~(1ull << 63);
    }
    C->n++;
}

static void propagate(ectx* C, const cray* R, const ehist* h);

/* R66 validation of IE i from source (o, lam, prev); R65 handling.  L0 = length so far. */
static void try_ie(ectx* C, const ehist* h, const float o[3], const float* lam, int n_lam, int64_t prev,
                   int64_t i, float L0) {
    const or_env* E = C->E;
    const ie_t* I = &E->ie[i];
    /* R66: an interaction the caps do not allow is not validated (it could not extend the path) */
    if (I->kind == IE_PC && (h->n_refl >= C->P->max_refl || h->n >= OR_MAX_INT)) return;
    if (I->kind == IE_DE && (h->n_diff >= C->P->max_diff || h->n >= OR_MAX_INT)) return;
    float dv[3] = {I->p[0] - o[0], I->p[1] - o[1], I->p[2] - o[2]};
    const float Ls = sqrtf(dot3(dv, dv));
    if (!(Ls > 0.0f)) return;
    float d[3] = {dv[0] / Ls, dv[1] / Ls, dv[2] / Ls};
    float t, nh[3];
    int64_t cell;
    C->rays++;
    const int64_t pid = or_sdf_nearest(C->S, C->S->sdf, &C->P->sdf, o, d, lam, n_lam, prev, C->P->tau, C->cos_ex,
                                       &t, &cell, nh);
    const or_launch_params* P = C->P;
    if (I->kind == IE_RX) {
        if (pid >= 0 && t < Ls) return;
        emit(C, h, I->ref, L0 + Ls);
        return;
    }
    if (I->kind == IE_DE) {
        if (pid >= 0 && t < Ls - 0.5f * E->a) return;
        if (h->n_diff >= P->max_diff || h->n >= OR_MAX_INT) return;
        const or_edge* Ed = &C->S->edges[I->ref];
        float ev[3] = {Ed->b[0] - Ed->a[0], Ed->b[1] - Ed->a[1], Ed->b[2] - Ed->a[2]};
        const float len = sqrtf(dot3(ev, ev));
        const float e[3] = {ev[0] / len, ev[1] / len, ev[2] / len};
        ehist hh = *h;
        hh.label[hh.n] = I->label;
        hh.prim[hh.n] = (uint32_t)I->ref;
        for (int a = 0; a < 3; ++a) hh.v[hh.n][a] = I->p[a];
        hh.kinds = (uint16_t)(hh.kinds | (1u << hh.n));
        hh.n++;
        hh.n_diff++;
        hh.s_edge = I->s_edge;
        /* R15 fan of incident d at the reception point */
        double ct = (double)dot3(d, e);
        double st = sqrt(fmax(0.0, 1.0 - ct * ct));
        if (st < 1e-6) return;
        int M0 = (int)ceil((double)Ed->n_exp * 180.0 / (double)P->dphi_deg);
        int M = (int)ceil((double)M0 * st);
        if (M < 1) M = 1;
        double wedge = (double)Ed->n_exp * 3.14159265358979311600;
        cray R;
        memset(&R, 0, sizeof(R));
        R.kind = 1;
        for (int a = 0; a < 3; ++a) {
            R.o[a] = I->p[a];
            R.lam[a] = Ed->n0[a];
            R.lam[3 + a] = Ed->n1[a];
        }
        R.n_lam = 2;
        R.prev_cell = -1;
        R.src = i;
        R.L = L0 + Ls;
        for (int m = 0; m < M; ++m) {
            double phi = (((double)m + 0.5) * wedge) / (double)M;
            double sp, cp, sl, cl, sh, ch;
            or_sincos(phi, &sp, &cp);
            or_sincos(((double)m * wedge) / (double)M, &sl, &cl);
            or_sincos((((double)m + 1.0) * wedge) / (double)M, &sh, &ch);
            for (int k = 0; k < 3; ++k) {
                double x2 = cp * (double)Ed->t0[k] + sp * (double)Ed->n0[k];
                R.d[k] = (float)(x2 * st + (double)e[k] * ct);
                R.nlo[k] = (float)(-sl * (double)Ed->t0[k] + cl * (double)Ed->n0[k]);
                R.nhi[k] = (float)(sh * (double)Ed->t0[k] - ch * (double)Ed->n0[k]);
            }
            ehist hm = hh;
            hm.hash = mix(h->hash, ((uint64_t)i << 12) | (uint64_t)(m + 1));
            propagate(C, &R, &hm);
        }
        return;
    }
    /* PCIE: the first hit must lie in one of its AABBs */
    if (pid < 0) return;
    {
        int64_t c3[3] = {cell % E->sd[0], (cell / E->sd[0]) % E->sd[1], cell / (E->sd[0] * E->sd[1])};
        const int64_t s = c3[0] / 4 + E->sv[0] * (c3[1] / 4 + E->sv[1] * (c3[2] / 4));
        if (E->pc_of_sub[s] != i) return;
    }
    if (h->n_refl >= P->max_refl || h->n >= OR_MAX_INT) return;
    float x[3] = {o[0] + t * d[0], o[1] + t * d[1], o[2] + t * d[2]};
    ehist hh = *h;
    hh.label[hh.n] = I->label;
    hh.prim[hh.n] = (uint32_t)pid;
    for (int a = 0; a < 3; ++a) hh.v[hh.n][a] = x[a];
    hh.n++;
    hh.n_refl++;
    hh.hash = mix(h->hash, (uint64_t)i << 12);
    cray R;
    memset(&R, 0, sizeof(R));
    R.kind = 0;
    for (int a = 0; a < 3; ++a) R.o[a] = x[a];
    or_reflect(d, nh, R.d);
    const float s = dot3(R.d, nh) >= 0.0f ? 1.0f : -1.0f;
    for (int a = 0; a < 3; ++a) {
        R.nf[a] = s * nh[a];
        R.lam[a] = nh[a];
    }
    R.n_lam = 1;
    R.prev_cell = cell;
    R.src = i;
    R.L = L0 + Ls;
    propagate(C, &R, &hh);
}

/* R64: one cone ray */
static void propagate(ectx* C, const cray* R, const ehist* h) {
    const or_env* E = C->E;
    int64_t ring[64];
    int nring = 0, head = 0;
    float vpos[3];
    for (int k = 0; k < 3; ++k) vpos[k] = (R->o[k] - E->org[k]) / E->V;
    const float rv = E->V * 0.8660254f, rs = E->S * 0.8660254f;
    for (int it = 0; it < 1 << 16; ++it) {
        int64_t c[3];
        int out = 0;
        for (int k = 0; k < 3; ++k) {
            c[k] = (int64_t)floorf(vpos[k]);
            out |= c[k] < 0 || c[k] >= E->vd[k];
        }
        if (out) break;
        const int64_t cv = c[0] + E->vd[0] * (c[1] + E->vd[1] * c[2]);
        const int32_t a = E->march[cv];
        if (E->vstart[cv + 1] > E->vstart[cv] || a == 1) {
            for (int64_t dz = -1; dz <= 1; ++dz)
                for (int64_t dy = -1; dy <= 1; ++dy)
                    for (int64_t dx = -1; dx <= 1; ++dx) {
                        const int64_t q3[3] = {c[0] + dx, c[1] + dy, c[2] + dz};
                        if (q3[0] < 0 || q3[0] >= E->vd[0] || q3[1] < 0 || q3[1] >= E->vd[1] || q3[2] < 0 ||
                            q3[2] >= E->vd[2])
                            continue;
                        const int64_t q = q3[0] + E->vd[0] * (q3[1] + E->vd[1] * q3[2]);
                        int seen = 0;
                        for (int r = 0; r < nring; ++r) seen |= ring[r] == q;
                        if (seen) continue;
                        ring[head] = q;
                        head = (head + 1) & 63;
                        if (nring < 64) nring++;
                        if (E->vstart[q + 1] == E->vstart[q]) continue;
                        float cq[3];
                        for (int k = 0; k < 3; ++k) cq[k] = E->org[k] + ((float)q3[k] + 0.5f) * E->V;
                        if (!or_env_cone_sphere(R->o, R->d, E->tan_c, E->sec_c, cq, rv)) continue;
                        for (int64_t u = E->vstart[q]; u < E->vstart[q + 1]; ++u) {
                            const int64_t i = E->vids[u];
                            if (i == R->src) continue;
                            const ie_t* I = &E->ie[i];
                            if (!(I->kind == IE_RX && h->n <= 2)) {
                                float cs[3];
                                for (int k = 0; k < 3; ++k) cs[k] = E->org[k] + ((float)I->sub[k] + 0.5f) * E->S;
                                if (!or_env_cone_sphere(R->o, R->d, E->tan_c, E->sec_c, cs, rs)) continue;
                                float w[3] = {I->p[0] - R->o[0], I->p[1] - R->o[1], I->p[2] - R->o[2]};
                                if (R->kind == 0) {
                                    if (!(dot3(w, R->nf) > 0.0f)) continue;
                                } else if (!(dot3(w, R->nlo) >= 0.0f && dot3(w, R->nhi) >= 0.0f)) {
                                    continue;
                                }
                            }
                            try_ie(C, h, R->o, R->lam, R->n_lam, R->prev_cell, i, R->L);
                        }
                    }
        }
        float nv[3];
        or_env_march(vpos, R->d, a, nv);
        for (int k = 0; k < 3; ++k) vpos[k] = nv[k];
    }
}

/* R63: transmission from the TX to IEs i == part (mod parts), with their propagation */
int or_env_launch(const or_scene* S, const or_launch_params* P, const or_env* E, int32_t part, int32_t parts,
                  or_coarse* raw, int64_t raw_cap, int64_t* n_raw, uint64_t* n_rays) {
    ectx C;
    memset(&C, 0, sizeof(C));
    C.S = S;
    C.P = P;
    C.E = E;
    C.cos_ex = or_cos_ex(P->theta_ex_deg);
    C.raw = raw;
    C.cap = raw_cap;
    ehist h0;
    memset(&h0, 0, sizeof(h0));
    h0.hash = 14695981039346656037ull;
    for (int64_t i = part; i < E->n_ie; i += parts)
        try_ie(&C, &h0, P->tx, NULL, 0, -1, i, 0.0f);
    *n_raw = C.n;
    *n_rays = C.rays;
    return C.n > raw_cap ? 4 : 0;
}
