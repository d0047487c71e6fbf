/* grid.c — CPU ORACLE, tier 1: an independent uniform grid for the nearest-hit argmin.
 * TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * the coarse result is defined by the GLOBAL lexicographic argmin over all
 * surfels of (t, id) under the HIT predicate (tier 0 = or_nearest's brute force).  Tier 1
 * computes the same argmin faster so that whole-configuration sets (1e6-1e7 surfels, 1e6-1e8
 * rays) can be produced on the CPU; it is pinned to tier 0 bit for bit on small scenes and
 * must be invariant to the voxel size and the grid origin (tests/test_oracle_grid_pins.py).
 *
 * Why it equals tier 0.  A hit of surfel i at parameter t has its point h = o + t d within
 * r_i of p_i on the disk's plane, up to FP32 rounding (< 1e-5 m at room scale).  Every surfel
 * is registered in each cell overlapped by its disk's axis-aligned box inflated by PAD (1e-4 m
 * + 1e-6 of the scene extent, >> that rounding), so the exact ray point at t lies in a cell
 * where i is registered.  The walk visits the cells the exact ray crosses in increasing t (DDA
 * in FP64) and tests every registered surfel with the tier-0 predicate (the same hit_impl); it
 * stops after a cell only when best_t < t_exit(cell) - PAD: any surfel not tested yet has its
 * point in a later cell, so its t > best_t.  Hence the same (t, id) minimum.
 *
 * Nothing here is shared with the CUDA path: own box, own registration rule (disk box, not
 * the GPU's), own voxel (chosen by the caller, tests use sizes the GPU never does), FP64 walk.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

/* a copy of surfel i's inputs, stored contiguously per cell (memory layout only) */
typedef struct {
    float p[3], n[3], r;
    int32_t pad_;
    int64_t id;
} gref;

struct or_grid {
    double org[3];   /* grid origin (m) */
    double v;        /* voxel edge (m) */
    double pad;      /* registration inflation and stop margin (m) */
    int64_t dims[3];
    int64_t* start;  /* [ncell + 1] CSR offsets */
    gref* ref;       /* surfel copies per cell, ids ascending */
    uint64_t* occ;   /* bit c set <=> cell c is non-empty (a cache-resident copy of start) */
};

int or_hit(const float o[3], const float d[3], const float p[3], const float n[3], float r,
           const float* lam, int n_lam, float tau, float cos_ex, float* t);

/* half extents of disk i's axis-aligned box: r sqrt(1 - nhat_a^2) per axis */
static void disk_box(const or_scene* S, int64_t i, double lo[3], double hi[3], double pad) {
    const float* p = S->p + 3 * i;
    const float* n = S->nrm + 3 * i;
    double nn = (double)n[0] * n[0] + (double)n[1] * n[1] + (double)n[2] * n[2];
    double r = S->r[i];
    for (int a = 0; a < 3; ++a) {
        double c = nn > 0.0 ? ((double)n[a] * n[a]) / nn : 0.0;
        double e = r * sqrt(c < 1.0 ? 1.0 - c : 0.0);
        lo[a] = (double)p[a] - e - pad;
        hi[a] = (double)p[a] + e + pad;
    }
}

or_grid* or_grid_build(const or_scene* S, double voxel, const double shift[3]) {
    if (S->n <= 0 || !(voxel > 0.0)) return NULL;
    double bmin[3] = {INFINITY, INFINITY, INFINITY}, bmax[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = 0; i < S->n; ++i) {
        double lo[3], hi[3];
        disk_box(S, i, lo, hi, 0.0);
        for (int a = 0; a < 3; ++a) {
            if (lo[a] < bmin[a]) bmin[a] = lo[a];
            if (hi[a] > bmax[a]) bmax[a] = hi[a];
        }
    }
    double ext = 0.0;
    for (int a = 0; a < 3; ++a) ext = fmax(ext, fmax(fabs(bmin[a]), fabs(bmax[a])));
    or_grid* G = (or_grid*)calloc(1, sizeof(or_grid));
    G->v = voxel;
    G->pad = 1e-4 + 1e-6 * ext;
    for (int a = 0; a < 3; ++a) {
        /* the shift moves the cell boundaries (taken modulo the voxel: the box always holds
         * every surfel's box) */
        double sh = shift ? fmod(shift[a], voxel) : 0.0;
        if (sh < 0.0) sh += voxel;
        G->org[a] = bmin[a] - 2.0 * G->pad - sh;
        G->dims[a] = (int64_t)ceil((bmax[a] + 2.0 * G->pad - G->org[a]) / voxel) + 1;
    }
    const int64_t nc = G->dims[0] * G->dims[1] * G->dims[2];
    G->start = (int64_t*)calloc((size_t)nc + 1, sizeof(int64_t));
    /* two passes over the surfels: count, then fill (ids ascend within every cell) */
    for (int pass = 0; pass < 2; ++pass) {
        int64_t* fill = NULL;
        if (pass == 1) {
            for (int64_t c = 0; c < nc; ++c) G->start[c + 1] += G->start[c];
            G->ref = (gref*)malloc(sizeof(gref) * (size_t)(G->start[nc] > 0 ? G->start[nc] : 1));
            fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)nc);
            memcpy(fill, G->start, sizeof(int64_t) * (size_t)nc);
        }
        for (int64_t i = 0; i < S->n; ++i) {
            double lo[3], hi[3];
            disk_box(S, i, lo, hi, G->pad);
            int64_t c0[3], c1[3];
            for (int a = 0; a < 3; ++a) {
                c0[a] = (int64_t)floor((lo[a] - G->org[a]) / voxel);
                c1[a] = (int64_t)floor((hi[a] - G->org[a]) / voxel);
                if (c0[a] < 0) c0[a] = 0;
                if (c1[a] > G->dims[a] - 1) c1[a] = G->dims[a] - 1;
            }
            for (int64_t z = c0[2]; z <= c1[2]; ++z)
                for (int64_t y = c0[1]; y <= c1[1]; ++y)
                    for (int64_t x = c0[0]; x <= c1[0]; ++x) {
                        int64_t c = x + G->dims[0] * (y + G->dims[1] * z);
                        if (pass == 0) G->start[c + 1]++;
                        else {
                            gref* g = &G->ref[fill[c]++];
                            for (int a = 0; a < 3; ++a) {
                                g->p[a] = S->p[3 * i + a];
                                g->n[a] = S->nrm[3 * i + a];
                            }
                            g->r = S->r[i];
                            g->pad_ = 0;
                            g->id = i;
                        }
                    }
        }
        free(fill);
    }
    G->occ = (uint64_t*)calloc((size_t)(nc / 64 + 1), sizeof(uint64_t));
    for (int64_t c = 0; c < nc; ++c)
        if (G->start[c + 1] > G->start[c]) G->occ[c >> 6] |= 1ull << (c & 63);
    return G;
}

void or_grid_free(or_grid* G) {
    if (!G) return;
    free(G->start);
    free(G->ref);
    free(G->occ);
    free(G);
}

void or_grid_info(const or_grid* G, int64_t dims[3], int64_t* n_refs, double* pad) {
    for (int a = 0; a < 3; ++a) dims[a] = G->dims[a];
    *n_refs = G->start[G->dims[0] * G->dims[1] * G->dims[2]];
    *pad = G->pad;
}

/* the tier-0 argmin restricted to the surfels registered along the ray (see header) */
int64_t or_grid_nearest(const or_scene* S, const or_grid* G, const float o[3], const float d[3],
                        const float* lam, int n_lam, int64_t prev, float tau, float cos_ex,
                        float* t_hit) {
    int64_t best = -1;
    float bt = INFINITY;
    double od[3] = {o[0], o[1], o[2]}, dd[3] = {d[0], d[1], d[2]};
    /* entry into the grid box (slab test, FP64) */
    double t0 = 0.0, t1 = INFINITY;
    for (int a = 0; a < 3; ++a) {
        double lo = G->org[a], hi = G->org[a] + (double)G->dims[a] * G->v;
        if (dd[a] != 0.0) {
            double ta = (lo - od[a]) / dd[a], tb = (hi - od[a]) / dd[a];
            t0 = fmax(t0, fmin(ta, tb));
            t1 = fmin(t1, fmax(ta, tb));
        } else if (od[a] < lo || od[a] > hi) {
            t1 = -1.0;
        }
    }
    if (t0 > t1) {
        *t_hit = bt;
        return best;
    }
    int64_t c[3];
    double tm[3];
    for (int a = 0; a < 3; ++a) {
        double x = od[a] + t0 * dd[a];
        c[a] = (int64_t)floor((x - G->org[a]) / G->v);
        if (c[a] < 0) c[a] = 0;
        if (c[a] > G->dims[a] - 1) c[a] = G->dims[a] - 1;
        tm[a] = dd[a] != 0.0 ? (G->org[a] + (double)(c[a] + (dd[a] > 0.0)) * G->v - od[a]) / dd[a]
                             : INFINITY;
    }
    for (;;) {
        int64_t cell = c[0] + G->dims[0] * (c[1] + G->dims[1] * c[2]);
        int64_t k0 = 0, k1 = 0;
        if ((G->occ[cell >> 6] >> (cell & 63)) & 1ull) {
            k0 = G->start[cell];
            k1 = G->start[cell + 1];
        }
        for (int64_t k = k0; k < k1; ++k) {
            const gref* g = &G->ref[k];
            int64_t i = g->id;
            if (i == prev) continue;
            float t;
            if (!or_hit(o, d, g->p, g->n, g->r, lam, n_lam, tau, cos_ex, &t)) continue;
            if (t < bt || (t == bt && i < best)) {
                bt = t;
                best = i;
            }
        }
        int ax = 0;
        if (tm[1] < tm[ax]) ax = 1;
        if (tm[2] < tm[ax]) ax = 2;
        if ((double)bt < tm[ax] - G->pad) break;
        c[ax] += dd[ax] > 0.0 ? 1 : -1;
        if (c[ax] < 0 || c[ax] >= G->dims[ax]) break;
        tm[ax] = (G->org[ax] + (double)(c[ax] + (dd[ax] > 0.0)) * G->v - od[ax]) / dd[ax];
    }
    *t_hit = bt;
    return best;
}
