/* oracle.h — CPU ORACLE for arXiv 2403.06648's hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load this library.  It shares no code, header, constant table or helper with
 * the CUDA path (paper_2403_06648_b200/csrc); both are written from PAPER.md and the
 * readings R1-R32 listed in DESIGN.md.
 *
 * Coarse part (FP32, compiled with -ffp-contract=off, no fast-math): the plain
 * definition of SURVEY §8(c) C.1 — at every segment the hit is the GLOBAL lexicographic
 * argmin over ALL surfels of (t, id) under the HIT predicate (brute force; no grid).
 * Refinement part (FP64, refine.c): damped Gauss-Newton on the stationarity residual
 * of Eqs. 9-11 with the Eq. 1-4 MLS surface.
 */
#ifndef NRT_ORACLE_H
#define NRT_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OR_MAX_INT 8

typedef struct {
    float a[3], b[3];   /* edge segment endpoints (m) */
    float t0[3];        /* face-0 tangent, perpendicular to e, pointing into face 0 */
    float n0[3];        /* face-0 outward normal */
    float n1[3];        /* face-1 outward normal */
    float n_exp;        /* exterior angle = n_exp * pi, 1 < n_exp < 2 */
    int32_t label;      /* unique edge label */
} or_edge;

typedef struct or_grid or_grid;  /* tier-1 uniform grid (grid.c); NULL = brute force */
typedef struct or_sdf or_sdf;    /* NEXT-1 AABB primitives of the SDF intersection (sdf.c) */

/* NEXT-1 SDF intersection parameters (R40-R45) */
typedef struct {
    float cell;    /* AABB cell edge a (m); 0 = the disk intersection (R7) */
    float r_s;     /* sample radius (coarse tracing: 0.015, Table II) */
    float t_sdf;   /* hit threshold (coarse tracing: 0.0015, Table II) */
    float xi;      /* sigma = xi r_s (Table I: 2) */
} or_sdf_params;

typedef struct {
    const float* p;        /* n x 3 positions */
    const float* nrm;      /* n x 3 normals (as given) */
    const float* r;        /* n radii */
    const int32_t* label;  /* n labels, 0 <= label < 4096 */
    int64_t n;
    const or_edge* edges;
    int32_t n_edges;
    const or_grid* grid;   /* optional tier-1 grid: same argmin, faster */
    const or_sdf* sdf;     /* AABB primitives for the SDF intersection (launch sdf.cell > 0) */
} or_scene;

typedef struct {
    float tx[3];
    const float* rx;       /* n_rx x 3 */
    int32_t n_rx;
    int64_t n_rays;        /* N of the Fibonacci lattice (global) */
    int32_t max_refl, max_diff;
    int32_t kappa;
    float tau;             /* departure-sheet noise tolerance (R8) */
    float c_R;             /* reception-sphere scale (R12) */
    float dphi_deg;        /* Keller fan step (R15) */
    float theta_ex_deg;    /* departure-sheet angle (R8) */
    float edge_bin;        /* event s-bin (R14) */
    int32_t rank, world;   /* ray shard i == rank (mod world) */
    or_sdf_params sdf;     /* NEXT-1: cell > 0 selects the SDF intersection */
} or_launch_params;

/* coarse path record (R17 key + representative) */
typedef struct {
    uint32_t rx;
    uint8_t n_int, n_diff;
    uint16_t kinds;                 /* bit k set <=> interaction k is a diffraction */
    int32_t label[OR_MAX_INT];      /* surfel label or edge label; 0 beyond n_int */
    uint32_t prim[OR_MAX_INT];      /* surfel id or edge id; 0 beyond n_int */
    float v[OR_MAX_INT][3];         /* interaction points; 0 beyond n_int */
    float s_edge;                   /* edge parameter of the diffraction (0 if none) */
    float L;                        /* unfolded length at the RX closest approach */
    uint64_t ray_id;
} or_coarse;

/* interaction history of a ray (internal state, also carried by events) */
typedef struct {
    int32_t n;                      /* interactions so far */
    int32_t n_diff;
    uint16_t kinds;
    uint16_t pad_;
    int32_t label[OR_MAX_INT];
    uint32_t prim[OR_MAX_INT];
    float v[OR_MAX_INT][3];
    float s_edge;
} or_hist;

/* diffraction event (R13/R14) */
typedef struct {
    or_hist h;
    uint32_t edge;
    int32_t sbin;
    float s;
    float d[3];
    float L;        /* unfolded length at the edge point */
    float dist2;
    uint64_t ray_id;
} or_event;

/* ---- building blocks exposed for the pin tests ---- */
void or_sincos(double x, double* s, double* c);
void or_fib_dir(uint64_t i, uint64_t n, float d[3]);
float or_cos_ex(float theta_ex_deg);
float or_cRw(float c_R, int64_t n_rays);
/* HIT predicate R7-R8 for one surfel; returns 1 and writes *t on hit */
int or_hit(const float o[3], const float d[3], const float p[3], const float n[3], float r,
           const float* lam, int n_lam, float tau, float cos_ex, float* t);
void or_reflect(const float d[3], const float n[3], float out[3]);
/* brute-force nearest hit; returns surfel id or -1 (escape) */
int64_t or_nearest(const or_scene* S, const float o[3], const float d[3], const float* lam,
                   int n_lam, int64_t prev, float tau, float cos_ex, float* t_hit);

/* tier 1 (grid.c): independent uniform grid of cell size `voxel`, origin shifted by `shift`
 * (may be NULL); or_nearest uses it when S->grid is set.  Pinned to tier 0 bit for bit. */
or_grid* or_grid_build(const or_scene* S, double voxel, const double shift[3]);
void or_grid_free(or_grid* G);
void or_grid_info(const or_grid* G, int64_t dims[3], int64_t* n_refs, double* pad);
int64_t or_grid_nearest(const or_scene* S, const or_grid* G, const float o[3], const float d[3],
                        const float* lam, int n_lam, int64_t prev, float tau, float cos_ex,
                        float* t_hit);

/* NEXT-1 (sdf.c): AABB primitives of cell edge a; the SDF intersection tier 0 */
or_sdf* or_sdf_build(const or_scene* S, float a);
void or_sdf_free(or_sdf* G);
int64_t or_sdf_count(const or_sdf* G);
void or_sdf_aabb(const or_sdf* G, int64_t j, float lo[3], float hi[3], int64_t* cell, int64_t* n_pts);
float or_sdf_expf(float x);
int or_sdf_eval(const or_scene* S, const or_sdf* G, int64_t j, const float x[3], float sigma, float* f,
                float nbar[3]);
/* tier 1 for the SDF intersection: a uniform grid (edge `voxel`) over the AABBs; afterwards
 * or_sdf_nearest walks it (same argmin as tier 0, pinned) */
void or_sdf_grid_build(or_sdf* G, double voxel);
/* nearest SDF hit of (o, d): returns the record's surfel id (-1: escape), *t_out, the hit
 * AABB's cell (for the departure rule of the next segment) and the unit hit normal */
int64_t or_sdf_nearest(const or_scene* S, const or_sdf* G, const or_sdf_params* Q, const float o[3],
                       const float d[3], const float* lam, int n_lam, int64_t prev_cell, float tau,
                       float cos_ex, float* t_out, int64_t* cell_out, float n_out[3]);

/* R13 closest approach of ray (o,d) to edge E; 0 if parallel */
int or_edge_closest(const float o[3], const float d[3], const or_edge* E, float* te, float* s,
                    float* dist2);
/* R15 Keller fan directions (Eq. 14) for incident d; returns M (writes min(M,cap)) */
int or_fan_dirs(const or_edge* E, const float d[3], float dphi_deg, float* out, int cap);

/* ---- the coarse operation ---- */
/* Trace the rays of the shard (all diffraction handled inside), dedupe (R17).
 * raw/out are caller buffers; returns 0 ok, 4 overflow (sizes still reported). */
int or_launch(const or_scene* S, const or_launch_params* P, or_coarse* raw, int64_t raw_cap,
              int64_t* n_raw, or_coarse* out, int64_t out_cap, int64_t* n_out,
              uint64_t* n_bounces);
/* The same operation in phases (so tests may run shards in parallel processes):
 * primary rays i == P->rank (mod P->world) -> raw records + raw events;
 * event dedupe (sorted by key, min (dist2, ray id) kept; returns count);
 * fans of events r == part (mod parts), r = global event rank. */
int or_trace_primary(const or_scene* S, const or_launch_params* P, or_coarse* raw,
                     int64_t raw_cap, int64_t* n_raw, or_event* ev, int64_t ev_cap,
                     int64_t* n_ev, uint64_t* n_bounces);
int64_t or_event_dedupe(or_event* ev, int64_t n);
int or_trace_fans(const or_scene* S, const or_launch_params* P, const or_event* ev, int64_t n_ev,
                  int32_t part, int32_t parts, or_coarse* raw, int64_t raw_cap, int64_t* n_raw,
                  uint64_t* n_bounces);
/* Trace only primary rays with ids ray_ids[0..n) (sampled parity / cpu baseline).
 * Emits raw (not deduped) records; hit_ids (n x (max_refl+1)) gets the per-segment surfel
 * id or -1 (escape) or -2 (not traced).  Diffraction events are not followed. */
int or_trace_rays(const or_scene* S, const or_launch_params* P, const uint64_t* ray_ids,
                  int64_t n, or_coarse* raw, int64_t raw_cap, int64_t* n_raw, int64_t* hit_ids,
                  uint64_t* n_bounces);
/* R17 dedupe of an arbitrary record array (sort by key, L, ray id; keep first kappa) */
int64_t or_dedupe(or_coarse* recs, int64_t n, int32_t kappa);

/* ---- refinement (refine.c, FP64) ---- */
enum { NRT_OR_OK = 0, NRT_OR_NO_CONVERGE = 1, NRT_OR_OFF_EDGE = 2, NRT_OR_NO_SUPPORT = 3,
       NRT_OR_WRONG_SIDE = 4, NRT_OR_OCCLUDED = 5, NRT_OR_DEGENERATE = 6 };

typedef struct {
    double xi, r_s;        /* sigma = xi * r_s */
    double tol_m;          /* converged when the GN step |D|_inf < tol_m */
    int32_t max_iter;
    double alpha, beta;    /* Eq. 12 backtracking */
    double tau;            /* support / sheet tolerance (R25) */
    double theta_ex_deg;   /* sheet angle for the shadow rays */
    float tx[3];
    const float* rx;       /* RX table indexed by the record's rx */
    int32_t jac_fd;        /* 0: analytic Jacobian (R37, default); 1: central differences */
} or_refine_params;

typedef struct {
    uint32_t rx;
    uint8_t n_int, n_diff;
    uint16_t kinds;
    int32_t label[OR_MAX_INT];
    uint32_t prim[OR_MAX_INT];
    double v[OR_MAX_INT][3];
    double L, delay;
    float aod_az, aod_el, aoa_az, aoa_el;
    float inc[OR_MAX_INT];
    int32_t status, iters;
    double resid, gradsq;
    uint64_t ray_id;
} or_refined;

/* refine every coarse record (out[q] for in[q], no dedupe; status per path) */
int or_refine(const or_scene* S, const or_refine_params* R, const or_coarse* in, int64_t n,
              or_refined* out);
/* 1 (default): or_refine finds MLS neighbourhoods through a cell index (same ids, same
 * order, bitwise the same sums); 0: the plain label-list loop (pin tests compare both) */
void or_refine_set_grid(int on);
/* residual of record c at its seed (z_in NULL) or at z_in; returns dim or -1 (pin helper) */
int or_path_residual(const or_scene* S, const or_refine_params* R, const or_coarse* c,
                     const double* z_in, double* r_out, double* z_out);
/* Jacobian dr/dz (m x m, row-major) of record c at its seed (z_in NULL) or at z_in, analytic
 * (fd = 0) or by central differences with step h (fd = 1); returns dim or -1 (pin helper) */
int or_path_jacobian(const or_scene* S, const or_refine_params* R, const or_coarse* c,
                     const double* z_in, int fd, double h, double* J_out);
/* Eqs. 1-4 at x over the label's surfels within 4 sigma (pin helper); 0 if empty */
int or_mls(const or_scene* S, const or_refine_params* R, int32_t label, const double nseed[3],
           const double x[3], double pbar[3], double nbar[3], double* f);

/* ---- NEXT-4 (gd.c): the paper's gradient-descent refinement, FP32 (R50-R56) ---- */
typedef struct {
    or_sdf_params sdf;     /* reprojection tracing: cell = the scene's AABB edge; r_s, t_sdf of
                              Table II's refinement rows; xi (sigma = xi r_s also for R53) */
    int32_t rho;           /* iterations (Table I: 2000) */
    float alpha, beta;     /* Eq. 12 line search (Table I: 0.4, 0.4) */
    float delta;           /* ||grad f||^2 < delta (Table I: 1e-4) */
    float t_d, t_a_deg;    /* Table III thresholds */
    float tau, theta_ex_deg; /* departure rule of the traces (R43) */
    float tx[3];
    const float* rx;       /* RX table indexed by the record's rx */
} or_gd_params;
/* refine every coarse record (out[q] for in[q], no dedupe); needs S->sdf; 2 if missing */
int or_refine_gd(const or_scene* S, const or_gd_params* Q, const or_coarse* in, int64_t n,
                 or_refined* out);
void or_gd_basis(const float n[3], float u[3], float v[3]);
float or_gd_line_search(const float x[3], const float P[3], const float Q3[3], const float u[3],
                        const float v[3], int diffraction, float alpha, float beta, float y[3]);
int64_t or_sdf_cell_of(const or_scene* S, const or_sdf* G, int64_t id);
int or_sdf_normal27(const or_scene* S, const or_sdf* G, int64_t cell, const float x[3], float sigma,
                    float n_out[3]);

/* ---- NEXT-2 (env.c): environment-driven launch + voxel cone tracing (R60-R67) ---- */
typedef struct or_env or_env;
or_env* or_env_build(const or_scene* S, const float* rx, int32_t n_rx);  /* needs S->sdf */
void or_env_free(or_env* E);
int64_t or_env_count(const or_env* E, int64_t* n_pc);
void or_env_ie(const or_env* E, int64_t i, float p[3], int32_t* kind, int32_t* label, int64_t* voxel);
void or_env_grid(const or_env* E, int64_t vd[3], float* V, float* tan_c, const int32_t** march);
void or_env_march(const float vpos[3], const float dir[3], int32_t a_dist, float out[3]);
int or_env_cone_sphere(const float o[3], const float d[3], float tan_c, float sec_c, const float c[3], float r);
/* transmission to IEs i == part (mod parts) + their propagation; raw records (not deduped) */
int or_env_launch(const or_scene* S, const or_launch_params* P, const or_env* E, int32_t part, int32_t parts,
                  or_coarse* raw, int64_t raw_cap, int64_t* n_raw, uint64_t* n_rays);

/* refined-path post-processing (post.c; NEXT-3, readings R33-R36) */
typedef struct {
    double lambda_m;       /* wavelength of the first Fresnel zone (Eq. 13) */
    double angle_deg;      /* ray-angle threshold of the duplicate test */
    double r_s;            /* exact-label search radius = 2 r_s */
    float tx[3];
    const float* rx;       /* RX table indexed by the record's rx */
} or_post_params;
int64_t or_postprocess(const or_scene* S, const or_post_params* Q, const or_refined* in, int64_t n,
                       or_refined* out);
int or_fresnel_dup(const or_post_params* Q, double cos_max, const or_refined* a, const or_refined* b);

#ifdef __cplusplus
}
#endif
#endif
