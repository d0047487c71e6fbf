/* nrt.h — C ABI of the B200-native ray launcher for arXiv 2403.06648
 * ("Ray Launching-Based Computation of Exact Paths with Noisy Dense Point Clouds").
 *
 * Citations: P:n = line n of the paper's LaTeX source, with its section /
 * equation; R<k> = reading k of DESIGN.md §2 (where the paper is silent or replaced by
 * the north_star in BASELINE.json).
 *
 * Conventions for every function below:
 *   - all functions are extern "C", never throw, never abort; they return nrt_status;
 *   - on failure a thread-local message is available from nrt_last_error();
 *   - input pointers are HOST or DEVICE memory as the accompanying nrt_mem says; inputs
 *     are copied (or consumed on the stream) before return and never retained;
 *   - handles own all their device memory; *_free is NULL-safe;
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Functions that must know
 *     a device-side count synchronise that stream before returning.
 *   - units: metres, seconds; float = IEEE binary32, double = binary64.
 */
#ifndef NRT_H
#define NRT_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct nrt_scene_s* nrt_scene; /* immutable after build; usable from many streams */
typedef struct nrt_paths_s* nrt_paths; /* a coarse or refined path set (device memory)   */

typedef enum {
    NRT_OK = 0,
    NRT_E_INVALID = 1,  /* bad argument or bad record (first bad index in nrt_last_error) */
    NRT_E_NOMEM = 2,    /* device allocation failed */
    NRT_E_CUDA = 3,     /* CUDA runtime / kernel error */
    NRT_E_OVERFLOW = 4, /* caller buffer too small; required size in nrt_last_error */
    NRT_E_EMPTY = 5,    /* nothing to do (N = 0 points, or no intersectable geometry) */
    NRT_E_STATE = 6     /* wrong handle kind / stage */
} nrt_status;

typedef enum { NRT_MEM_HOST = 0, NRT_MEM_DEVICE = 1 } nrt_mem;

#define NRT_MAX_INT 8 /* max_refl + max_diff <= NRT_MAX_INT */

/* ---------------------------------------------------------------------------------------
 * Scene (A1: GPU voxelisation).
 * Points are oriented surfels: thin two-sided disks (p, n, r) with a surface label
 * ("a label, a normal vector, and a position"; radius per R4/R5).  The build
 * registers every surfel in every grid cell its exact disk AABB (inflated by
 * max(1e-3*voxel, 2e-5) m) overlaps, sorts (Morton(cell), id) pairs by radix sort and stores
 * the per-cell records contiguously (AoS, 32 B: position, r^2, normal, id).
 * voxel_size is a pure performance knob: results do not depend on it (R29).
 * ------------------------------------------------------------------------------------- */
typedef struct {
    float a[3], b[3]; /* edge segment endpoints */
    float t0[3];      /* face-0 tangent: perpendicular to e, lying in face 0, pointing away from the edge */
    float n0[3];      /* face-0 outward normal */
    float n1[3];      /* face-1 outward normal */
    float n_exp;      /* exterior angle = n_exp*pi with 1 < n_exp < 2 */
    int32_t label;    /* unique edge label, 0 <= label < 4096 */
} nrt_edge;

typedef struct {
    const float* points;   /* n x 3, row-major */
    const float* normals;  /* n x 3; | |n| - 1 | <= 1e-3 required */
    const float* radii;    /* n, or NULL to use `radius` for every surfel */
    float radius;          /* used when radii == NULL; default r_s = 0.015 m */
    const int32_t* labels; /* n, 0 <= label < 4096, or NULL for pseudo-labels (R6) */
    int64_t n;
    float voxel_size;      /* fine-grid cell edge (m) */
    const nrt_edge* edges; /* n_edges exterior diffraction edges (always HOST memory) */
    int32_t n_edges;
    nrt_mem mem;           /* where points/normals/radii/labels live */
    int32_t device;        /* CUDA device ordinal */
    void* stream;          /* cudaStream_t */
    float sdf_cell;        /* NEXT-1: edge a (m) of the cubic cells that bin the points into AABB
                              primitives (the paper's voxel / (D_v D_sv) = 0.0625 m,
                              Table I), 0 = none (disk intersection only).  Each non-empty cell's
                              AABB is its points' extent per axis, or the cell's full extent on an
                              axis where that extent exceeds a/2 (DESIGN R40). */
} nrt_scene_desc;

/* north_star 4-argument form: host arrays, radius 0.015 m, pseudo-labels, no edges,
 * device 0, default stream. */
nrt_status nrt_scene_build(const float* points, const float* normals, int64_t n,
                           float voxel_size, nrt_scene* out);
/* Errors: NRT_E_INVALID (non-finite value, bad normal, r <= 0, label out of range,
 * n_exp outside (1,2) — the message names the first bad index), NRT_E_EMPTY (n == 0). */
nrt_status nrt_scene_build_ex(const nrt_scene_desc* desc, nrt_scene* out);
void nrt_scene_free(nrt_scene s);

typedef struct {
    int64_t n_surfels, n_refs, n_cells;
    int32_t dims[3];
    float origin[3], voxel;
    float r_max;
    int64_t n_aabb;        /* NEXT-1 AABB primitives (0 when sdf_cell == 0) */
    int64_t n_aabb_refs;   /* their registrations in the AABB traversal grid */
    float sdf_cell;
} nrt_scene_info;
nrt_status nrt_scene_info_get(nrt_scene s, nrt_scene_info* info);

/* ---------------------------------------------------------------------------------------
 * Launch (A2-A8): Fibonacci rays from the TX (R1), nearest-surfel traversal under the
 * HIT predicate (R7-R9), specular reflection, RX reception spheres
 * (R12), edge capture + Keller fans (R13-R16, Eq. 14), exact-key
 * dedupe keeping the kappa shortest per (rx, interaction kinds, labels) (R17).
 * The result is bit-identical to the brute-force definition for any
 * voxel size, launch configuration and world size.
 * ------------------------------------------------------------------------------------- */
typedef struct {
    int32_t kappa;        /* paths kept per key (default 1; Table I uses 100) */
    float tau;            /* departure-sheet tolerance (R8), default 0.0015 m */
    float c_R;            /* reception-sphere scale (R12), default 1 */
    float dphi_deg;       /* Keller fan step (R15), default 2.5 deg */
    float theta_ex_deg;   /* departure-sheet angle (R8), default 25 deg */
    float edge_bin;       /* event bin along the edge (R14), default 0.25 m */
    int32_t rank, world;  /* primary-ray shard: lattice index i == rank (mod world) */
    int32_t stage;        /* 0 = full launch (world must be 1 when diffraction is on);
                             1 = primary rays only, keep events (multi-GPU phase 1) */
    int32_t counters;     /* 1 = instrumented kernels also count surfel tests and cells
                             visited (nrt_paths_info); results are unchanged, speed is not */
    nrt_mem mem;          /* where tx / rx live */
    void* stream;
    int32_t intersect;    /* 0 = oriented-surfel disk hit (R7-R9, default); 1 = NEXT-1: the
                             paper's point-set SDF intersection (DESIGN R40-R45):
                             per AABB primitive the ray marches Eqs. 1-4 over the AABB's points;
                             the scene must have been built with sdf_cell > 0 (else NRT_E_STATE) */
    float sdf_r_s;        /* NEXT-1 r_s (m): sigma = sdf_xi * sdf_r_s, and the step where the
                             SDF fails; default 0.015 */
    float sdf_t_sdf;      /* NEXT-1 hit threshold |f| < t_sdf; default 0.0015 */
    float sdf_xi;         /* NEXT-1 xi; default 2 */
    int32_t tracer;       /* 0 = Fibonacci-lattice wavefront (north_star, default); 1 = NEXT-2:
                             the paper's environment-driven launch + voxel cone tracing (P:86-180,
                             Alg. 1; DESIGN R60-R67): IEs on voxels of 8 sdf_cell, rays
                             from the TX to every IE, cone rays marched with the voxels' march
                             distances, every candidate validated by the SDF trace (needs
                             intersect = 1); n_rays is unused; bounces = validation rays; rank /
                             world shard the TX->IE rays */
} nrt_launch_desc;
void nrt_launch_desc_default(nrt_launch_desc* d);

/* north_star form: host tx/rx, defaults above, single shard. */
nrt_status nrt_launch(nrt_scene s, const float tx[3], const float* rx, int32_t n_rx,
                      int64_t n_rays, int32_t max_refl, int32_t max_diff, nrt_paths* coarse_out);
/* Errors: NRT_E_INVALID (n_rays < 1 or >= 2^32, max_refl < 0, max_diff < 0,
 * max_refl + max_diff > NRT_MAX_INT, n_rx > 65535, non-finite tx/rx), NRT_E_STATE
 * (stage 0 with world > 1 and diffraction on). */
nrt_status nrt_launch_ex(nrt_scene s, const float tx[3], const float* rx, int32_t n_rx,
                         int64_t n_rays, int32_t max_refl, int32_t max_diff,
                         const nrt_launch_desc* desc, nrt_paths* coarse_out);

/* Multi-GPU phase 2 (after an all-gather of the stage-1 events of every rank):
 * dedupes the gathered events globally (R14), traces the fans of events r == rank
 * (mod world) (r = rank of the event in global key order) and appends their records to
 * `coarse` (a stage-1 handle), then dedupes `coarse` locally. */
nrt_status nrt_launch_fans(nrt_scene s, nrt_paths coarse, const void* events, int64_t n_events,
                           nrt_mem mem, const nrt_launch_desc* desc);

/* ---------------------------------------------------------------------------------------
 * Refinement (A9-A10): per coarse path, damped Gauss-Newton in FP64 on the stationarity
 * residual of Eqs. 9-11 with the MLS surface of Eqs. 1-4,
 * sigma = xi * r_s, then FP64 visibility, delay = L/c, angles, and
 * shortest-per-key dedupe.  See DESIGN.md §5.
 * ------------------------------------------------------------------------------------- */
typedef struct {
    double xi;        /* sigma = xi * r_s; default 2.0 (Table I) */
    double r_s;       /* refinement sample radius; default 0.003 (Table II) */
    double tol_m;     /* convergence: max |step| < tol_m; default 1e-10 */
    int32_t max_iter; /* default 100 */
    double alpha, beta; /* backtracking (Eq. 12), default 0.4, 0.4 (Table I) */
    double delta;     /* reported ||grad f||^2 < delta test, default 1e-4 */
    double tau;       /* support / sheet tolerance (R25), default 0.0015 */
    double theta_ex_deg; /* sheet angle for shadow rays, default 25 */
    int32_t rank, world; /* path shard: j == rank (mod world) */
    int32_t keep_invalid; /* 1 = keep failed paths in the output (with their status) */
    int32_t select;       /* 0 = every path; 1 = only paths without a diffraction; 2 = only
                             paths with one (R17 keys of the two kinds are disjoint, so the two
                             refined sets are independent — refine the primary-ray paths while
                             the fans are still being traced, then merge) */
    int32_t blocks_per_sm; /* 0 = as many resident path blocks per SM as fit; k > 0 caps it
                             (leaves room for kernels running concurrently on other streams) */
    void* stream;
    int32_t counters;     /* 1 = also count the MLS candidate evaluations (nrt_paths_info
                             mls_value / mls_deriv: the algorithmic FP64 work); results are
                             unchanged */
    int32_t method;       /* 0 = Gauss-Newton (above, default); 1 = NEXT-4: the paper's own
                             gradient descent (DESIGN R50-R56): per interaction Eq. 12
                             backtracking GD (alpha, beta), reflection points re-traced from
                             I_{k-1} with the SDF intersection (sigma = xi r_s, gd_t_sdf; the
                             scene must have sdf_cell > 0, else NRT_E_STATE), normals of Eq. 3
                             over the hit AABB's 3x3x3 cells kept under gd_t_d / gd_t_a_deg,
                             gd_rho iterations, valid iff ||grad f||^2 < delta, SDF visibility.
                             FP32; tol_m, max_iter and select are not used (select must be 0) */
    int32_t gd_rho;       /* iterations rho (Table I: 2000) */
    double gd_t_sdf;      /* refinement t_sdf (Table II: noisy 0.001, noiseless 0.0005) */
    double gd_t_d;        /* distance threshold t_d (m) (Table III: 0.02 noisy, 0.002 noiseless) */
    double gd_t_a_deg;    /* angle threshold t_a (Table III: 1 with true normals, 25 estimated) */
} nrt_refine_desc;
void nrt_refine_desc_default(nrt_refine_desc* d);
nrt_status nrt_refine(nrt_scene s, nrt_paths coarse, nrt_paths* refined_out);
nrt_status nrt_refine_ex(nrt_scene s, nrt_paths coarse, const nrt_refine_desc* desc,
                         nrt_paths* refined_out);

/* ---------------------------------------------------------------------------------------
 * Path sets: fixed-size POD records so that a caller can all-gather raw bytes.
 * ------------------------------------------------------------------------------------- */
enum { NRT_PATHS_COARSE = 0, NRT_PATHS_REFINED = 1, NRT_PATHS_EVENTS = 2 };

typedef struct {
    uint32_t rx;
    uint8_t n_int, n_diff;
    uint16_t kinds;                 /* bit k = 1: interaction k is a diffraction */
    int32_t label[NRT_MAX_INT];     /* surfel or edge label, 0 beyond n_int */
    uint32_t prim[NRT_MAX_INT];     /* surfel id or edge index, 0 beyond n_int */
    float v[NRT_MAX_INT][3];        /* interaction points, 0 beyond n_int */
    float s_edge;                   /* edge parameter of the diffraction point (0 if none) */
    float L;                        /* unfolded length at the RX closest approach */
    uint64_t ray_id;                /* lattice index, or 2^63 | event_rank << 8 | m (fans) */
} nrt_coarse_rec;                   /* 184 bytes */

typedef struct {
    int32_t n_hist, n_diff;
    uint16_t kinds, pad_;
    int32_t label[NRT_MAX_INT];
    uint32_t prim[NRT_MAX_INT];
    float v[NRT_MAX_INT][3];
    float s_edge;
    uint32_t edge;
    int32_t sbin;
    float s;
    float d[3];                     /* incident direction */
    float L;                        /* unfolded length at the edge point */
    float dist2;                    /* squared closest distance ray-edge */
    uint64_t ray_id;
} nrt_event_rec;                    /* 216 bytes */

enum { NRT_REF_OK = 0, NRT_REF_NO_CONVERGE = 1, NRT_REF_OFF_EDGE = 2, NRT_REF_NO_SUPPORT = 3,
       NRT_REF_WRONG_SIDE = 4, NRT_REF_OCCLUDED = 5, NRT_REF_DEGENERATE = 6 };

typedef struct {
    uint32_t rx;
    uint8_t n_int, n_diff;
    uint16_t kinds;
    int32_t label[NRT_MAX_INT];
    uint32_t prim[NRT_MAX_INT];
    double v[NRT_MAX_INT][3];       /* refined interaction points */
    double L;                       /* path length (Eq. 5) */
    double delay;                   /* L / 299792458 */
    float aod_az, aod_el, aoa_az, aoa_el; /* degrees (R27) */
    float inc[NRT_MAX_INT];         /* incidence angle at each vertex (deg) */
    int32_t status, iters;
    double resid;                   /* max |r| at the root */
    double gradsq;                  /* ||grad f||^2 of Eqs. 9-11 at the root */
    uint64_t ray_id;                /* representative coarse ray */
} nrt_refined_rec;

typedef struct {
    int32_t kind;            /* NRT_PATHS_* */
    int64_t n;               /* records */
    int64_t n_raw;           /* raw records before dedupe (launch) */
    int64_t n_events;        /* diffraction events after local dedupe (launch) */
    int64_t n_fan_rays;      /* fan rays traced (launch) */
    uint64_t bounces;        /* segments traced: primary + fan (launch) */
    uint64_t surfel_tests;   /* records tested (launch with counters = 1; else 0); with
                                intersect = 1: Gaussian terms evaluated (one point in one SDF
                                evaluation), and cells_nonempty counts AABB marches */
    uint64_t cells_visited;  /* grid cells visited by the DDA, empty or not (idem) */
    uint64_t cells_nonempty; /* non-empty cells visited (idem) */
    float ms_trace;          /* device time of the primary traversal kernel */
    float ms_fans;           /* device time of the fan traversal kernel */
    float ms_dedupe;         /* device time of event + record dedupe */
    float ms_refine;         /* device time of the refinement kernels */
    float ms_total;          /* device time of the whole call */
    uint64_t mls_value;      /* refine with counters = 1: surfel terms of Eqs. 2-4 evaluated
                                (neighbourhood members within 4 sigma, value passes) */
    uint64_t mls_deriv;      /* idem, derivative passes of the analytic Jacobian (R37) */
} nrt_paths_info;

/* ---------------------------------------------------------------------------------------
 * Post-processing of refined paths (PAPER §II-E; DESIGN.md
 * R33-R36): (1) every reflection vertex takes the label of the nearest surfel within 2 r_s
 * ("the label of the closest point to the intersection point"; lowest id on ties; none
 * -> unchanged); (2) the shortest path per (rx, interaction chain, labels) is kept;
 * (3) paths are ordered by delay (ties in key order); (4) walking that order, a path
 * is dropped when every interaction point lies inside the first Fresnel zone
 * psi_k = sqrt(lambda s1 s2 / (s1 + s2)) (Eq. 13) of an earlier kept path with the same rx and
 * chain and every pair of k-th rays is closer than angle_deg.  Input: a refined set
 * (invalid records are ignored); output: a new refined set in delay order.  The input
 * handle is not modified.  Errors: NRT_E_INVALID (null, lambda_m <= 0, angle_deg outside
 * (0, 180), r_s < 0), NRT_E_STATE (not a refined set), NRT_E_NOMEM, NRT_E_CUDA.
 * ------------------------------------------------------------------------------------- */
typedef struct {
    double lambda_m;  /* wavelength; default 299792458 / 60e9 m (60 GHz carrier, Table I) */
    double angle_deg; /* ray-angle threshold of the duplicate test; default 10 */
    double r_s;       /* exact-label search radius is 2 r_s; default 0.003 (Table II) */
    void* stream;
} nrt_post_desc;
void nrt_post_desc_default(nrt_post_desc* d);
nrt_status nrt_postprocess(nrt_scene s, nrt_paths refined, const nrt_post_desc* desc,
                           nrt_paths* out);

nrt_status nrt_paths_count(nrt_paths p, int64_t* n);
nrt_status nrt_paths_record_size(nrt_paths p, int64_t* bytes);
nrt_status nrt_paths_info_get(nrt_paths p, nrt_paths_info* info);
/* Copy the records into dst (capacity_bytes); NRT_E_OVERFLOW if too small. */
nrt_status nrt_paths_export(nrt_paths p, void* dst, int64_t capacity_bytes, nrt_mem mem);
/* Copy the stage-1 events of a launch handle (nrt_event_rec) into dst. */
nrt_status nrt_paths_export_events(nrt_paths p, void* dst, int64_t capacity_bytes,
                                   int64_t* n_events, nrt_mem mem);
/* Build a coarse set from raw records (e.g. gathered from every rank); tx/rx (host) are
 * the launch endpoints the refinement needs. */
nrt_status nrt_paths_import(const void* src, int64_t n, int32_t kind, nrt_mem mem,
                            const float tx[3], const float* rx, int32_t n_rx, nrt_paths* out);
/* Global dedupe of several coarse (or refined) sets: same key order, keep kappa. */
nrt_status nrt_paths_merge(const nrt_paths* parts, int32_t n_parts, int32_t kappa,
                           nrt_paths* out);
void nrt_paths_free(nrt_paths p);

/* Diagnostic: trace primary rays ray_ids[0..n) (host array) and write, per segment,
 * the hit surfel id or -1 (escape) or -2 (not traced) into hit_ids (host, n x (max_refl+1)). */
nrt_status nrt_debug_trace_rays(nrt_scene s, const float tx[3], int64_t n_rays,
                                int32_t max_refl, const nrt_launch_desc* desc,
                                const uint64_t* ray_ids, int64_t n, int64_t* hit_ids);

const char* nrt_last_error(void);
const char* nrt_version(void);
/* Number of CUDA kernels this library has launched in the process so far (evidence counter). */
uint64_t nrt_kernel_launches(void);
/* Bytes of device memory the library keeps cached between launches (wavefront workspaces:
 *  per-ray state of the rays in flight, up to ~440 B x 2^26 rays), and a call that returns
 * all idle cached blocks to the CUDA memory pool.  Must not race with a running launch. */
/* Diagnostic: FP64 fused multiply-add throughput of this device, TFLOP/s (2 flops per FMA),
 * measured by a synthetic kernel of independent FMA chains (~20 ms).  The roofline denominator
 * of the FP64-bound refinement kernel (bench.py).  <= 0 on failure. */
double nrt_probe_fp64_tflops(int device);
uint64_t nrt_workspace_bytes(void);
void nrt_workspace_trim(void);

#ifdef __cplusplus
}
#endif
#endif
