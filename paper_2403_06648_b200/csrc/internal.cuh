// internal.cuh — shared internals of libnrt (CUDA path).  Independent of oracle/.
//
// Compiled with -fmad=false (no FMA contraction) and IEEE div/sqrt so that every FP32
// quantity on the coarse path is the exact value the definition (DESIGN.md §2 R1-R17)
// prescribes, whatever the grid or launch configuration.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/nrt.h"

namespace nrt {

// ------------------------------------------------------------------------------------
// error plumbing
// ------------------------------------------------------------------------------------
nrt_status set_error(nrt_status st, const char* fmt, ...);
void clear_error();
void count_launch();  // every kernel launch of the library increments a process-wide counter
void ensure_pool(int dev);  // default mempool keeps freed memory cached
void pool_keep_headroom(int dev, cudaStream_t st);  // pool backing >= 1.5x its high-water mark
// Workspace cache for large per-launch buffers (wavefront state).  Growing the stream-ordered
// pool by gigabytes maps fresh physical pages (~50 ms/GB measured), so the biggest buffers are
// kept across launches: ws_get returns an idle cached block of >= bytes on dev (or a new one);
// ws_put marks it idle again and may only be called once no queued work still uses it.
void* ws_get(int dev, size_t bytes, cudaStream_t st);
void ws_put(void* p);

#define NRT_CUDA(call)                                                                    \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess) {                                                          \
            return ::nrt::set_error(e_ == cudaErrorMemoryAllocation ? NRT_E_NOMEM         \
                                                                    : NRT_E_CUDA,         \
                                    "%s:%d %s: %s", __FILE__, __LINE__, #call,            \
                                    cudaGetErrorString(e_));                              \
        }                                                                                 \
    } while (0)

#define NRT_TRY(call)                                                                     \
    do {                                                                                  \
        nrt_status s_ = (call);                                                           \
        if (s_ != NRT_OK) return s_;                                                      \
    } while (0)

// ------------------------------------------------------------------------------------
// R2: FP64 sincos, pi/2 Cody-Waite (2 parts) + minimax kernels, fixed order, no FMA.
// Used on the device (ray generation, fan angles) and on the host (cos theta_ex).
// ------------------------------------------------------------------------------------
__host__ __device__ inline double k_sin(double x) {
    const double S1 = -1.66666666666666324348e-01, S2 = 8.33333333332248946124e-03,
                 S3 = -1.98412698298579493134e-04, S4 = 2.75573137070700676789e-06,
                 S5 = -2.50507602534068634195e-08, S6 = 1.58969099521155010221e-10;
    double z = x * x;
    double v = z * x;
    double r = S2 + z * (S3 + z * (S4 + z * (S5 + z * S6)));
    return x + v * (S1 + z * r);
}
__host__ __device__ inline double k_cos(double x) {
    const double C1 = 4.16666666666666019037e-02, C2 = -1.38888888888741095749e-03,
                 C3 = 2.48015872894767294178e-05, C4 = -2.75573143513906633035e-07,
                 C5 = 2.08757232129817482790e-09, C6 = -1.13596475577881948265e-11;
    double z = x * x;
    double r = z * (C1 + z * (C2 + z * (C3 + z * (C4 + z * (C5 + z * C6)))));
    return 1.0 - (0.5 * z - z * r);
}
constexpr double kPi = 3.14159265358979311600e+00;
__host__ __device__ inline void nrt_sincos(double x, double* s, double* c) {
    const double PIO2_1 = 1.57079632673412561417e+00, PIO2_1T = 6.07710050650619224932e-11,
                 INVPIO2 = 6.36619772367581382433e-01;
    double kf = floor(x * INVPIO2 + 0.5);
    double y = (x - kf * PIO2_1) - kf * PIO2_1T;
    long long k = (long long)kf;
    double sy = k_sin(y), cy = k_cos(y);
    switch (k & 3) {
        case 0: *s = sy; *c = cy; break;
        case 1: *s = cy; *c = -sy; break;
        case 2: *s = -sy; *c = -cy; break;
        default: *s = -cy; *c = sy; break;
    }
}

// R1: spherical Fibonacci lattice direction i of n (FP64, rounded to f32, not renormalised)
__host__ __device__ inline float3 fib_dir(uint64_t i, uint64_t n) {
    const double g = 0.3819660112501051;
    double z = 1.0 - (2.0 * (double)i + 1.0) / (double)n;
    double x = (double)i * g;
    double fr = x - floor(x);
    double phi = (2.0 * kPi) * fr;
    double s, c;
    nrt_sincos(phi, &s, &c);
    double rr = sqrt(1.0 - z * z);
    return make_float3((float)(rr * c), (float)(rr * s), (float)z);
}

__host__ __device__ inline float dot3(float3 a, float3 b) {
    return (a.x * b.x + a.y * b.y) + a.z * b.z;
}

// ------------------------------------------------------------------------------------
// device-side tables
// ------------------------------------------------------------------------------------
struct DevEdge {
    float a[3], e[3], len;
    float t0[3], n0[3], n1[3];
    float n_exp;
    int32_t label;
    float c[3], hl;  // bounding sphere (centre, half length) for conservative culling
    float b_[3];     // the input end point b (refinement works in FP64 from a and b)
};

// a ray's interaction history: a 32 B header and one 32 B sector per interaction, so that the
// per-segment append is one full-sector write
struct __align__(32) HEnt {
    int32_t label;
    uint32_t prim;
    float v[3];
    int32_t pad_[3];
};
struct __align__(32) Hist {
    int32_t n, n_diff;
    uint32_t kinds;
    float s_edge;
    int32_t pad_[4];
    HEnt e[NRT_MAX_INT];
};

}  // namespace nrt

// ------------------------------------------------------------------------------------
// handles
// ------------------------------------------------------------------------------------
struct nrt_scene_s {
    int device = 0;
    int64_t n = 0, nref = 0, ncell = 0;
    int dims[3] = {0, 0, 0};
    float org[3] = {0, 0, 0};
    float v = 0, inv_v = 0, pad = 0, r_max = 0;
    float slack = 1e-4f;  // absolute slack (m) of the traversal's division-free disk prefilter
    uint2* cell = nullptr;     // [ncell] (start, end) into rec
    float4* rec = nullptr;     // [2*nref] AoS: (p, r^2), (n, id bits)
    float4* sp = nullptr;      // [n] (p, r)
    float4* sn = nullptr;      // [n] (n, label bits)
    // home grid for neighbourhood queries (refinement): every surfel once, in the cell of
    // size hv = 2 v that contains p; hrec = (p, r), (n, label bits) sorted by cell
    float hv = 0, inv_hv = 0;
    int hdims[3] = {0, 0, 0};
    uint2* hcell = nullptr;
    float4* hrec = nullptr;
    unsigned* hid = nullptr;   // [n] surfel id of each home record
    unsigned* hoff = nullptr;  // [nh + 1] exclusive prefix of the home-cell counts: the records of
                               // cells a..b (consecutive linear indices) are [hoff[a], hoff[b+1])
    int32_t* label = nullptr;  // [n]
    nrt::DevEdge* edges = nullptr;
    int n_edges = 0;
    std::vector<nrt::DevEdge> h_edges;
    // NEXT-1 AABB primitives (DESIGN R40, §6.4): the points binned into cubic cells of edge
    // sdf_a from sdf_org (the points' minimum); one AABB per non-empty cell, ascending cell.
    //   sdf_pts  [2n]       (p, 0), (n, id bits) of the points in (cell, id) order
    //   sdf_box  [2 n_aabb] (lo, first point bits), (hi, end point bits)
    //   sdf_acell[n_aabb]   linear cell index of each AABB
    // traversal grid: cells of sdf_a from sdf_gorg = sdf_org - sdf_a (one empty margin cell),
    // every AABB registered (sdf_aref, AABB indices) in all cells its box padded by sdf_pad
    // overlaps; sdf_gcell = (start, end), or (D, D) for empty cells (Chebyshev skip distance).
    float sdf_a = 0, sdf_pad = 0;
    float sdf_bmax[3] = {0, 0, 0};  // the points' maximum (NEXT-2 cone angle: the scene diagonal)
    float sdf_org[3] = {0, 0, 0}, sdf_gorg[3] = {0, 0, 0};
    int sdf_dims[3] = {0, 0, 0}, sdf_gdims[3] = {0, 0, 0};
    int64_t n_aabb = 0, n_aref = 0;
    float4* sdf_pts = nullptr;
    float4* sdf_box = nullptr;
    unsigned* sdf_acell = nullptr;
    uint2* sdf_gcell = nullptr;
    unsigned* sdf_aref = nullptr;
    uint2* sdf_crange = nullptr;  // [AABB-grid cells] (first, end) point of the cell's AABB (NEXT-4)
    // output-buffer size hints (largest counts seen by launches on this scene)
    unsigned long long hint_raw = 1 << 16, hint_ev = 1 << 14, hint_fan = 1 << 16;
};

struct nrt_paths_s {
    int kind = NRT_PATHS_COARSE;
    int device = 0;
    int64_t n = 0;
    void* d_rec = nullptr;  // device records
    int64_t n_ev = 0;
    void* d_ev = nullptr;   // stage-1 events (nrt_event_rec, deduped locally, key order)
    float tx[3] = {0, 0, 0};
    std::vector<float> rx;
    nrt_paths_info info{};
    // launch parameters (for stage-2 fans)
    int64_t n_rays = 0;
    int32_t max_refl = 0, max_diff = 0;
    bool pool_owned = true;  // d_rec/d_ev from cudaMallocAsync (false: cudaMalloc)
};

namespace nrt {
// scene.cu
nrt_status scene_build(const nrt_scene_desc* d, nrt_scene* out);
// dedupe.cu
nrt_status dedupe_coarse(const nrt_coarse_rec* in, int64_t n, int32_t kappa, nrt_coarse_rec* out,
                         int64_t* n_out, cudaStream_t st);
nrt_status dedupe_events(const nrt_event_rec* in, int64_t n, nrt_event_rec* out, int64_t* n_out,
                         cudaStream_t st);
nrt_status dedupe_refined(const nrt_refined_rec* in, int64_t n, nrt_refined_rec* out,
                          int64_t* n_out, cudaStream_t st);
// post.cu
nrt_status postprocess(nrt_scene s, nrt_paths in, const nrt_post_desc* d, nrt_paths out, cudaStream_t st);
// launch.cu
struct RxGrid {  // receiver home grid (device arrays; null when the RX set is small)
    uint2* cell = nullptr;
    float4* rx = nullptr;
    float o[3] = {0, 0, 0}, v = 0, tmax = 0;
    float lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};  // tight bounding box of the receivers
    int n[3] = {0, 0, 0};
};
struct LaunchArgs {
    float tx[3];
    const float* d_rx;  // device
    int32_t n_rx;
    int64_t n_rays;
    int32_t max_refl, max_diff;
    nrt_launch_desc desc;
    RxGrid rxg;
    const float* h_rx = nullptr;  // host copy of the receivers (NEXT-2 IE tables)
};
// build / free the receiver grid for rx (host, n_rx x 3) around the scene grid
nrt_status rxgrid_build(nrt_scene s, const float* rx, int32_t n_rx, float rreg, RxGrid* g,
                        cudaStream_t st);
void capture_radius_bounds(nrt_scene s, const LaunchArgs& a, float* r_primary, float* r_fan);
void rxgrid_free(RxGrid* g, cudaStream_t st);
struct KernelStats {
    float ms_kernel = 0;  // device time of the traversal kernel alone
    unsigned long long tests = 0, cells = 0, nonempty = 0;  // counters build only
};
nrt_status launch_primary(nrt_scene s, const LaunchArgs& a, nrt_coarse_rec** raw, int64_t* n_raw,
                          nrt_event_rec** ev, int64_t* n_ev, uint64_t* bounces, KernelStats* ks,
                          cudaStream_t st);
nrt_status launch_fans(nrt_scene s, const LaunchArgs& a, const nrt_event_rec* ev, int64_t n_ev,
                       nrt_coarse_rec** raw, int64_t* n_raw, int64_t* n_fan_rays,
                       uint64_t* bounces, KernelStats* ks, cudaStream_t st);
nrt_status debug_trace(nrt_scene s, const LaunchArgs& a, const uint64_t* ids, int64_t n,
                       int64_t* hit_ids, cudaStream_t st);
float cos_ex_of(float theta_deg);
float cRw_of(float c_R, int64_t n_rays);
// refine.cu
double probe_fp64_tflops(int device);
nrt_status launch_env(nrt_scene s, const LaunchArgs& a, nrt_coarse_rec** raw_out, int64_t* n_raw,
                      uint64_t* rays, float* ms_kernel, uint64_t* terms, cudaStream_t st);  // NEXT-2
nrt_status refine_gd(nrt_scene s, nrt_paths coarse, const nrt_refine_desc* d, nrt_paths out,
                     cudaStream_t st);  // NEXT-4 (launch.cu)
nrt_status refine(nrt_scene s, nrt_paths coarse, const nrt_refine_desc* d, nrt_paths out,
                  cudaStream_t st);
}  // namespace nrt
