// launch.cu — A2-A7: Fibonacci ray generation, 3D-DDA nearest-surfel traversal, specular
// reflection, RX reception spheres, edge capture and Keller fans.
//
// Per ray, per segment, the hit is the lexicographic min (t, id) of the HIT predicate
// (R7-R9).  The grid walk only accelerates that argmin: every surfel is registered in all
// cells its padded disk AABB overlaps, and the walk stops only once best_t < t_exit - pad
// (DESIGN.md §6), so the result equals the brute-force definition for any voxel size.
// All FP32 arithmetic of the definition is done in the order DESIGN.md R3 fixes; the
// library is compiled with -fmad=false so no FMA contraction alters a rounding (explicit
// __fmaf_rn appears only in the prefilter and grid walk, which never decide a result).
//
// Execution model (wavefront): per bounce, one persistent TRACE kernel finds
// the nearest hit of every live ray segment (tight loop: record tests + grid moves, lanes
// refill from a device counter), then one SHADE kernel does the per-segment work uniformly
// across threads (RX captures, edge captures, reflection, history) and compacts the live
// list for the next bounce.  Counts stay on the device: no host round trip between bounces.
#include <cooperative_groups.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "internal.cuh"

namespace cg = cooperative_groups;

namespace nrt {

float cos_ex_of(float theta_deg) {
    double s, c;
    nrt_sincos((double)theta_deg * (kPi / 180.0), &s, &c);
    return (float)c;
}
float cRw_of(float c_R, int64_t n_rays) {
    return (float)((double)c_R * sqrt(4.0 * kPi / (double)n_rays));
}

namespace {

constexpr int kMaxIter = NRT_MAX_INT + 1;  // bounce iterations per wavefront launch
constexpr int kShadeEdges = 1024;  // edge tables up to this size are staged in SHADE's smem
#ifndef NRT_SHADE_RX
#define NRT_SHADE_RX 32  // receiver sets up to this size are staged in smem (else receiver grid)
#endif

// per-ray state that only the shade kernel touches: a 64 B header (two sectors, read as
// vectors), then the history (its header sector and one sector per interaction)
struct __align__(32) RayCold {
    float L, Ls, kR, R0;
    int32_t seg, budget, flags;  // flags: bit0 edge captures on, bit1 after a diffraction
    int32_t pad_;
    uint64_t rid;
    uint64_t pad2_[3];
    Hist h;
};

// per-ray hot state, one 64 B record (two full sectors): TRACE reads it whole, SHADE rewrites
// it whole (no partial-sector read-modify-writes); the hit goes into l1.xy once the segment's
// departure normals are no longer needed
struct __align__(64) RayHot {
    float4 o;   // origin xyz, prev surfel id / cell (int bits)
    float4 d;   // direction
    float4 l0;  // departure-sheet normal 0
    float4 l1;  // departure-sheet normal 1; after TRACE: (best_t, best id bits, -, -)
};

struct Wave {
    void* slab;      // one workspace block holding all arrays below
    RayHot* ray;     // [cap]
    float4* hitn;    // [cap] SDF mode: (unit MLS normal at the hit, AABB cell bits)
    RayCold* cold;   // [cap]
    unsigned* alive[2];       // ping-pong live lists
    unsigned* okey[2];        // ordering keys (primary batches)
    unsigned* oval;           // ordering values (slot ids)
    unsigned* skey;           // SHADE: ordering keys of the next live list (null: no reorder)
    void* otmp;               // radix-sort temporary storage
    size_t otmp_bytes;
    unsigned long long* n_alive;  // [kMaxIter + 1]
    unsigned long long* ctr;      // [kMaxIter] trace work counters
};

struct TP {  // trace parameters (by value into the kernels)
    // grid
    const uint2* cell;
    const float4* rec;
    const float4* sn;
    const int32_t* label;
    float ox, oy, oz, v, inv_v, pad;
    int nx, ny, nz;
    // launch
    float tx, ty, tz;
    const float* rx;
    int n_rx;
    uint64_t n_rays;
    int rank, world;
    int max_refl, max_diff;
    float tau, cos_ex, cRw, b_e, edge_bin, c_R, dphi_deg;
    float slack;  // absolute slack of the division-free disk prefilter (m)
    float ok_inv;  // 1 / (coarse ordering cell): 64 coarse cells span the grid's longest axis
    // receiver home grid (many RX): cells of rxg_v, RX sorted by cell as (x, y, z, j bits)
    const uint2* rxg_cell;
    const float4* rxg_rx;
    float rxg_o[3], rxg_v, rxg_inv, rxg_tmax;
    float rxg_lo[3], rxg_hi[3];  // tight bounding box of the receivers
    int rxg_n[3];
    const DevEdge* edges;
    int n_edges;
    int shade_rx, shade_edges;  // receivers / edge cull spheres staged in SHADE's shared memory
    // outputs
    nrt_coarse_rec* raw;
    unsigned long long raw_cap;
    unsigned long long* raw_n;
    nrt_event_rec* ev;
    unsigned long long ev_cap;
    unsigned long long* ev_n;
    unsigned long long* bounces;
    unsigned long long* counters;  // [tests, cells, nonempty cells] (instrumented build)
    int64_t* hit_out;              // debug: per-segment hit ids
    // NEXT-1 point-set SDF intersection (DESIGN R40-R45, §6.4); sdf == 0: disk hit
    int sdf;
    const float4* sdf_pts;    // (p, 0), (n, id bits) in (cell, id) order
    const float4* sdf_box;    // (lo, first point bits), (hi, end point bits) per AABB
    const unsigned* sdf_acell;
    const uint2* sdf_gcell;   // traversal grid (start, end) into sdf_aref, or (D, D) empty
    const unsigned* sdf_aref;
    float sg_o[3], sdf_a, sdf_inv_a, sdf_stop;  // sdf_stop = 2 * half + pad (early exit)
    int sg_n[3];
    float sdf_half, sdf_rs, sdf_tsdf, sdf_inv;  // sdf_inv = 1 / (2 sigma^2), sigma = xi r_s
    const uint2* sdf_crange;  // [AABB-grid cells] point range of the cell's AABB, (0, 0) if none
    int sd_n[3];              // AABB-grid dims (R40)
    float sd_o[3];            // AABB-grid origin (the points' minimum)
    float sdf_sigma;          // xi r_s (FP32)
    const float4* sn_p;       // per-point (p, r) (NEXT-4: the record point's cell)
};

__device__ __forceinline__ unsigned long long agg_inc(unsigned long long* ctr) {
    cg::coalesced_group g = cg::coalesced_threads();
    unsigned long long base = 0;
    if (g.thread_rank() == 0) base = atomicAdd(ctr, (unsigned long long)g.size());
    base = g.shfl(base, 0);
    return base + g.thread_rank();
}

struct Cnt {
    unsigned long long tests = 0, cells = 0, nonempty = 0;
};

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
[[maybe_unused]] __device__ __forceinline__ unsigned long long lane_inc(unsigned long long* ctr) {
    return atomicAdd(ctr, 1ull);
}
#ifndef NRT_TRACE_MINB
#define NRT_TRACE_MINB 8  // min resident blocks/SM for k_trace: 64 registers, 50% occupancy
                          // (measured best of 4/6/8 on C2, scripts/variant_sweep.sh)
#endif
#ifndef NRT_TRACE_COOP
#define NRT_TRACE_COOP 0  // warp-cooperative record tests (k_trace_coop); 0 = per-lane k_trace
#endif
#ifndef NRT_TRACE_FETCH
#define NRT_TRACE_FETCH lane_inc
#endif
#ifndef NRT_TRACE_UNROLL
#define NRT_TRACE_UNROLL 3  // records loaded per k_trace iteration before testing them (C5 A/B,
                            // 1 / 2 / 3 / 4 / 6 / 8: trace 430 / 375 / 359 / 379 / 535 / 676 ms)
#endif
#ifndef NRT_TRACE_REFILL
#define NRT_TRACE_REFILL 8  // 1: each lane refills alone; k > 1: warp refills k+ idle lanes together
#endif

__device__ void write_record(const TP& P, const Hist& h, int rx, float L, uint64_t ray_id) {
    unsigned long long slot = agg_inc(P.raw_n);
    if (slot >= P.raw_cap) return;
    nrt_coarse_rec c;
    c.rx = (uint32_t)rx;
    c.n_int = (uint8_t)h.n;
    c.n_diff = (uint8_t)h.n_diff;
    c.kinds = (uint16_t)h.kinds;
#pragma unroll
    for (int k = 0; k < NRT_MAX_INT; ++k) {
        bool on = k < h.n;
        c.label[k] = on ? h.e[k].label : 0;
        c.prim[k] = on ? h.e[k].prim : 0u;
        c.v[k][0] = on ? h.e[k].v[0] : 0.0f;
        c.v[k][1] = on ? h.e[k].v[1] : 0.0f;
        c.v[k][2] = on ? h.e[k].v[2] : 0.0f;
    }
    c.s_edge = h.s_edge;
    c.L = L;
    c.ray_id = ray_id;
    P.raw[slot] = c;
}

// ---- A5: RX reception spheres (R12 / R16) ---------------------------------------------
// the capture test of RX j exactly as the definition orders it
__device__ __forceinline__ void rx_test(const TP& P, const Hist& h, float3 o, float3 d, float t_hit,
                                        float L, float Ls, float kR, float R0, bool after_diff,
                                        uint64_t ray_id, int j, float x0, float x1, float x2) {
    const float wx = x0 - o.x, wy = x1 - o.y, wz = x2 - o.z;
    const float tj = (wx * d.x + wy * d.y) + wz * d.z;
    if (!(tj > 0.0f && tj < t_hit)) return;
    const float px = wx - tj * d.x, py = wy - tj * d.y, pz = wz - tj * d.z;
    const float pp = (px * px + py * py) + pz * pz;
    const float R = after_diff ? kR * (Ls + tj) + R0 : kR * (L + tj);
    if (!(pp <= R * R)) return;
    write_record(P, h, j, L + tj, ray_id);
}

__device__ void rx_captures(const TP& P, const Hist& h, float3 o, float3 d, float t_hit, float L,
                            float Ls, float kR, float R0, bool after_diff, uint64_t ray_id) {
    if (!P.rxg_cell) {  // few receivers: test them all
        for (int j = 0; j < P.n_rx; ++j)
            rx_test(P, h, o, d, t_hit, L, Ls, kR, R0, after_diff, ray_id, j, P.rx[3 * j],
                    P.rx[3 * j + 1], P.rx[3 * j + 2]);
        return;
    }
    // many receivers: every receiver is registered in all cells of the receiver grid within
    // the launch's largest capture radius Rreg (+ pad) of it.  The segment walks that grid by
    // 3D-DDA; the walk's cell t-intervals partition the segment, and receiver j is tested only
    // in the cell whose interval holds its closest-approach parameter t_j — whose point lies
    // within R <= Rreg of the receiver, so the receiver is registered there: every capturable
    // receiver is tested exactly once.
    float T = fminf(t_hit, P.rxg_tmax);
    float t0 = 0.0f;
    const float ov[3] = {o.x, o.y, o.z}, dv[3] = {d.x, d.y, d.z};
    for (int a = 0; a < 3; ++a) {  // clip to the grid box (it holds every receiver's ball)
        const float lo = P.rxg_o[a], hi = P.rxg_o[a] + P.rxg_n[a] * P.rxg_v;
        if (dv[a] != 0.0f) {
            const float inv = 1.0f / dv[a];
            const float ta = (lo - ov[a]) * inv, tb = (hi - ov[a]) * inv;
            t0 = fmaxf(t0, fminf(ta, tb));
            T = fminf(T, fmaxf(ta, tb));
        } else if (ov[a] < lo || ov[a] > hi) {
            T = -1.0f;
        }
    }
    if (!(t0 < T)) return;
    int c[3];
    float tm[3], inv[3];
    for (int a = 0; a < 3; ++a) {
        const float p = ov[a] + t0 * dv[a];
        c[a] = min(P.rxg_n[a] - 1, max(0, (int)floorf((p - P.rxg_o[a]) * P.rxg_inv)));
        inv[a] = 1.0f / dv[a];
        tm[a] = dv[a] != 0.0f ? ((P.rxg_o[a] + (float)(c[a] + (dv[a] > 0.0f)) * P.rxg_v) - ov[a]) * inv[a]
                              : INFINITY;
    }
    float t_in = t0;
    for (;;) {
        int ax = 0;
        if (tm[1] < tm[ax]) ax = 1;
        if (tm[2] < tm[ax]) ax = 2;
        const float t_out = tm[ax];
        const bool last = !(t_out < T);
        const uint2 rg = __ldg(&P.rxg_cell[c[0] + P.rxg_n[0] * (c[1] + P.rxg_n[1] * c[2])]);
        for (unsigned q = rg.x; q < rg.y; ++q) {
            const float4 r = __ldg(&P.rxg_rx[q]);
            const float wx = r.x - o.x, wy = r.y - o.y, wz = r.z - o.z;
            const float tj = (wx * d.x + wy * d.y) + wz * d.z;
            if (!((tj >= t_in || t_in == t0) && (tj < t_out || last))) continue;  // owner cell
            rx_test(P, h, o, d, t_hit, L, Ls, kR, R0, after_diff, ray_id, __float_as_int(r.w), r.x,
                    r.y, r.z);
        }
        if (last) break;
        c[ax] += dv[ax] > 0.0f ? 1 : -1;
        if (c[ax] < 0 || c[ax] >= P.rxg_n[ax]) break;
        t_in = t_out;
        tm[ax] = ((P.rxg_o[ax] + (float)(c[ax] + (dv[ax] > 0.0f)) * P.rxg_v) - ov[ax]) * inv[ax];
    }
}

// receivers staged in shared memory (x, y, z, index bits): the all-receivers loop of
// rx_captures with a warp-uniform trip count (lanes stay converged, so each receiver is one
// broadcast read); `on` masks lanes without a segment.  Same tests, same order.
__device__ __forceinline__ void rx_captures_staged(const TP& P, const float4* srx, bool on, const Hist& h,
                                                   float3 o, float3 d, float t_hit, float L, float Ls,
                                                   float kR, float R0, bool after_diff, uint64_t ray_id) {
    for (int q = 0; q < P.shade_rx; ++q) {
        const float4 r = srx[q];
        if (on) rx_test(P, h, o, d, t_hit, L, Ls, kR, R0, after_diff, ray_id, __float_as_int(r.w), r.x, r.y, r.z);
        __syncwarp();
    }
}

// ---- A6: edge capture -> diffraction events (R13) --------------------------------------
// the capture test of edge j (R13) after the cull, and the event record
__device__ __forceinline__ void edge_event(const TP& P, const Hist& h, float3 o, float3 d, float t_hit,
                                           float L, uint64_t ray_id, int j) {
    const DevEdge& E = P.edges[j];
    const float b = (d.x * E.e[0] + d.y * E.e[1]) + d.z * E.e[2];
    const float w0x = o.x - E.a[0], w0y = o.y - E.a[1], w0z = o.z - E.a[2];
    const float den = 1.0f - b * b;
    if (!(den > 1e-12f)) return;
    const float de = (E.e[0] * w0x + E.e[1] * w0y) + E.e[2] * w0z;
    const float dd = (d.x * w0x + d.y * w0y) + d.z * w0z;
    const float te = (b * de - dd) / den;
    const float s = (de - b * dd) / den;
    if (!(s >= 0.0f && s <= E.len)) return;
    if (!(te > 0.0f && te < t_hit + P.b_e)) return;
    const float pcx = o.x + te * d.x, pcy = o.y + te * d.y, pcz = o.z + te * d.z;
    const float pex = E.a[0] + s * E.e[0], pey = E.a[1] + s * E.e[1], pez = E.a[2] + s * E.e[2];
    const float dx = pcx - pex, dy = pcy - pey, dz = pcz - pez;
    const float dist2 = (dx * dx + dy * dy) + dz * dz;
    const float R = P.cRw * (L + te);
    if (!(dist2 <= R * R)) return;
    unsigned long long slot = agg_inc(P.ev_n);
    if (slot >= P.ev_cap) return;
    nrt_event_rec e;
    e.n_hist = h.n;
    e.n_diff = h.n_diff;
    e.kinds = (uint16_t)h.kinds;
    e.pad_ = 0;
#pragma unroll
    for (int k = 0; k < NRT_MAX_INT; ++k) {
        bool on = k < h.n;
        e.label[k] = on ? h.e[k].label : 0;
        e.prim[k] = on ? h.e[k].prim : 0u;
        e.v[k][0] = on ? h.e[k].v[0] : 0.0f;
        e.v[k][1] = on ? h.e[k].v[1] : 0.0f;
        e.v[k][2] = on ? h.e[k].v[2] : 0.0f;
    }
    e.s_edge = h.s_edge;
    e.edge = (uint32_t)j;
    e.sbin = (int32_t)floorf(s / P.edge_bin);
    e.s = s;
    e.d[0] = d.x;
    e.d[1] = d.y;
    e.d[2] = d.z;
    e.L = L + te;
    e.dist2 = dist2;
    e.ray_id = ray_id;
    P.ev[slot] = e;
}

// all edges from global memory (edge tables larger than the shared staging)
__device__ void edge_captures(const TP& P, const Hist& h, float3 o, float3 d, float t_hit,
                              float L, uint64_t ray_id) {
    // conservative cull: a capture needs a ray point at t < t_hit + b_e within
    // R(L + t) <= Rmax of an edge point, hence within hl + Rmax of the edge centre
    const float T = fminf(t_hit + P.b_e, 1e4f);
    const float Rmax = P.cRw * (L + T) * 1.001f + 1e-4f;
    for (int j = 0; j < P.n_edges; ++j) {
        const DevEdge& E = P.edges[j];
        const float cx = E.c[0] - o.x, cy = E.c[1] - o.y, cz = E.c[2] - o.z;
        const float tc = fminf(fmaxf(cx * d.x + cy * d.y + cz * d.z, 0.0f), T);
        const float ux = cx - tc * d.x, uy = cy - tc * d.y, uz = cz - tc * d.z;
        const float lim = E.hl + Rmax;
        if (ux * ux + uy * uy + uz * uz > lim * lim) continue;
        edge_event(P, h, o, d, t_hit, L, ray_id, j);
    }
}

// edges with their cull spheres (c, hl) staged in shared memory; warp-uniform loop as above
__device__ __forceinline__ void edge_captures_staged(const TP& P, const float4* sed, bool on, const Hist& h,
                                                     float3 o, float3 d, float t_hit, float L,
                                                     uint64_t ray_id) {
    const float T = fminf(t_hit + P.b_e, 1e4f);
    const float Rmax = P.cRw * (L + T) * 1.001f + 1e-4f;
    for (int j = 0; j < P.shade_edges; ++j) {
        const float4 c4 = sed[j];
        if (on) {
            const float cx = c4.x - o.x, cy = c4.y - o.y, cz = c4.z - o.z;
            const float tc = fminf(fmaxf(cx * d.x + cy * d.y + cz * d.z, 0.0f), T);
            const float ux = cx - tc * d.x, uy = cy - tc * d.y, uz = cz - tc * d.z;
            const float lim = c4.w + Rmax;
            if (ux * ux + uy * uy + uz * uz <= lim * lim) edge_event(P, h, o, d, t_hit, L, ray_id, j);
        }
        __syncwarp();
    }
}

// ---- A7: fans -------------------------------------------------------------------------
struct FanGeo {
    int M;
    double ct, st;
};
__device__ __forceinline__ FanGeo fan_geo(const TP& P, const nrt_event_rec& ev) {
    const DevEdge& E = P.edges[ev.edge];
    FanGeo g;
    g.ct = (double)((ev.d[0] * E.e[0] + ev.d[1] * E.e[1]) + ev.d[2] * E.e[2]);
    g.st = sqrt(fmax(0.0, 1.0 - g.ct * g.ct));
    if (g.st < 1e-6) {
        g.M = 0;
        return g;
    }
    int M0 = (int)ceil((double)E.n_exp * 180.0 / (double)P.dphi_deg);
    int M = (int)ceil((double)M0 * g.st);
    g.M = M < 1 ? 1 : M;
    return g;
}

__global__ void k_fan_count(TP P, const nrt_event_rec* ev, int64_t n_ev, unsigned int* cnt) {
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_ev) return;
    int mine = (int)(r % P.world) == P.rank;
    cnt[r] = mine ? (unsigned)fan_geo(P, ev[r]).M : 0u;
}

// =======================================================================================
// Wavefront engine
// =======================================================================================
struct Seg {  // trace-kernel lane state for one segment
    float3 o, d, inv, l0, l1;
    int prev;
    float best_t, tmx, tmy, tmz;
    int best, ix, iy, iz, cellD;
    unsigned k, kend;
};

template <bool CNT>
__device__ __forceinline__ void load_cell(const TP& P, Seg& s, Cnt& cnt) {
    const uint2 rg = __ldg(&P.cell[s.ix + P.nx * (s.iy + P.ny * s.iz)]);
    if (CNT) cnt.cells++;
    if (rg.y > rg.x) {
        s.k = rg.x;
        s.kend = rg.y;
        s.cellD = 1;
        if (CNT) {
            cnt.nonempty++;
            cnt.tests += rg.y - rg.x;
        }
    } else {
        s.cellD = (int)rg.x;
    }
}

// grid entry, first cell, first header load; false when the ray misses the grid
template <bool CNT>
__device__ __forceinline__ bool seg_begin(const TP& P, Seg& s, Cnt& cnt) {
    s.best_t = INFINITY;
    s.best = -1;
    s.k = s.kend = 0;
    const float3 o = s.o, d = s.d;
    s.inv = make_float3(rcp_approx(d.x), rcp_approx(d.y), rcp_approx(d.z));  // walk only: approximate is fine (§6.2)
    const float gx1 = P.ox + P.nx * P.v, gy1 = P.oy + P.ny * P.v, gz1 = P.oz + P.nz * P.v;
    float t0 = 0.0f, t1 = INFINITY;
    {
        float a = (P.ox - o.x) * s.inv.x, b = (gx1 - o.x) * s.inv.x;
        if (d.x != 0.0f) { t0 = fmaxf(t0, fminf(a, b)); t1 = fminf(t1, fmaxf(a, b)); }
        else if (o.x < P.ox || o.x > gx1) t1 = -1.0f;
        a = (P.oy - o.y) * s.inv.y; b = (gy1 - o.y) * s.inv.y;
        if (d.y != 0.0f) { t0 = fmaxf(t0, fminf(a, b)); t1 = fminf(t1, fmaxf(a, b)); }
        else if (o.y < P.oy || o.y > gy1) t1 = -1.0f;
        a = (P.oz - o.z) * s.inv.z; b = (gz1 - o.z) * s.inv.z;
        if (d.z != 0.0f) { t0 = fmaxf(t0, fminf(a, b)); t1 = fminf(t1, fmaxf(a, b)); }
        else if (o.z < P.oz || o.z > gz1) t1 = -1.0f;
    }
    if (t0 > t1) return false;
    const float sx = o.x + t0 * d.x, sy = o.y + t0 * d.y, sz = o.z + t0 * d.z;
    s.ix = min(P.nx - 1, max(0, (int)floorf((sx - P.ox) * P.inv_v)));
    s.iy = min(P.ny - 1, max(0, (int)floorf((sy - P.oy) * P.inv_v)));
    s.iz = min(P.nz - 1, max(0, (int)floorf((sz - P.oz) * P.inv_v)));
    s.tmx = d.x != 0.0f ? ((P.ox + (float)(s.ix + (d.x > 0.0f)) * P.v) - o.x) * s.inv.x : INFINITY;
    s.tmy = d.y != 0.0f ? ((P.oy + (float)(s.iy + (d.y > 0.0f)) * P.v) - o.y) * s.inv.y : INFINITY;
    s.tmz = d.z != 0.0f ? ((P.oz + (float)(s.iz + (d.z > 0.0f)) * P.v) - o.z) * s.inv.z : INFINITY;
    load_cell<CNT>(P, s, cnt);
    return true;
}

// one grid move out of the current (exhausted) cell: a DDA step, or, from an empty cell
// whose Chebyshev distance to the nearest non-empty cell is D >= 2, a jump across the empty
// box [c-(D-1), c+(D-1)] (the paper's march distance, P:154 / P:281).  false = left the grid.
template <bool CNT>
__device__ __forceinline__ bool grid_move(const TP& P, Seg& s, Cnt& cnt) {
    const float3 o = s.o, d = s.d;
    const int D = s.cellD;
    if (D <= 1) {
        if (s.tmx <= s.tmy && s.tmx <= s.tmz) {
            s.ix += d.x > 0.0f ? 1 : -1;
            if (s.ix < 0 || s.ix >= P.nx) return false;
            s.tmx = ((P.ox + (float)(s.ix + (d.x > 0.0f)) * P.v) - o.x) * s.inv.x;
        } else if (s.tmy <= s.tmz) {
            s.iy += d.y > 0.0f ? 1 : -1;
            if (s.iy < 0 || s.iy >= P.ny) return false;
            s.tmy = ((P.oy + (float)(s.iy + (d.y > 0.0f)) * P.v) - o.y) * s.inv.y;
        } else {
            s.iz += d.z > 0.0f ? 1 : -1;
            if (s.iz < 0 || s.iz >= P.nz) return false;
            s.tmz = ((P.oz + (float)(s.iz + (d.z > 0.0f)) * P.v) - o.z) * s.inv.z;
        }
    } else {
        const int r = D - 1;
        const int fx = d.x > 0.0f ? s.ix + r + 1 : s.ix - r;
        const int fy = d.y > 0.0f ? s.iy + r + 1 : s.iy - r;
        const int fz = d.z > 0.0f ? s.iz + r + 1 : s.iz - r;
        const float Tx = d.x != 0.0f ? ((P.ox + (float)fx * P.v) - o.x) * s.inv.x : INFINITY;
        const float Ty = d.y != 0.0f ? ((P.oy + (float)fy * P.v) - o.y) * s.inv.y : INFINITY;
        const float Tz = d.z != 0.0f ? ((P.oz + (float)fz * P.v) - o.z) * s.inv.z : INFINITY;
        const float T = fminf(Tx, fminf(Ty, Tz));
        const float px = o.x + T * d.x, py = o.y + T * d.y, pz = o.z + T * d.z;
        int nx = (int)floorf((px - P.ox) * P.inv_v), ny = (int)floorf((py - P.oy) * P.inv_v),
            nz = (int)floorf((pz - P.oz) * P.inv_v);
        nx = min(s.ix + r, max(s.ix - r, nx));
        ny = min(s.iy + r, max(s.iy - r, ny));
        nz = min(s.iz + r, max(s.iz - r, nz));
        if (Tx <= Ty && Tx <= Tz) nx = d.x > 0.0f ? s.ix + r + 1 : s.ix - r - 1;
        else if (Ty <= Tz) ny = d.y > 0.0f ? s.iy + r + 1 : s.iy - r - 1;
        else nz = d.z > 0.0f ? s.iz + r + 1 : s.iz - r - 1;
        if (nx < 0 || nx >= P.nx || ny < 0 || ny >= P.ny || nz < 0 || nz >= P.nz) return false;
        s.ix = nx;
        s.iy = ny;
        s.iz = nz;
        s.tmx = d.x != 0.0f ? ((P.ox + (float)(nx + (d.x > 0.0f)) * P.v) - o.x) * s.inv.x : INFINITY;
        s.tmy = d.y != 0.0f ? ((P.oy + (float)(ny + (d.y > 0.0f)) * P.v) - o.y) * s.inv.y : INFINITY;
        s.tmz = d.z != 0.0f ? ((P.oz + (float)(nz + (d.z > 0.0f)) * P.v) - o.z) * s.inv.z : INFINITY;
    }
    load_cell<CNT>(P, s, cnt);
    return true;
}

// HIT predicate (R7-R9) on one loaded record, keeping the lexicographic min (t, id).
// A division-free prefilter rejects records whose disk the ray clearly misses:
// q * dn = w * dn - f0 * d (w = o - p), so |q| > r  <=>  |w dn - f0 d|^2 > r^2 dn^2; the
// reject threshold carries an absolute slack P.slack (>> the FP32 error of either form), so
// only records that might pass reach the exact, definition-ordered arithmetic.
__device__ __forceinline__ void test_record(const TP& P, Seg& s, const float4 A, const float4 B) {
    const int id = __float_as_int(B.w);
    const float wx = s.o.x - A.x, wy = s.o.y - A.y, wz = s.o.z - A.z;
    const float f0 = (wx * B.x + wy * B.y) + wz * B.z;
    const float dn = (s.d.x * B.x + s.d.y * B.y) + s.d.z * B.z;
    if (!(f0 * dn < 0.0f)) return;
    {
        const float ex = __fmaf_rn(-f0, s.d.x, wx * dn), ey = __fmaf_rn(-f0, s.d.y, wy * dn),
                    ez = __fmaf_rn(-f0, s.d.z, wz * dn);
        const float rs = A.w + P.slack;
        if (__fmaf_rn(ex, ex, __fmaf_rn(ey, ey, ez * ez)) > rs * rs * (dn * dn)) return;
    }
    if (id == s.prev) return;
    if (fabsf(f0) <= P.tau) {
        const float c0 = (B.x * s.l0.x + B.y * s.l0.y) + B.z * s.l0.z;
        const float c1 = (B.x * s.l1.x + B.y * s.l1.y) + B.z * s.l1.z;
        if (fabsf(c0) >= P.cos_ex || fabsf(c1) >= P.cos_ex) return;
    }
    const float t = (-f0) / dn;
    if (t > s.best_t) return;
    const float hx = s.o.x + t * s.d.x, hy = s.o.y + t * s.d.y, hz = s.o.z + t * s.d.z;
    const float qx = hx - A.x, qy = hy - A.y, qz = hz - A.z;
    const float qq = (qx * qx + qy * qy) + qz * qz;
    if (qq <= A.w * A.w && (t < s.best_t || id < s.best)) {
        s.best_t = t;
        s.best = id;
    }
}

__device__ __forceinline__ void flush_counts(const TP& P, unsigned long long bounces, const Cnt& c,
                                             bool cnt_on) {
    for (int off = 16; off > 0; off >>= 1) bounces += __shfl_down_sync(0xffffffffu, bounces, off);
    if ((threadIdx.x & 31) == 0 && bounces) atomicAdd(P.bounces, bounces);
    if (cnt_on) {
        unsigned long long t = c.tests, ce = c.cells, ne = c.nonempty;
        for (int off = 16; off > 0; off >>= 1) {
            t += __shfl_down_sync(0xffffffffu, t, off);
            ce += __shfl_down_sync(0xffffffffu, ce, off);
            ne += __shfl_down_sync(0xffffffffu, ne, off);
        }
        if ((threadIdx.x & 31) == 0) {
            atomicAdd(P.counters, t);
            atomicAdd(P.counters + 1, ce);
            atomicAdd(P.counters + 2, ne);
        }
    }
}

// TRACE: nearest hit of every live segment of bounce b (persistent, dynamic refill)
template <bool CNT>
__global__ void __launch_bounds__(128, NRT_TRACE_MINB) k_trace(TP P, Wave W, int b) {
    const unsigned long long n = W.n_alive[b];
    const unsigned* alive = W.alive[b & 1];
    unsigned long long bounces = 0;
    Cnt cnt;
    Seg s;
    unsigned ray = 0;
    bool have = false;
#if NRT_TRACE_REFILL > 1
    // warp refill: idle lanes take consecutive live-list entries together once at least
    // NRT_TRACE_REFILL of them are idle (or nothing else is running) -> coherent lanes
    const int lane = threadIdx.x & 31;
    bool done = false;
    for (;;) {
        const unsigned idle = __ballot_sync(0xffffffffu, !have && !done);
        const unsigned busy = __ballot_sync(0xffffffffu, have);
        if (!idle && !busy) break;
        if (idle && (__popc(idle) >= NRT_TRACE_REFILL || busy == 0)) {
            const int leader = __ffs(idle) - 1;
            unsigned long long base = 0;
            if (lane == leader) base = atomicAdd(&W.ctr[b], (unsigned long long)__popc(idle));
            base = __shfl_sync(0xffffffffu, base, leader);
            if (!have && !done) {
                const unsigned long long j = base + __popc(idle & ((1u << lane) - 1u));
                if (j >= n) {
                    done = true;
                } else {
                    ray = alive[j];
                    const RayHot R = W.ray[ray];
                    const float4 o = R.o, d = R.d, a = R.l0, c = R.l1;
                    s.o = make_float3(o.x, o.y, o.z);
                    s.prev = __float_as_int(o.w);
                    s.d = make_float3(d.x, d.y, d.z);
                    s.l0 = make_float3(a.x, a.y, a.z);
                    s.l1 = make_float3(c.x, c.y, c.z);
                    ++bounces;
                    if (!seg_begin<CNT>(P, s, cnt)) *(float2*)&W.ray[ray].l1 = make_float2(INFINITY, __int_as_float(-1));
                    else have = true;
                }
            }
        }
        if (!have) continue;
#else
    for (;;) {
        if (!have) {
            const unsigned long long j = NRT_TRACE_FETCH(&W.ctr[b]);
            if (j >= n) break;
            ray = alive[j];
            const RayHot R = W.ray[ray];
            const float4 o = R.o, d = R.d, a = R.l0, c = R.l1;
            s.o = make_float3(o.x, o.y, o.z);
            s.prev = __float_as_int(o.w);
            s.d = make_float3(d.x, d.y, d.z);
            s.l0 = make_float3(a.x, a.y, a.z);
            s.l1 = make_float3(c.x, c.y, c.z);
            ++bounces;
            if (!seg_begin<CNT>(P, s, cnt)) {
                *(float2*)&W.ray[ray].l1 = make_float2(INFINITY, __int_as_float(-1));
                continue;
            }
            have = true;
        }
#endif
        if (s.k < s.kend) {
            // NRT_TRACE_UNROLL records per iteration, all loads issued before any test; indices
            // past the cell end repeat the last record (the (t, id) argmin is idempotent)
            const unsigned last = s.kend - 1;
            float4 A[NRT_TRACE_UNROLL], B[NRT_TRACE_UNROLL];
#pragma unroll
            for (int u = 0; u < NRT_TRACE_UNROLL; ++u) {
                const unsigned ku = min(s.k + u, last);
                A[u] = __ldg(&P.rec[2 * ku]);
                B[u] = __ldg(&P.rec[2 * ku + 1]);
            }
#pragma unroll
            for (int u = 0; u < NRT_TRACE_UNROLL; ++u) test_record(P, s, A[u], B[u]);
            s.k = min(s.k + NRT_TRACE_UNROLL, s.kend);
            continue;
        }
        const float te = fminf(s.tmx, fminf(s.tmy, s.tmz));
        if (s.best_t < te - P.pad || !grid_move<CNT>(P, s, cnt)) {
            *(float2*)&W.ray[ray].l1 = make_float2(s.best_t, __int_as_float(s.best));
            have = false;
        }
    }
    flush_counts(P, bounces, cnt, CNT);
}

// HIT predicate (R7-R9) of one record against one segment, as a packed lexicographic key
// (t bits << 32 | id): t > 0 here, so the unsigned order of the key is the (t, id) order, and
// the nearest hit is the minimum key (~0 = no hit).  Same arithmetic as test_record.
[[maybe_unused]] __device__ __forceinline__ unsigned long long hit_key(const TP& P, const float4 o, const float4 d,
                                                      const float4 l0, const float4 l1,
                                                      const float4 A, const float4 B) {
    const int id = __float_as_int(B.w);
    const float wx = o.x - A.x, wy = o.y - A.y, wz = o.z - A.z;
    const float f0 = (wx * B.x + wy * B.y) + wz * B.z;
    const float dn = (d.x * B.x + d.y * B.y) + d.z * B.z;
    if (!(f0 * dn < 0.0f)) return ~0ull;
    {
        const float ex = __fmaf_rn(-f0, d.x, wx * dn), ey = __fmaf_rn(-f0, d.y, wy * dn),
                    ez = __fmaf_rn(-f0, d.z, wz * dn);
        const float rs = A.w + P.slack;
        if (__fmaf_rn(ex, ex, __fmaf_rn(ey, ey, ez * ez)) > rs * rs * (dn * dn)) return ~0ull;
    }
    if (id == __float_as_int(o.w)) return ~0ull;
    if (fabsf(f0) <= P.tau) {
        const float c0 = (B.x * l0.x + B.y * l0.y) + B.z * l0.z;
        const float c1 = (B.x * l1.x + B.y * l1.y) + B.z * l1.z;
        if (fabsf(c0) >= P.cos_ex || fabsf(c1) >= P.cos_ex) return ~0ull;
    }
    const float t = (-f0) / dn;
    const float hx = o.x + t * d.x, hy = o.y + t * d.y, hz = o.z + t * d.z;
    const float qx = hx - A.x, qy = hy - A.y, qz = hz - A.z;
    const float qq = (qx * qx + qy * qy) + qz * qz;
    if (!(qq <= A.w * A.w)) return ~0ull;
    return ((unsigned long long)__float_as_uint(t) << 32) | (unsigned)id;
}

// TRACE, warp-cooperative (NRT_TRACE_COOP=1; C5 trace 564 vs 358 ms per-lane): every lane walks its own segment through the grid
// (refill, Chebyshev jumps, early exit) until it stands in a non-empty cell; then the warp
// tests the union of the 32 lanes' cell ranges together — record g of the flattened list on
// lane g mod 32 (consecutive lanes read consecutive records: coalesced), against its owner's
// segment staged in shared memory, and the owner's nearest hit kept by a shared 64-bit
// atomicMin on the (t, id) key.  The argmin is order-independent, so the result is the
// per-lane kernel's, bit for bit.
template <bool CNT>
__global__ void __launch_bounds__(128, NRT_TRACE_MINB) k_trace_coop(TP P, Wave W, int b) {
    __shared__ float4 sray[4][4][32];  // [warp][o, d, l0, l1][lane]; o.w = previous surfel id
    __shared__ unsigned long long sbest[4][32];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned long long n = W.n_alive[b];
    const unsigned* alive = W.alive[b & 1];
    unsigned long long bounces = 0;
    Cnt cnt;
    Seg s;
    s.k = s.kend = 0;
    unsigned ray = 0;
    bool have = false, done = false;
    for (;;) {
        // ---- per lane: refill / walk until a non-empty cell (or no work left)
        while (!done) {
            if (!have) {
                const unsigned long long j = NRT_TRACE_FETCH(&W.ctr[b]);
                if (j >= n) {
                    done = true;
                    break;
                }
                ray = alive[j];
                const RayHot R = W.ray[ray];
                const float4 o = R.o, d = R.d, a = R.l0, c = R.l1;
                sray[wid][0][lane] = o;
                sray[wid][1][lane] = d;
                sray[wid][2][lane] = a;
                sray[wid][3][lane] = c;
                sbest[wid][lane] = ~0ull;
                s.o = make_float3(o.x, o.y, o.z);
                s.d = make_float3(d.x, d.y, d.z);
                ++bounces;
                if (!seg_begin<CNT>(P, s, cnt)) {
                    *(float2*)&W.ray[ray].l1 = make_float2(INFINITY, __int_as_float(-1));
                    continue;
                }
                have = true;
                if (s.k < s.kend) break;
            }
            const unsigned long long bk = sbest[wid][lane];
            const float bt = bk == ~0ull ? INFINITY : __uint_as_float((unsigned)(bk >> 32));
            const float te = fminf(s.tmx, fminf(s.tmy, s.tmz));
            if (bt < te - P.pad || !grid_move<CNT>(P, s, cnt)) {
                *(float2*)&W.ray[ray].l1 = make_float2(bt, __int_as_float(bk == ~0ull ? -1 : (int)(unsigned)bk));
                have = false;
                continue;
            }
            if (s.k < s.kend) break;
        }
        // ---- warp: test the union of the lanes' cell ranges
        const unsigned mine = (have && s.k < s.kend) ? s.kend - s.k : 0u;
        unsigned incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const unsigned total = __shfl_sync(0xffffffffu, incl, 31);
        if (total == 0) break;  // every lane is out of work
        for (unsigned g0 = 0; g0 < total; g0 += 32) {
            const unsigned g = g0 + lane;
            int lo = 0;  // owner: first lane whose inclusive prefix exceeds g
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const unsigned pm = __shfl_sync(0xffffffffu, incl, lo + step - 1);
                if (pm <= g) lo += step;
            }
            const unsigned excl = __shfl_sync(0xffffffffu, incl - mine, lo);
            const unsigned k0 = __shfl_sync(0xffffffffu, s.k, lo);
            if (g < total) {
                const unsigned k = k0 + (g - excl);
                const float4 A = __ldg(&P.rec[2 * k]), B = __ldg(&P.rec[2 * k + 1]);
                const unsigned long long key =
                    hit_key(P, sray[wid][0][lo], sray[wid][1][lo], sray[wid][2][lo], sray[wid][3][lo], A, B);
                if (key != ~0ull) atomicMin(&sbest[wid][lo], key);
            }
        }
        __syncwarp();
        if (mine) s.k = s.kend;
    }
    flush_counts(P, bounces, cnt, CNT);
}

// coherence key of a segment (origin h, direction d): Morton code of its coarse cell (6 bits
// per axis), then the octahedral direction (7 + 7 bits).  Only the processing order of the
// next bounce depends on it, never a result.
__device__ __forceinline__ unsigned spread3(unsigned x) {  // 6 bits -> every third bit
    x &= 63u;
    x = (x | (x << 8)) & 0x0000F00Fu;
    x = (x | (x << 4)) & 0x000C30C3u;
    x = (x | (x << 2)) & 0x00249249u;
    return x;
}
__device__ __forceinline__ unsigned order_key(const TP& P, float3 h, float3 d) {
    const unsigned cx = (unsigned)min(63, max(0, (int)((h.x - P.ox) * P.ok_inv)));
    const unsigned cy = (unsigned)min(63, max(0, (int)((h.y - P.oy) * P.ok_inv)));
    const unsigned cz = (unsigned)min(63, max(0, (int)((h.z - P.oz) * P.ok_inv)));
    const unsigned m = spread3(cx) | (spread3(cy) << 1) | (spread3(cz) << 2);
    const float sa = fabsf(d.x) + fabsf(d.y) + fabsf(d.z);
    float px = d.x / sa, py = d.y / sa;
    if (d.z < 0.0f) {
        const float qx = (1.0f - fabsf(py)) * (px < 0.0f ? -1.0f : 1.0f);
        const float qy = (1.0f - fabsf(px)) * (py < 0.0f ? -1.0f : 1.0f);
        px = qx;
        py = qy;
    }
    const unsigned u = (unsigned)min(127, max(0, (int)((px + 1.0f) * 64.0f)));
    const unsigned v = (unsigned)min(127, max(0, (int)((py + 1.0f) * 64.0f)));
    return min((m << 14) | (u << 7) | v, 0xFFFFFFFEu);  // 0xFFFFFFFF pads the sorted list
}


// =======================================================================================
// NEXT-1: the paper's point-set SDF intersection (DESIGN R40-R45, §6.4)
// =======================================================================================
// IEEE a / b with an exact shortcut for a zero dividend (+-0 with the quotient's sign): the
// hardware division's fast path rejects zero dividends (FCHK), and axis-aligned normals and
// ray origins on AABB faces make them common.  Bitwise the result of a / b.
__device__ __forceinline__ float div0(float a, float b) {
    const bool z = a == 0.0f;
    const float q = (z ? 1.0f : a) / b;  // branch-free: a zero dividend divides 1 instead
    return z ? __int_as_float((__float_as_int(a) ^ __float_as_int(b)) & 0x80000000) : q;
}

// R41: FP32 exp for x <= 0, the definition's fixed operation order (identical to the oracle's:
// Cody-Waite split and Horner steps as single-rounding FMAs); 0 below -87 (branch-free)
__device__ __forceinline__ float sdf_expf(float x) {
    const float kf = floorf(__fmaf_rn(x, 1.44269504f, 0.5f));
    float r = __fmaf_rn(kf, -0.693359375f, x);
    r = __fmaf_rn(kf, 2.12194440e-4f, r);
    float p = 1.98412698e-4f;
    p = __fmaf_rn(p, r, 1.38888889e-3f);
    p = __fmaf_rn(p, r, 8.33333333e-3f);
    p = __fmaf_rn(p, r, 4.16666667e-2f);
    p = __fmaf_rn(p, r, 1.66666667e-1f);
    p = __fmaf_rn(p, r, 0.5f);
    p = __fmaf_rn(p, r, 1.0f);
    p = __fmaf_rn(p, r, 1.0f);
    const float e = p * __int_as_float(((int)kf + 127) << 23);
    return x < -87.0f ? 0.0f : e;
}

// R41/R41b: f and nbar (unnormalised) of the AABB whose points are [k0, k1) at x; false = fails.
// Warp-cooperative (called by all 32 lanes with the same arguments).  The definition sums the
// terms in chunks of 32 points, each chunk by the pairwise tree (pairs i, i + s for s = 16, 8,
// 4, 2, 1), the chunk totals in ascending order.  Here half-warp h takes chunk 2m + h of
// iteration m; its lane i computes the terms of points i and i + 16 and adds them (tree level
// s = 16, in registers), then levels 8, 4, 2, 1 run across the half-warp's lanes as a
// multi-value butterfly (at s = 8 a lane keeps four of the eight quantities and trades the
// other four, at s = 4 two, at s = 2 one), so quantity q = (lane >> 1) & 7 ends in lanes 2q,
// 2q + 1 of both halves; the two chunk totals are added to the running sums in chunk order.
// Padding terms (past k1) are zero, as in the definition.
template <bool CNT>
__device__ __forceinline__ void sdf_accum(const TP& P, unsigned k0, unsigned k1, float x0, float x1, float x2,
                                          float& acc, Cnt& cnt) {
    const unsigned lane = threadIdx.x & 31, i = lane & 15, h = lane >> 4;
    if (CNT && lane == 0) cnt.tests += k1 - k0;  // Gaussian terms (the SDF mode's unit of work)
    const bool u8 = lane & 8, u4 = lane & 4, u2 = lane & 2;
    for (unsigned kb = k0; kb < k1; kb += 64) {
        if (k1 - kb <= 32) {
            // a single (last) chunk: one point per lane; tree levels 16, 8, 4 as a multi-value
            // butterfly (quantity bits = lane bits 4, 3, 2), levels 2, 1 plain, then one shuffle
            // moves quantity q to lanes with (lane >> 1) & 7 == q, the layout of `acc`
            const unsigned k = kb + lane;
            const unsigned kc = k < k1 ? k : k1 - 1;
            const float4 A = __ldg(&P.sdf_pts[2 * kc]), B = __ldg(&P.sdf_pts[2 * kc + 1]);
            const float d0 = A.x - x0, d1 = A.y - x1, d2 = A.z - x2;
            const float q = __fmaf_rn(d2, d2, __fmaf_rn(d1, d1, d0 * d0));
            const float w = k < k1 ? sdf_expf(-(q * P.sdf_inv)) : 0.0f;
            const float v[8] = {w, w * A.x, w * A.y, w * A.z, w * B.x, w * B.y, w * B.z, 0.0f};
            const bool u16 = lane & 16;
            float a[4], b2[2];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const float snd = u16 ? v[c] : v[c + 4], kp = u16 ? v[c + 4] : v[c];
                a[c] = kp + __shfl_xor_sync(0xffffffffu, snd, 16);
            }
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const float snd = u8 ? a[c] : a[c + 2], kp = u8 ? a[c + 2] : a[c];
                b2[c] = kp + __shfl_xor_sync(0xffffffffu, snd, 8);
            }
            float t = (u4 ? b2[1] : b2[0]) + __shfl_xor_sync(0xffffffffu, u4 ? b2[0] : b2[1], 4);
            t = t + __shfl_xor_sync(0xffffffffu, t, 2);
            t = t + __shfl_xor_sync(0xffffffffu, t, 1);
            const unsigned src = (((lane >> 3) & 1u) << 4) | (((lane >> 2) & 1u) << 3) | (((lane >> 1) & 1u) << 2);
            acc = acc + __shfl_sync(0xffffffffu, t, src);
            break;
        }
        float v[8];
        v[7] = 0.0f;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            const unsigned k = kb + 32 * h + i + 16 * half;
            const unsigned kc = k < k1 ? k : k1 - 1;  // padding: a valid load, weight 0
            const float4 A = __ldg(&P.sdf_pts[2 * kc]), B = __ldg(&P.sdf_pts[2 * kc + 1]);
            const float d0 = A.x - x0, d1 = A.y - x1, d2 = A.z - x2;
            const float q = __fmaf_rn(d2, d2, __fmaf_rn(d1, d1, d0 * d0));
            const float w = k < k1 ? sdf_expf(-(q * P.sdf_inv)) : 0.0f;
            const float t[7] = {w, w * A.x, w * A.y, w * A.z, w * B.x, w * B.y, w * B.z};
#pragma unroll
            for (int c = 0; c < 7; ++c) v[c] = half ? v[c] + t[c] : t[c];  // level s = 16
        }
        float a[4], b2[2];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const float snd = u8 ? v[c] : v[c + 4], kp = u8 ? v[c + 4] : v[c];
            a[c] = kp + __shfl_xor_sync(0xffffffffu, snd, 8);
        }
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const float snd = u4 ? a[c] : a[c + 2], kp = u4 ? a[c + 2] : a[c];
            b2[c] = kp + __shfl_xor_sync(0xffffffffu, snd, 4);
        }
        float t = (u2 ? b2[1] : b2[0]) + __shfl_xor_sync(0xffffffffu, u2 ? b2[0] : b2[1], 2);
        t = t + __shfl_xor_sync(0xffffffffu, t, 1);
        const float o = __shfl_xor_sync(0xffffffffu, t, 16);
        acc = acc + (h ? o : t);                  // chunk 2m
        if (kb + 32 < k1) acc = acc + (h ? t : o);  // chunk 2m + 1
    }
}

template <bool CNT>
__device__ __forceinline__ bool sdf_eval(const TP& P, unsigned k0, unsigned k1, float x0, float x1, float x2,
                                         float& f, float& nb0, float& nb1, float& nb2, Cnt& cnt) {
    float acc = 0.0f;
    sdf_accum<CNT>(P, k0, k1, x0, x1, x2, acc, cnt);
    const float W = __shfl_sync(0xffffffffu, acc, 0);
    if (!(W > 0.0f)) return false;
    const float p0 = __shfl_sync(0xffffffffu, acc, 2), p1 = __shfl_sync(0xffffffffu, acc, 4),
                p2 = __shfl_sync(0xffffffffu, acc, 6), n0 = __shfl_sync(0xffffffffu, acc, 8),
                n1 = __shfl_sync(0xffffffffu, acc, 10), n2 = __shfl_sync(0xffffffffu, acc, 12);
    const float b0 = div0(p0, W), b1 = div0(p1, W), b2 = div0(p2, W);
    nb0 = div0(n0, W);
    nb1 = div0(n1, W);
    nb2 = div0(n2, W);
    const float e0 = x0 - b0, e1 = x1 - b1, e2 = x2 - b2;
    f = (e0 * nb0 + e1 * nb1) + e2 * nb2;
    return true;
}

// R53 (NEXT-4): the unit normal of Eq. 3 at x over the points of the AABBs in the 3x3x3 cells
// around `cell` (warp-cooperative).  Rows (dz, dy) ascending; a row = the points of its cells
// x-1..x+1, one contiguous range of sdf_pts (AABBs of consecutive cells are consecutive), summed
// in chunks from the row's first point (R41b); rows added in order.  false if W <= 0.
template <bool CNT>
__device__ __forceinline__ bool sdf_normal27(const TP& P, unsigned cell, float x0, float x1, float x2,
                                             float& n0, float& n1, float& n2, Cnt& cnt) {
    const int dx = P.sd_n[0], dy = P.sd_n[1], dz = P.sd_n[2];
    const int cx = (int)(cell % (unsigned)dx), cy = (int)((cell / (unsigned)dx) % (unsigned)dy),
              cz = (int)(cell / ((unsigned)dx * (unsigned)dy));
    float acc = 0.0f;
    for (int oz = -1; oz <= 1; ++oz)
        for (int oy = -1; oy <= 1; ++oy) {
            const int y = cy + oy, z = cz + oz;
            if (y < 0 || y >= dy || z < 0 || z >= dz) continue;
            unsigned first = 0xffffffffu, last = 0;
            for (int ox = -1; ox <= 1; ++ox) {
                const int xx = cx + ox;
                if (xx < 0 || xx >= dx) continue;
                const uint2 r = __ldg(&P.sdf_crange[(size_t)xx + (size_t)dx * ((size_t)y + (size_t)dy * z)]);
                if (r.y > r.x) {
                    if (first == 0xffffffffu) first = r.x;
                    last = r.y;
                }
            }
            if (first != 0xffffffffu) sdf_accum<CNT>(P, first, last, x0, x1, x2, acc, cnt);
        }
    const float W = __shfl_sync(0xffffffffu, acc, 0);
    if (!(W > 0.0f)) return false;
    const float a0 = __shfl_sync(0xffffffffu, acc, 8), a1 = __shfl_sync(0xffffffffu, acc, 10),
                a2 = __shfl_sync(0xffffffffu, acc, 12);
    const float b0 = div0(a0, W), b1 = div0(a1, W), b2 = div0(a2, W);
    const float l = sqrtf((b0 * b0 + b1 * b1) + b2 * b2);
    if (!(l > 0.0f)) return false;
    n0 = div0(b0, l);
    n1 = div0(b1, l);
    n2 = div0(b2, l);
    return true;
}

// R42 slab test of AABB (L, H) against the ray (t >= 0): the entry tn, or -1 when it misses
__device__ __forceinline__ float sdf_slab(const float3 o, const float3 d, const float4 L, const float4 H) {
    float tn = 0.0f, tf = INFINITY;
    const float lo[3] = {L.x, L.y, L.z}, hi[3] = {H.x, H.y, H.z}, ov[3] = {o.x, o.y, o.z},
                dv[3] = {d.x, d.y, d.z};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        if (dv[k] != 0.0f) {
            float ta = (lo[k] - ov[k]) / dv[k], tb = (hi[k] - ov[k]) / dv[k];
            if (ta > tb) {
                const float t = ta;
                ta = tb;
                tb = t;
            }
            if (ta > tn) tn = ta;
            if (tb < tf) tf = tb;
        } else if (ov[k] < lo[k] || ov[k] > hi[k]) {
            return -1.0f;
        }
    }
    return tn <= tf ? tn : -1.0f;
}

// R42: the march of AABB (L, H) along the ray; true and t on a hit
template <bool CNT>
__device__ __forceinline__ bool sdf_march(const TP& P, const float3 o, const float3 d, const float4 L,
                                          const float4 H, float& t_hit, Cnt& cnt) {
    const unsigned k0 = __float_as_uint(L.w), k1 = __float_as_uint(H.w);
    const float c0 = 0.5f * (L.x + H.x), c1 = 0.5f * (L.y + H.y), c2 = 0.5f * (L.z + H.z);
    const float w0 = c0 - o.x, w1 = c1 - o.y, w2 = c2 - o.z;
    const float tc = (w0 * d.x + w1 * d.y) + w2 * d.z;
    float t = tc - P.sdf_half;
    const float te = tc + P.sdf_half;
    if (t < 0.0f) t = 0.0f;
    float f0, f1, nb0, nb1, nb2;
    bool ok0 = sdf_eval<CNT>(P, k0, k1, o.x + t * d.x, o.y + t * d.y, o.z + t * d.z, f0, nb0, nb1, nb2, cnt);
    for (int it = 0; it < 4096; ++it) {
        if (ok0 && fabsf(f0) < P.sdf_tsdf) {
            t_hit = t;
            return true;
        }
        const float step = ok0 ? fabsf(f0) : P.sdf_rs;
        const float t1 = t + step;
        if (t1 > te) return false;
        const bool ok1 =
            sdf_eval<CNT>(P, k0, k1, o.x + t1 * d.x, o.y + t1 * d.y, o.z + t1 * d.z, f1, nb0, nb1, nb2, cnt);
        if (ok0 && ok1 && ((f0 < 0.0f) != (f1 < 0.0f))) {
            t_hit = t + step * (f0 / (f0 - f1));
            return true;
        }
        t = t1;
        f0 = f1;
        ok0 = ok1;
    }
    return false;
}

// R43 departure sheet: the AABB is transparent when its SDF at the origin is defined with
// |f| <= tau and its unit normal lies within theta_ex of a departure normal (l0, l1; zero
// vectors stand for "no departure normal", which never excludes since cos_ex > 0)
template <bool CNT>
__device__ __forceinline__ bool sdf_excluded(const TP& P, const float3 o, const float3 l0, const float3 l1,
                                             const float4 L, const float4 H, Cnt& cnt) {
    float f, nb0, nb1, nb2;
    if (!sdf_eval<CNT>(P, __float_as_uint(L.w), __float_as_uint(H.w), o.x, o.y, o.z, f, nb0, nb1, nb2, cnt))
        return false;
    if (!(fabsf(f) <= P.tau)) return false;
    const float l = sqrtf((nb0 * nb0 + nb1 * nb1) + nb2 * nb2);
    if (!(l > 0.0f)) return false;
    const float u0 = div0(nb0, l), u1 = div0(nb1, l), u2 = div0(nb2, l);
    if (fabsf((u0 * l0.x + u1 * l0.y) + u2 * l0.z) >= P.cos_ex) return true;
    return fabsf((u0 * l1.x + u1 * l1.y) + u2 * l1.z) >= P.cos_ex;
}

#ifndef NRT_SDF_MINB
#define NRT_SDF_MINB 8  // k_trace_sdf, k_env_*: min resident blocks/SM (64 registers; A/B on C4 /
                        // C2 / C2 cone tracing, 4 / 6 / 8 / 10 / 12: 8 best, -9 / -14 / -15 % vs 4)
#endif
#ifndef NRT_GD_MINB
#define NRT_GD_MINB 4   // k_refine_gd (latency-bound per path: registers over occupancy)
#endif
// TRACE (SDF mode): one WARP per segment.  A 3D-DDA over the AABB traversal grid (Chebyshev
// jumps over empty cells), executed uniformly by the warp; in a non-empty cell the lanes slab-
// test the cell's registered AABBs in parallel, and the warp marches the candidates one after
// the other, each SDF evaluation spread over the lanes (sdf_eval).  AABB j is marched once per
// segment, in the non-empty cell whose interval [t_lo, t_out) holds its slab entry tn (t_lo =
// exit of the previous non-empty cell: the intervals tile the segment, and the padded
// registration puts j in that cell); the walk stops once best_t < t_out - (2 half + pad),
// below which no later AABB's march can start.  The hit is the lexicographic min (t, AABB
// index) = min (t, cell), as R43 defines it.
// R42/R43 (warp-cooperative): the nearest SDF hit of the ray (o, d) with departure normals
// l0, l1 (zero = none) and the previous hit's cell `prev` skipped; returns the AABB index (-1:
// escape) and best_t.  Called by all 32 lanes with the same arguments.
template <bool CNT>
// t_max (optional, exact): the caller only needs hits with t <= t_max; the walk then also stops
// once no AABB owned by a later cell can produce a hit before t_max (t_out - (L + pad) > t_max).
// Every hit with t <= t_max is found exactly; a returned hit with t > t_max may not be the first.
__device__ __forceinline__ int sdf_trace_w(const TP& P, const float3 o, const float3 d, const float3 l0,
                                           const float3 l1, const unsigned prev, float& best_t_out, Cnt& cnt,
                                           const float t_max = INFINITY) {
    const unsigned lane = threadIdx.x & 31;
    const bool has_lam = l0.x != 0.0f || l0.y != 0.0f || l0.z != 0.0f || l1.x != 0.0f || l1.y != 0.0f ||
                         l1.z != 0.0f;
    float best_t = INFINITY;
    int best = -1;
    // grid entry (uniform across the warp)
    const float ov[3] = {o.x, o.y, o.z}, dv[3] = {d.x, d.y, d.z};
    float inv[3], t0 = 0.0f, t1 = INFINITY;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        inv[k] = rcp_approx(dv[k]);  // walk only (§6.4)
        const float lo = P.sg_o[k], hi = P.sg_o[k] + (float)P.sg_n[k] * P.sdf_a;
        if (dv[k] != 0.0f) {
            const float ta = (lo - ov[k]) * inv[k], tb = (hi - ov[k]) * inv[k];
            t0 = fmaxf(t0, fminf(ta, tb));
            t1 = fminf(t1, fmaxf(ta, tb));
        } else if (ov[k] < lo || ov[k] > hi) {
            t1 = -1.0f;
        }
    }
    if (t0 <= t1) {
        int c[3];
        float tm[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float p = ov[k] + t0 * dv[k];
            c[k] = min(P.sg_n[k] - 1, max(0, (int)floorf((p - P.sg_o[k]) * P.sdf_inv_a)));
            tm[k] = dv[k] != 0.0f ? ((P.sg_o[k] + (float)(c[k] + (dv[k] > 0.0f)) * P.sdf_a) - ov[k]) * inv[k]
                                  : INFINITY;
        }
        float t_lo = t0;
        bool first = true;
        for (;;) {
            const float t_out = fminf(tm[0], fminf(tm[1], tm[2]));
            const uint2 rg = __ldg(&P.sdf_gcell[c[0] + P.sg_n[0] * (c[1] + P.sg_n[1] * c[2])]);
            if (CNT && lane == 0) cnt.cells++;
            int D = 1;
            if (rg.y > rg.x) {
                for (unsigned base = rg.x; base < rg.y; base += 32) {
                    // lanes: slab test + owner rule of one registered AABB each
                    const unsigned q = base + lane;
                    unsigned j = 0;
                    bool cand = false;
                    if (q < rg.y) {
                        j = __ldg(&P.sdf_aref[q]);
                        if (__ldg(&P.sdf_acell[j]) != prev) {
                            const float tn = sdf_slab(o, d, __ldg(&P.sdf_box[2 * j]), __ldg(&P.sdf_box[2 * j + 1]));
                            cand = tn >= 0.0f && (first || !(tn < t_lo)) && tn < t_out;  // owner cell only
                        }
                    }
                    unsigned m = __ballot_sync(0xffffffffu, cand);
                    while (m) {  // warp: march the candidates
                        const int src = __ffs(m) - 1;
                        m &= m - 1;
                        const unsigned jm = __shfl_sync(0xffffffffu, j, src);
                        if (CNT && lane == 0) cnt.nonempty++;  // SDF mode: AABB marches
                        const float4 L = __ldg(&P.sdf_box[2 * jm]), H = __ldg(&P.sdf_box[2 * jm + 1]);
                        float t;
                        if (!sdf_march<CNT>(P, o, d, L, H, t, cnt)) continue;
                        if (!(t < best_t || (t == best_t && (int)jm < best))) continue;
                        if (has_lam && sdf_excluded<CNT>(P, o, l0, l1, L, H, cnt)) continue;
                        best_t = t;
                        best = (int)jm;
                    }
                }
                first = false;
                t_lo = t_out;
            } else {
                D = (int)rg.x;
            }
            if (best_t < t_out - P.sdf_stop || t_out - P.sdf_stop > t_max) break;
            // grid move: DDA step, or a Chebyshev jump across the empty box (as k_trace)
            if (D <= 1) {
                const int ax = (tm[0] <= tm[1] && tm[0] <= tm[2]) ? 0 : (tm[1] <= tm[2] ? 1 : 2);
                const float dva = ax == 0 ? dv[0] : (ax == 1 ? dv[1] : dv[2]);
                int ca = (ax == 0 ? c[0] : (ax == 1 ? c[1] : c[2])) + (dva > 0.0f ? 1 : -1);
                const int na = ax == 0 ? P.sg_n[0] : (ax == 1 ? P.sg_n[1] : P.sg_n[2]);
                if (ca < 0 || ca >= na) break;
                const float oa = ax == 0 ? ov[0] : (ax == 1 ? ov[1] : ov[2]);
                const float ia = ax == 0 ? inv[0] : (ax == 1 ? inv[1] : inv[2]);
                const float ga = ax == 0 ? P.sg_o[0] : (ax == 1 ? P.sg_o[1] : P.sg_o[2]);
                const float tn = ((ga + (float)(ca + (dva > 0.0f)) * P.sdf_a) - oa) * ia;
                if (ax == 0) { c[0] = ca; tm[0] = tn; }
                else if (ax == 1) { c[1] = ca; tm[1] = tn; }
                else { c[2] = ca; tm[2] = tn; }
            } else {
                const int r = D - 1;
                float T = INFINITY;
                int ax = 0;
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    const int fk = dv[k] > 0.0f ? c[k] + r + 1 : c[k] - r;
                    const float Tk = dv[k] != 0.0f ? ((P.sg_o[k] + (float)fk * P.sdf_a) - ov[k]) * inv[k] : INFINITY;
                    if (Tk < T) {
                        T = Tk;
                        ax = k;
                    }
                }
                int nc[3];
                bool out = false;
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    const float pk = ov[k] + T * dv[k];
                    nc[k] = min(c[k] + r, max(c[k] - r, (int)floorf((pk - P.sg_o[k]) * P.sdf_inv_a)));
                    if (k == ax) nc[k] = dv[k] > 0.0f ? c[k] + r + 1 : c[k] - r - 1;
                    out |= nc[k] < 0 || nc[k] >= P.sg_n[k];
                }
                if (out) break;
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    c[k] = nc[k];
                    tm[k] = dv[k] != 0.0f
                                ? ((P.sg_o[k] + (float)(c[k] + (dv[k] > 0.0f)) * P.sdf_a) - ov[k]) * inv[k]
                                : INFINITY;
                }
            }
        }
    }
    best_t_out = best_t;
    return best;
}

// R44 (warp-cooperative): the unit MLS normal at the hit (zero if undefined, cell bits in .w)
// and the AABB's point nearest to the hit point (its id)
template <bool CNT>
__device__ __forceinline__ void sdf_hit_attr(const TP& P, const int best, const float best_t, const float3 o,
                                             const float3 d, float4& hn_out, int& pid_out, Cnt& cnt) {
    const unsigned lane = threadIdx.x & 31;
    int pid = -1;
    float4 hn = make_float4(0.0f, 0.0f, 0.0f, __uint_as_float(~0u));
    if (best >= 0) {
        // R44: normal nbar(x*)/|nbar(x*)|; record point = the AABB's point nearest x*
        const float4 L = __ldg(&P.sdf_box[2 * best]), H = __ldg(&P.sdf_box[2 * best + 1]);
        const unsigned k0 = __float_as_uint(L.w), k1 = __float_as_uint(H.w);
        const float x0 = o.x + best_t * d.x, x1 = o.y + best_t * d.y, x2 = o.z + best_t * d.z;
        float f, nb0, nb1, nb2;
        if (sdf_eval<CNT>(P, k0, k1, x0, x1, x2, f, nb0, nb1, nb2, cnt)) {
            const float l = sqrtf((nb0 * nb0 + nb1 * nb1) + nb2 * nb2);
            if (l > 0.0f) {
                hn.x = div0(nb0, l);
                hn.y = div0(nb1, l);
                hn.z = div0(nb2, l);
            }
        }
        // warp argmin of (q, k): per lane ascending k with strict <, then lexicographic
        float bq = INFINITY;
        unsigned bk = 0xffffffffu;
        for (unsigned k = k0 + lane; k < k1; k += 32) {
            const float4 A = __ldg(&P.sdf_pts[2 * k]);
            const float e0 = A.x - x0, e1 = A.y - x1, e2 = A.z - x2;
            const float q = (e0 * e0 + e1 * e1) + e2 * e2;
            if (q < bq) {
                bq = q;
                bk = k;
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const float oq = __shfl_xor_sync(0xffffffffu, bq, off);
            const unsigned ok = __shfl_xor_sync(0xffffffffu, bk, off);
            if (oq < bq || (oq == bq && ok < bk)) {
                bq = oq;
                bk = ok;
            }
        }
        pid = __float_as_int(__ldg(&P.sdf_pts[2 * bk + 1]).w);
        hn.w = __uint_as_float(__ldg(&P.sdf_acell[best]));
    }
    hn_out = hn;
    pid_out = pid;
}

template <bool CNT>
__global__ void __launch_bounds__(128, NRT_SDF_MINB) k_trace_sdf(TP P, Wave W, int b) {
    const unsigned long long n = W.n_alive[b];
    const unsigned* alive = W.alive[b & 1];
    const unsigned lane = threadIdx.x & 31;
    unsigned long long bounces = 0;
    Cnt cnt;
    for (;;) {
        unsigned long long jj = 0;
        if (lane == 0) jj = atomicAdd(&W.ctr[b], 1ull);
        jj = __shfl_sync(0xffffffffu, jj, 0);
        if (jj >= n) break;
        const unsigned ray = alive[jj];
        if (lane == 0) ++bounces;
        const RayHot R = W.ray[ray];
        const float4 o4 = R.o, d4 = R.d, a4 = R.l0, c4 = R.l1;
        const float3 o = make_float3(o4.x, o4.y, o4.z), d = make_float3(d4.x, d4.y, d4.z);
        const float3 l0 = make_float3(a4.x, a4.y, a4.z), l1 = make_float3(c4.x, c4.y, c4.z);
        const unsigned prev = __float_as_uint(o4.w);  // cell of the previous hit (~0: none)
        float best_t;
        const int best = sdf_trace_w<CNT>(P, o, d, l0, l1, prev, best_t, cnt);
        float4 hn;
        int pid;
        sdf_hit_attr<CNT>(P, best, best_t, o, d, hn, pid, cnt);
        if (lane == 0) {
            *(float2*)&W.ray[ray].l1 = make_float2(best >= 0 ? best_t : INFINITY, __int_as_float(pid));
            W.hitn[ray] = hn;
        }
    }
    flush_counts(P, bounces, cnt, CNT);
}

// =======================================================================================
// NEXT-4: the paper's gradient-descent refinement (Tables I-III; DESIGN R50-R56)
// =======================================================================================
// One warp per coarse path; every lane computes the same scalars (uniform control flow), the
// warp-cooperative pieces are the reprojection traces (sdf_trace_w), the hit attributes and
// the 27-cell normals.  FP32 throughout, every operation in the oracle's order (gd.c).
struct GdArgs {
    const nrt_coarse_rec* in;
    int64_t n_in;
    int rank, world;
    nrt_refined_rec* out;
    unsigned long long* n_ok;   // valid records written (keep_invalid == 0)
    unsigned long long* work;   // path counter
    unsigned long long* terms;  // Gaussian terms (counters)
    int keep_invalid;
    const float* rx;
    float tx[3];
    int rho;
    float alpha, beta, delta, t_d, cos_ta, margin;  // margin = 2 sigma (R56)
};

struct GdVert {  // per-warp shared state of one interaction (written identically by all lanes)
    float x[3], n[3], u[3], v[3], w[3], a[3];
    float len;
    unsigned cell;
    int pid, kind, edge;
};

__device__ __forceinline__ float gd_dot(const float* a, const float* b) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }

// R54
__device__ __forceinline__ void gd_basis(const float* n, float* u, float* v) {
    int ax = 0;
    if (fabsf(n[1]) < fabsf(n[ax])) ax = 1;
    if (fabsf(n[2]) < fabsf(n[ax])) ax = 2;
    const float a0 = ax == 0 ? 1.0f : 0.0f, a1 = ax == 1 ? 1.0f : 0.0f, a2 = ax == 2 ? 1.0f : 0.0f;
    const float c0 = n[1] * a2 - n[2] * a1, c1 = n[2] * a0 - n[0] * a2, c2 = n[0] * a1 - n[1] * a0;
    const float l = sqrtf((c0 * c0 + c1 * c1) + c2 * c2);
    u[0] = div0(c0, l);
    u[1] = div0(c1, l);
    u[2] = div0(c2, l);
    v[0] = n[1] * u[2] - n[2] * u[1];
    v[1] = n[2] * u[0] - n[0] * u[2];
    v[2] = n[0] * u[1] - n[1] * u[0];
}

__device__ __forceinline__ float gd_fk(const float* y, const float* P, const float* Q) {
    const float e1[3] = {y[0] - Q[0], y[1] - Q[1], y[2] - Q[2]};
    const float e2[3] = {y[0] - P[0], y[1] - P[1], y[2] - P[2]};
    return sqrtf(gd_dot(e1, e1)) + sqrtf(gd_dot(e2, e2));
}
__device__ __forceinline__ float gd_grad(const float* x, const float* P, const float* Q, float* g) {
    const float e1[3] = {x[0] - Q[0], x[1] - Q[1], x[2] - Q[2]};
    const float e2[3] = {x[0] - P[0], x[1] - P[1], x[2] - P[2]};
    const float l1 = sqrtf(gd_dot(e1, e1)), l2 = sqrtf(gd_dot(e2, e2));
#pragma unroll
    for (int i = 0; i < 3; ++i) g[i] = e1[i] / l1 + e2[i] / l2;
    return l1 + l2;
}

// the SDF trace from vertex j (0 = TX) toward direction d: departure rule of vertex j (R55)
template <bool CNT>
__device__ __forceinline__ int gd_trace(const TP& P, const GdVert* V, int j, const float* o, const float* d,
                                        float& t, Cnt& cnt, const float t_max = INFINITY) {
    float3 l0 = make_float3(0.0f, 0.0f, 0.0f), l1 = l0;
    unsigned prev = ~0u;
    if (j > 0) {
        const GdVert& A = V[j - 1];
        if (A.kind == 0) {
            l0 = l1 = make_float3(A.n[0], A.n[1], A.n[2]);
            prev = A.cell;
        } else {
            const DevEdge& E = P.edges[A.edge];
            l0 = make_float3(E.n0[0], E.n0[1], E.n0[2]);
            l1 = make_float3(E.n1[0], E.n1[1], E.n1[2]);
        }
    }
    return sdf_trace_w<CNT>(P, make_float3(o[0], o[1], o[2]), make_float3(d[0], d[1], d[2]), l0, l1, prev, t, cnt,
                            t_max);
}

template <bool CNT>
__global__ void __launch_bounds__(128, NRT_GD_MINB) k_refine_gd(TP P, GdArgs A) {
    __shared__ GdVert sv[4][NRT_MAX_INT];
    const unsigned lane = threadIdx.x & 31;
    GdVert* V = sv[threadIdx.x >> 5];
    Cnt cnt;
    const int64_t n_mine = A.n_in > A.rank ? (A.n_in - A.rank + A.world - 1) / A.world : 0;
    for (;;) {
        unsigned long long jq = 0;
        if (lane == 0) jq = atomicAdd(A.work, 1ull);
        jq = __shfl_sync(0xffffffffu, jq, 0);
        if ((int64_t)jq >= n_mine) break;
        const nrt_coarse_rec& c = A.in[A.rank + (int64_t)jq * A.world];
        const int N = c.n_int;
        const float TX[3] = {A.tx[0], A.tx[1], A.tx[2]};
        const float RX[3] = {A.rx[3 * c.rx], A.rx[3 * c.rx + 1], A.rx[3 * c.rx + 2]};
        int status = NRT_REF_OK;
        // R50
        for (int k = 0; k < N; ++k) {
            GdVert& Vk = V[k];
            for (int i = 0; i < 3; ++i) Vk.n[i] = Vk.u[i] = Vk.v[i] = Vk.w[i] = Vk.a[i] = 0.0f;
            Vk.len = 0.0f;
            Vk.x[0] = c.v[k][0];
            Vk.x[1] = c.v[k][1];
            Vk.x[2] = c.v[k][2];
            if ((c.kinds >> k) & 1) {
                const DevEdge& E = P.edges[c.prim[k]];
                Vk.kind = 1;
                Vk.edge = (int)c.prim[k];
                for (int i = 0; i < 3; ++i) {
                    Vk.w[i] = E.e[i];
                    Vk.a[i] = E.a[i];
                }
                Vk.len = E.len;
            } else {
                Vk.kind = 0;
                Vk.pid = (int)c.prim[k];
                // R40 cell of the record point
                const float4 p = __ldg(&P.sn_p[c.prim[k]]);
                const float pp[3] = {p.x, p.y, p.z};
                int ci[3];
                for (int i = 0; i < 3; ++i)
                    ci[i] = min(P.sd_n[i] - 1, max(0, (int)floorf((pp[i] - P.sd_o[i]) / P.sdf_a)));
                Vk.cell = (unsigned)(ci[0] + P.sd_n[0] * (ci[1] + P.sd_n[1] * ci[2]));
            }
            __syncwarp();
            if (Vk.kind == 0) {
                float n0, n1, n2;
                if (!sdf_normal27<CNT>(P, Vk.cell, Vk.x[0], Vk.x[1], Vk.x[2], n0, n1, n2, cnt)) {
                    status = NRT_REF_NO_SUPPORT;
                } else {
                    Vk.n[0] = n0;
                    Vk.n[1] = n1;
                    Vk.n[2] = n2;
                    gd_basis(Vk.n, Vk.u, Vk.v);
                }
            }
            __syncwarp();
        }
        int it = 0;
        for (; it < A.rho && status == NRT_REF_OK; ++it) {
            for (int k = 0; k < N && status == NRT_REF_OK; ++k) {  // R51
                GdVert& Vk = V[k];
                float Pp[3], Qq[3], x[3];
                for (int i = 0; i < 3; ++i) {
                    Pp[i] = k == 0 ? TX[i] : V[k - 1].x[i];
                    Qq[i] = k == N - 1 ? RX[i] : V[k + 1].x[i];
                    x[i] = Vk.x[i];
                }
                float g[3], y[3];
                const float f0 = gd_grad(x, Pp, Qq, g);
                if (Vk.kind == 0) {
                    const float gu = gd_dot(g, Vk.u), gv = gd_dot(g, Vk.v);
                    const float slope = -(gu * gu + gv * gv);
                    float gam = 1.0f;
                    bool ok = false;
                    for (int s = 0; s < 64; ++s) {
                        const float du = -gu * gam, dv = -gv * gam;
                        for (int i = 0; i < 3; ++i) y[i] = (x[i] + du * Vk.u[i]) + dv * Vk.v[i];
                        if (!(gd_fk(y, Pp, Qq) > f0 + (A.alpha * gam) * slope)) {
                            ok = true;
                            break;
                        }
                        gam = A.beta * gam;
                    }
                    if (!ok)
                        for (int i = 0; i < 3; ++i) y[i] = x[i];
                    // R55: reproject by tracing from I_{k-1} toward y
                    float d[3] = {y[0] - Pp[0], y[1] - Pp[1], y[2] - Pp[2]};
                    const float ld = sqrtf(gd_dot(d, d));
                    for (int i = 0; i < 3; ++i) d[i] = d[i] / ld;
                    float t;
                    const int best = gd_trace<CNT>(P, V, k, Pp, d, t, cnt);
                    if (best < 0) {
                        status = NRT_REF_NO_SUPPORT;
                        break;
                    }
                    float4 hn;
                    int pid;
                    sdf_hit_attr<CNT>(P, best, t, make_float3(Pp[0], Pp[1], Pp[2]), make_float3(d[0], d[1], d[2]),
                                      hn, pid, cnt);
                    const float xn[3] = {Pp[0] + t * d[0], Pp[1] + t * d[1], Pp[2] + t * d[2]};
                    const unsigned cell = __ldg(&P.sdf_acell[best]);
                    float nn[3];
                    float nu[3] = {Vk.n[0], Vk.n[1], Vk.n[2]}, uu[3] = {Vk.u[0], Vk.u[1], Vk.u[2]},
                          vv[3] = {Vk.v[0], Vk.v[1], Vk.v[2]};
                    if (sdf_normal27<CNT>(P, cell, xn[0], xn[1], xn[2], nn[0], nn[1], nn[2], cnt)) {
                        const float dx[3] = {xn[0] - x[0], xn[1] - x[1], xn[2] - x[2]};
                        const float dist = fabsf(gd_dot(dx, nu));
                        const float ca = gd_dot(nu, nn);
                        if (!(dist < A.t_d && ca > A.cos_ta)) {
                            for (int i = 0; i < 3; ++i) nu[i] = nn[i];
                            gd_basis(nu, uu, vv);
                        }
                    }
                    __syncwarp();
                    for (int i = 0; i < 3; ++i) {
                        Vk.x[i] = xn[i];
                        Vk.n[i] = nu[i];
                        Vk.u[i] = uu[i];
                        Vk.v[i] = vv[i];
                    }
                    Vk.cell = cell;
                    Vk.pid = pid;
                    __syncwarp();
                } else {
                    const float gw = gd_dot(g, Vk.w);
                    const float slope = -(gw * gw);
                    float gam = 1.0f;
                    bool ok = false;
                    for (int s = 0; s < 64; ++s) {
                        const float dw = -gw * gam;
                        for (int i = 0; i < 3; ++i) y[i] = x[i] + dw * Vk.w[i];
                        if (!(gd_fk(y, Pp, Qq) > f0 + (A.alpha * gam) * slope)) {
                            ok = true;
                            break;
                        }
                        gam = A.beta * gam;
                    }
                    if (!ok)
                        for (int i = 0; i < 3; ++i) y[i] = x[i];
                    const float ya[3] = {y[0] - Vk.a[0], y[1] - Vk.a[1], y[2] - Vk.a[2]};
                    const float s = gd_dot(ya, Vk.w);
                    if (!(s >= 0.0f && s <= Vk.len)) {  // R52
                        status = NRT_REF_OFF_EDGE;
                        break;
                    }
                    __syncwarp();
                    for (int i = 0; i < 3; ++i) Vk.x[i] = y[i];
                    __syncwarp();
                }
            }
        }
        // R56
        float gs = 0.0f;
        for (int k = 0; k < N; ++k) {
            float Pp[3], Qq[3], g[3];
            for (int i = 0; i < 3; ++i) {
                Pp[i] = k == 0 ? TX[i] : V[k - 1].x[i];
                Qq[i] = k == N - 1 ? RX[i] : V[k + 1].x[i];
            }
            gd_grad(V[k].x, Pp, Qq, g);
            if (V[k].kind == 0) {
                const float gu = gd_dot(g, V[k].u), gv = gd_dot(g, V[k].v);
                gs = gs + (gu * gu + gv * gv);
            } else {
                const float gw = gd_dot(g, V[k].w);
                gs = gs + gw * gw;
            }
        }
        if (status == NRT_REF_OK && !(gs < A.delta)) status = NRT_REF_NO_CONVERGE;
        for (int j = 0; j <= N && status == NRT_REF_OK; ++j) {
            const float* o = j == 0 ? TX : V[j - 1].x;
            const float* to = j == N ? RX : V[j].x;
            float d[3] = {to[0] - o[0], to[1] - o[1], to[2] - o[2]};
            const float L = sqrtf(gd_dot(d, d));
            for (int i = 0; i < 3; ++i) d[i] = d[i] / L;
            float t;
            float oo[3] = {o[0], o[1], o[2]};
            if (gd_trace<CNT>(P, V, j, oo, d, t, cnt, L) >= 0 && t < L - A.margin) status = NRT_REF_OCCLUDED;
        }
        // output (FP64 from the FP32 points, as the oracle)
        if (lane == 0 && (A.keep_invalid || status == NRT_REF_OK)) {
            nrt_refined_rec r;
            memset(&r, 0, sizeof(r));
            r.rx = c.rx;
            r.n_int = c.n_int;
            r.n_diff = c.n_diff;
            r.kinds = c.kinds;
            r.ray_id = c.ray_id;
            r.status = status;
            r.iters = it;
            r.gradsq = (double)gs;
            double I[NRT_MAX_INT + 2][3];
            for (int i = 0; i < 3; ++i) {
                I[0][i] = TX[i];
                I[N + 1][i] = RX[i];
            }
            for (int k = 0; k < N; ++k) {
                for (int i = 0; i < 3; ++i) {
                    I[k + 1][i] = V[k].x[i];
                    r.v[k][i] = V[k].x[i];
                }
                if (V[k].kind == 0) {
                    r.prim[k] = (uint32_t)V[k].pid;
                    r.label[k] = __ldg(&P.label[V[k].pid]);
                } else {
                    r.prim[k] = c.prim[k];
                    r.label[k] = c.label[k];
                }
            }
            double L = 0.0;
            for (int j = 0; j <= N; ++j) {
                const double s0 = I[j + 1][0] - I[j][0], s1 = I[j + 1][1] - I[j][1], s2 = I[j + 1][2] - I[j][2];
                L += sqrt(s0 * s0 + s1 * s1 + s2 * s2);
            }
            r.L = L;
            r.delay = L / 299792458.0;
            const double d0[3] = {I[1][0] - I[0][0], I[1][1] - I[0][1], I[1][2] - I[0][2]};
            const double l0 = sqrt(d0[0] * d0[0] + d0[1] * d0[1] + d0[2] * d0[2]);
            const double dl[3] = {I[N][0] - I[N + 1][0], I[N][1] - I[N + 1][1], I[N][2] - I[N + 1][2]};
            const double ll = sqrt(dl[0] * dl[0] + dl[1] * dl[1] + dl[2] * dl[2]);
            const double R2D = 180.0 / 3.14159265358979323846;
            r.aod_az = (float)(atan2(d0[1], d0[0]) * R2D);
            r.aod_el = (float)(asin(fmax(-1.0, fmin(1.0, d0[2] / l0))) * R2D);
            r.aoa_az = (float)(atan2(dl[1], dl[0]) * R2D);
            r.aoa_el = (float)(asin(fmax(-1.0, fmin(1.0, dl[2] / ll))) * R2D);
            for (int k = 0; k < N; ++k) {
                const double din[3] = {I[k + 1][0] - I[k][0], I[k + 1][1] - I[k][1], I[k + 1][2] - I[k][2]};
                const double l = sqrt(din[0] * din[0] + din[1] * din[1] + din[2] * din[2]);
                const float* ax = V[k].kind == 0 ? V[k].n : V[k].w;
                double c2 = (din[0] * ax[0] + din[1] * ax[1] + din[2] * ax[2]) / l;
                if (V[k].kind == 0) c2 = fabs(c2);
                r.inc[k] = (float)(acos(fmax(-1.0, fmin(1.0, c2))) * R2D);
            }
            const unsigned long long at = A.keep_invalid ? jq : atomicAdd(A.n_ok, 1ull);
            A.out[at] = r;
        }
        __syncwarp();
    }
    if (CNT && A.terms) {
        unsigned long long t = cnt.tests;
        for (int off = 16; off > 0; off >>= 1) t += __shfl_down_sync(0xffffffffu, t, off);
        if (lane == 0 && t) atomicAdd(A.terms, t);
    }
}

// =======================================================================================
// NEXT-2: the paper's environment-driven launch + voxel cone tracing (P:86-95, P:145-180,
// Alg. 1; DESIGN R60-R67).  Level-synchronous wavefront of cone rays: level 0 is the
// transmission (one work item per IE), level k the cone rays spawned at level k-1.  One warp per
// item; every candidate is validated by the warp SDF trace of NEXT-1.
// =======================================================================================
struct EHist {
    int n, n_diff, n_refl;
    unsigned kinds;
    int label[NRT_MAX_INT];
    unsigned prim[NRT_MAX_INT];
    float v[NRT_MAX_INT][3];
    float s_edge;
    unsigned long long hash;
};
struct CRay {
    float o[3], d[3], nf[3], nlo[3], nhi[3], lam[6];
    int kind, n_lam;
    unsigned prev;
    int src;
    float L;
    EHist h;
};
struct EnvIE {
    float p[3];
    int kind, label, ref;
    int sub[3];
    float s_edge;
};
struct EnvArgs {
    const EnvIE* ie;
    int n_ie;
    const int* pc_of_sub;
    const int* vstart;
    const int* vids;
    const int* march;
    int vd[3], sv[3], sd[3];
    float org[3], V, S, a, tan_c, sec_c;
    float tx[3];
    int max_refl, max_diff;
    float dphi_deg;
    int rank, world;
    // queues
    const CRay* in;
    unsigned long long n_in;
    CRay* out;
    unsigned long long out_cap;
    unsigned long long* n_out;
    unsigned long long* work;
    unsigned long long* rays;  // validation traces
    unsigned long long* terms; // Gaussian terms (counters)
    nrt_coarse_rec* raw;
    unsigned long long raw_cap;
    unsigned long long* raw_n;
};

__device__ __forceinline__ unsigned long long env_mix(unsigned long long h, unsigned long long v) {
    return (h ^ v) * 1099511628211ull;
}
__device__ __forceinline__ float e_dot(const float* a, const float* b) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }

// R62
__device__ __forceinline__ bool env_cone_sphere(const float* o, const float* d, float tan_c, float sec_c, const float* c,
                                                float r) {
    const float v[3] = {c[0] - o[0], c[1] - o[1], c[2] - o[2]};
    const float t = e_dot(v, d);
    if (t < -r) return false;
    const float w[3] = {v[0] - t * d[0], v[1] - t * d[1], v[2] - t * d[2]};
    return sqrtf(e_dot(w, w)) <= t * tan_c + r * sec_c;
}

// Alg. 1
__device__ __forceinline__ void env_march(float* vpos, const float* dir, int a_dist) {
    float T[3];
#pragma unroll
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
#pragma unroll
    for (int k = 0; k < 3; ++k) vpos[k] = vpos[k] + dir[k] * st;
}

__device__ void env_emit(const EnvArgs& A, const EHist& h, int rx, float L) {
    const unsigned long long slot = atomicAdd(A.raw_n, 1ull);
    if (slot >= A.raw_cap) return;
    nrt_coarse_rec c;
    memset(&c, 0, sizeof(c));
    c.rx = (uint32_t)rx;
    c.n_int = (uint8_t)h.n;
    c.n_diff = (uint8_t)h.n_diff;
    c.kinds = (uint16_t)h.kinds;
    for (int k = 0; k < h.n; ++k) {
        c.label[k] = h.label[k];
        c.prim[k] = h.prim[k];
        c.v[k][0] = h.v[k][0];
        c.v[k][1] = h.v[k][1];
        c.v[k][2] = h.v[k][2];
    }
    c.s_edge = h.s_edge;
    c.L = L;
    c.ray_id = env_mix(h.hash, (1ull << 62) | (unsigned long long)rx) & ~(1ull << 63);
    A.raw[slot] = c;
}

__device__ __forceinline__ CRay* env_push(const EnvArgs& A) {
    const unsigned long long slot = atomicAdd(A.n_out, 1ull);
    return slot < A.out_cap ? &A.out[slot] : nullptr;
}

// R66 + R65 for IE i from source o (departure normals lam / n_lam, previous cell) with history
// h and length L0 so far.  Called by the whole warp (uniform); lane 0 writes children/records.
template <bool CNT>
__device__ void env_try_ie(const TP& P, const EnvArgs& A, const EHist& h, const float* o, const float* lam, int n_lam,
                           unsigned prev, int i, float L0, Cnt& cnt) {
    const unsigned lane = threadIdx.x & 31;
    const EnvIE I = A.ie[i];
    // R66: an interaction the caps do not allow is not validated
    if (I.kind == 0 && (h.n_refl >= A.max_refl || h.n >= NRT_MAX_INT)) return;
    if (I.kind == 1 && (h.n_diff >= A.max_diff || h.n >= NRT_MAX_INT)) return;
    const float dv[3] = {I.p[0] - o[0], I.p[1] - o[1], I.p[2] - o[2]};
    const float Ls = sqrtf(e_dot(dv, dv));
    if (!(Ls > 0.0f)) return;
    const float d[3] = {dv[0] / Ls, dv[1] / Ls, dv[2] / Ls};
    float3 l0 = make_float3(0.0f, 0.0f, 0.0f), l1 = l0;
    if (n_lam == 1) l0 = l1 = make_float3(lam[0], lam[1], lam[2]);
    if (n_lam == 2) {
        l0 = make_float3(lam[0], lam[1], lam[2]);
        l1 = make_float3(lam[3], lam[4], lam[5]);
    }
    if (lane == 0) atomicAdd(A.rays, 1ull);
    // the validation only needs hits up to: the receiver / the edge point; for a PCIE the first
    // hit, if it lies in one of its AABBs, is within Ls + S sqrt3 (subvoxel) + L (march window)
    const float t_max = I.kind == 0 ? Ls + (A.S * 1.7320508f + 2.0f * P.sdf_stop) : Ls;
    float t;
    const int best = sdf_trace_w<CNT>(P, make_float3(o[0], o[1], o[2]), make_float3(d[0], d[1], d[2]), l0, l1, prev, t,
                                      cnt, t_max);
    if (I.kind == 2) {  // RXIE
        if (best >= 0 && t < Ls) return;
        if (lane == 0) env_emit(A, h, I.ref, L0 + Ls);
        return;
    }
    if (I.kind == 1) {  // DEIE
        if (best >= 0 && t < Ls - 0.5f * A.a) return;
        if (h.n_diff >= A.max_diff || h.n >= NRT_MAX_INT) return;
        const DevEdge& E = P.edges[I.ref];
        const float ev[3] = {E.b_[0] - E.a[0], E.b_[1] - E.a[1], E.b_[2] - E.a[2]};
        const float len = sqrtf(e_dot(ev, ev));
        const float e[3] = {ev[0] / len, ev[1] / len, ev[2] / len};
        const double ct = (double)e_dot(d, e);
        const double st = sqrt(fmax(0.0, 1.0 - ct * ct));
        if (st < 1e-6) return;
        const int M0 = (int)ceil((double)E.n_exp * 180.0 / (double)A.dphi_deg);
        int M = (int)ceil((double)M0 * st);
        if (M < 1) M = 1;
        const double wedge = (double)E.n_exp * 3.14159265358979311600;
        if (lane != 0) return;
        for (int m = 0; m < M; ++m) {
            CRay* R = env_push(A);
            if (!R) continue;
            CRay r;
            r.h = h;
            r.h.label[r.h.n] = I.label;
            r.h.prim[r.h.n] = (unsigned)I.ref;
            for (int k = 0; k < 3; ++k) r.h.v[r.h.n][k] = I.p[k];
            r.h.kinds = r.h.kinds | (1u << r.h.n);
            r.h.n++;
            r.h.n_diff++;
            r.h.s_edge = I.s_edge;
            r.h.hash = env_mix(h.hash, ((unsigned long long)i << 12) | (unsigned long long)(m + 1));
            r.kind = 1;
            double sp, cp, sl, cl, sh, ch;
            nrt_sincos((((double)m + 0.5) * wedge) / (double)M, &sp, &cp);
            nrt_sincos(((double)m * wedge) / (double)M, &sl, &cl);
            nrt_sincos((((double)m + 1.0) * wedge) / (double)M, &sh, &ch);
            for (int k = 0; k < 3; ++k) {
                const double x2 = cp * (double)E.t0[k] + sp * (double)E.n0[k];
                r.d[k] = (float)(x2 * st + (double)e[k] * ct);
                r.nlo[k] = (float)(-sl * (double)E.t0[k] + cl * (double)E.n0[k]);
                r.nhi[k] = (float)(sh * (double)E.t0[k] - ch * (double)E.n0[k]);
                r.o[k] = I.p[k];
                r.nf[k] = 0.0f;
                r.lam[k] = E.n0[k];
                r.lam[3 + k] = E.n1[k];
            }
            r.n_lam = 2;
            r.prev = ~0u;
            r.src = i;
            r.L = L0 + Ls;
            *R = r;
        }
        return;
    }
    // PCIE: the first hit must lie in one of its AABBs (within t_max, see above)
    if (best < 0 || t > t_max) return;
    const unsigned cell = __ldg(&P.sdf_acell[best]);
    {
        const int c0 = (int)(cell % (unsigned)A.sd[0]), c1 = (int)((cell / (unsigned)A.sd[0]) % (unsigned)A.sd[1]),
                  c2 = (int)(cell / ((unsigned)A.sd[0] * (unsigned)A.sd[1]));
        const int s = c0 / 4 + A.sv[0] * (c1 / 4 + A.sv[1] * (c2 / 4));
        if (A.pc_of_sub[s] != i) return;
    }
    if (h.n_refl >= A.max_refl || h.n >= NRT_MAX_INT) return;
    float4 hn;
    int pid;
    sdf_hit_attr<CNT>(P, best, t, make_float3(o[0], o[1], o[2]), make_float3(d[0], d[1], d[2]), hn, pid, cnt);
    if (lane != 0) return;
    CRay* R = env_push(A);
    if (!R) return;
    CRay r;
    r.h = h;
    const float x[3] = {o[0] + t * d[0], o[1] + t * d[1], o[2] + t * d[2]};
    r.h.label[r.h.n] = I.label;
    r.h.prim[r.h.n] = (unsigned)pid;
    for (int k = 0; k < 3; ++k) r.h.v[r.h.n][k] = x[k];
    r.h.n++;
    r.h.n_refl++;
    r.h.hash = env_mix(h.hash, (unsigned long long)i << 12);
    r.kind = 0;
    const float nh[3] = {hn.x, hn.y, hn.z};
    const float k2 = 2.0f * e_dot(d, nh);
    const float xr[3] = {d[0] - k2 * nh[0], d[1] - k2 * nh[1], d[2] - k2 * nh[2]};
    const float l = sqrtf(e_dot(xr, xr));
    for (int k = 0; k < 3; ++k) r.d[k] = xr[k] / l;
    const float sg = e_dot(r.d, nh) >= 0.0f ? 1.0f : -1.0f;
    for (int k = 0; k < 3; ++k) {
        r.o[k] = x[k];
        r.nf[k] = sg * nh[k];
        r.lam[k] = nh[k];
        r.lam[3 + k] = 0.0f;
        r.nlo[k] = r.nhi[k] = 0.0f;
    }
    r.n_lam = 1;
    r.prev = cell;
    r.src = i;
    r.L = L0 + Ls;
    *R = r;
}

// level 0: transmission from the TX to IEs i == rank (mod world)
template <bool CNT>
__global__ void __launch_bounds__(128, NRT_SDF_MINB) k_env_tx(TP P, EnvArgs A) {
    const unsigned lane = threadIdx.x & 31;
    Cnt cnt;
    EHist h0;
    memset(&h0, 0, sizeof(h0));
    h0.hash = 14695981039346656037ull;
    const int n_mine = A.n_ie > A.rank ? (A.n_ie - A.rank + A.world - 1) / A.world : 0;
    for (;;) {
        unsigned long long q = 0;
        if (lane == 0) q = atomicAdd(A.work, 1ull);
        q = __shfl_sync(0xffffffffu, q, 0);
        if ((long long)q >= n_mine) break;
        env_try_ie<CNT>(P, A, h0, A.tx, nullptr, 0, ~0u, A.rank + (int)q * A.world, 0.0f, cnt);
        __syncwarp();
    }
    if (CNT && A.terms && lane == 0 && cnt.tests) atomicAdd(A.terms, cnt.tests);
}

// levels >= 1: one cone ray per warp (R64)
template <bool CNT>
__global__ void __launch_bounds__(128, NRT_SDF_MINB) k_env_prop(TP P, EnvArgs A) {
    __shared__ CRay sray[4];
    __shared__ int sring[4][64];
    const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    CRay& R = sray[wid];
    int* ring = sring[wid];
    Cnt cnt;
    for (;;) {
        unsigned long long q = 0;
        if (lane == 0) q = atomicAdd(A.work, 1ull);
        q = __shfl_sync(0xffffffffu, q, 0);
        if (q >= A.n_in) break;
        if (lane == 0) R = A.in[q];
        ring[lane] = -1;
        ring[lane + 32] = -1;
        __syncwarp();
        int head = 0, nring = 0;
        float vpos[3];
        for (int k = 0; k < 3; ++k) vpos[k] = (R.o[k] - A.org[k]) / A.V;
        const float rv = A.V * 0.8660254f, rs = A.S * 0.8660254f;
        for (int it = 0; it < (1 << 16); ++it) {
            int c[3];
            bool out = false;
            for (int k = 0; k < 3; ++k) {
                c[k] = (int)floorf(vpos[k]);
                out |= c[k] < 0 || c[k] >= A.vd[k];
            }
            if (out) break;
            const int cv = c[0] + A.vd[0] * (c[1] + A.vd[1] * c[2]);
            const int am = __ldg(&A.march[cv]);
            if (__ldg(&A.vstart[cv + 1]) > __ldg(&A.vstart[cv]) || am == 1) {
                for (int dz = -1; dz <= 1; ++dz)
                    for (int dy = -1; dy <= 1; ++dy)
                        for (int dx = -1; dx <= 1; ++dx) {
                            const int q3[3] = {c[0] + dx, c[1] + dy, c[2] + dz};
                            if (q3[0] < 0 || q3[0] >= A.vd[0] || q3[1] < 0 || q3[1] >= A.vd[1] || q3[2] < 0 ||
                                q3[2] >= A.vd[2])
                                continue;
                            const int qv = q3[0] + A.vd[0] * (q3[1] + A.vd[1] * q3[2]);
                            const bool hit = (lane < (unsigned)nring && ring[lane] == qv) ||
                                             (lane + 32 < (unsigned)nring && ring[lane + 32] == qv);
                            if (__any_sync(0xffffffffu, hit)) continue;
                            __syncwarp();
                            if (lane == 0) ring[head] = qv;
                            __syncwarp();
                            head = (head + 1) & 63;
                            if (nring < 64) nring++;
                            const int u0 = __ldg(&A.vstart[qv]), u1 = __ldg(&A.vstart[qv + 1]);
                            if (u1 == u0) continue;
                            float cq[3];
                            for (int k = 0; k < 3; ++k) cq[k] = A.org[k] + ((float)q3[k] + 0.5f) * A.V;
                            if (!env_cone_sphere(R.o, R.d, A.tan_c, A.sec_c, cq, rv)) continue;
                            for (int base = u0; base < u1; base += 32) {
                                // lanes: the candidate tests of one IE each (ascending)
                                const int uu = base + (int)lane;
                                bool cand = false;
                                int i = -1;
                                if (uu < u1) {
                                    i = __ldg(&A.vids[uu]);
                                    if (i != R.src) {
                                        const EnvIE I = A.ie[i];
                                        if (I.kind == 2 && R.h.n <= 2) {
                                            cand = true;
                                        } else {
                                            float cs[3];
                                            for (int k = 0; k < 3; ++k) cs[k] = A.org[k] + ((float)I.sub[k] + 0.5f) * A.S;
                                            if (env_cone_sphere(R.o, R.d, A.tan_c, A.sec_c, cs, rs)) {
                                                const float w[3] = {I.p[0] - R.o[0], I.p[1] - R.o[1], I.p[2] - R.o[2]};
                                                cand = R.kind == 0 ? e_dot(w, R.nf) > 0.0f
                                                                   : (e_dot(w, R.nlo) >= 0.0f && e_dot(w, R.nhi) >= 0.0f);
                                            }
                                        }
                                    }
                                }
                                unsigned m = __ballot_sync(0xffffffffu, cand);
                                while (m) {
                                    const int src = __ffs(m) - 1;
                                    m &= m - 1;
                                    const int ic = __shfl_sync(0xffffffffu, i, src);
                                    env_try_ie<CNT>(P, A, R.h, R.o, R.lam, R.n_lam, R.prev, ic, R.L, cnt);
                                    __syncwarp();
                                }
                            }
                        }
            }
            env_march(vpos, R.d, am);
        }
        __syncwarp();
    }
    if (CNT && A.terms && lane == 0 && cnt.tests) atomicAdd(A.terms, cnt.tests);
}

// live-list entries [n_alive, cap) get the largest key, so a sort of all cap entries puts the
// live ones first (in key order) and needs no host-side count
__global__ void k_pad_keys(unsigned* keys, const unsigned long long* n_alive, uint64_t cap) {
    const uint64_t na = *n_alive;
    for (uint64_t j = na + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < cap;
         j += (uint64_t)gridDim.x * blockDim.x)
        keys[j] = 0xFFFFFFFFu;
}

// SHADE: captures, edge events, reflection; compacts the live list for bounce b+1.
// Receivers (few) and edge cull spheres are staged in shared memory and looped over with a
// warp-uniform trip count (one broadcast read per receiver/edge for the whole warp).
#ifndef NRT_SHADE_MINB
#define NRT_SHADE_MINB 5  // k_shade: min resident blocks/SM (register cap)
#endif
__global__ void __launch_bounds__(128, NRT_SHADE_MINB) k_shade(TP P, Wave W, int b) {
    extern __shared__ float4 sh[];
    float4* srx = sh;
    float4* sed = sh + P.shade_rx;
    for (int i = threadIdx.x; i < P.shade_rx; i += blockDim.x)
        srx[i] = make_float4(P.rx[3 * i], P.rx[3 * i + 1], P.rx[3 * i + 2], __int_as_float(i));
    for (int i = threadIdx.x; i < P.shade_edges; i += blockDim.x) {
        const DevEdge& E = P.edges[i];
        sed[i] = make_float4(E.c[0], E.c[1], E.c[2], E.hl);
    }
    __syncthreads();
    const unsigned long long n = W.n_alive[b];
    const unsigned* alive = W.alive[b & 1];
    unsigned* next = W.alive[(b + 1) & 1];
    const unsigned lane = threadIdx.x & 31;
    const unsigned long long warps = (unsigned long long)gridDim.x * (blockDim.x >> 5);
    const unsigned long long gw = (unsigned long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    for (unsigned long long base = gw * 32; base < n; base += warps * 32) {  // warp-uniform
        const unsigned long long j = base + lane;
        const bool on = j < n;
        const unsigned ray = on ? alive[j] : 0u;
        float4 o4 = make_float4(0.0f, 0.0f, 0.0f, 0.0f), d4 = o4;
        float2 hit = make_float2(-1.0f, __int_as_float(-1));
        if (on) {
            o4 = W.ray[ray].o;
            d4 = W.ray[ray].d;
            hit = *(const float2*)&W.ray[ray].l1;
        }
        const float3 o = make_float3(o4.x, o4.y, o4.z), d = make_float3(d4.x, d4.y, d4.z);
        const float th = hit.x;
        const int sid = __float_as_int(hit.y);
        RayCold& c = W.cold[on ? ray : 0u];
        const int flags = on ? c.flags : 0;
        const float L = on ? c.L : 0.0f, Ls = on ? c.Ls : 0.0f;
        const float kR = on ? c.kR : 0.0f, R0 = on ? c.R0 : 0.0f;
        const uint64_t rid = on ? c.rid : 0ull;
        if (P.rxg_cell) {
            if (on) rx_captures(P, c.h, o, d, th, L, Ls, kR, R0, (flags & 2) != 0, rid);
        } else if (__any_sync(0xffffffffu, on)) {
            rx_captures_staged(P, srx, on, c.h, o, d, th, L, Ls, kR, R0, (flags & 2) != 0, rid);
        }
        const bool edges = on && (flags & 1) && c.h.n_diff < P.max_diff && c.h.n < NRT_MAX_INT;
        if (P.shade_edges > 0 || P.n_edges == 0) {
            if (__any_sync(0xffffffffu, edges)) edge_captures_staged(P, sed, edges, c.h, o, d, th, L, rid);
        } else if (edges) {
            edge_captures(P, c.h, o, d, th, L, rid);
        }
        if (P.hit_out && on) P.hit_out[(size_t)ray * (P.max_refl + 1) + c.seg] = sid;  // debug dump
        if (on && sid >= 0 && c.seg < c.budget) {
            // A4: reflect at the hit surfel: d' = d - (2 d.n) n, normalised
            const float3 hp = make_float3(o.x + th * d.x, o.y + th * d.y, o.z + th * d.z);
            const float4 nv = P.sdf ? W.hitn[ray] : __ldg(&P.sn[sid]);  // SDF: MLS normal (R44)
            const float3 nn = make_float3(nv.x, nv.y, nv.z);
            const int hn = c.h.n;
            HEnt en;
            en.label = __ldg(&P.label[sid]);
            en.prim = (uint32_t)sid;
            en.v[0] = hp.x;
            en.v[1] = hp.y;
            en.v[2] = hp.z;
            en.pad_[0] = en.pad_[1] = en.pad_[2] = 0;
            c.h.e[hn] = en;  // one full 32 B sector
            c.h.n = hn + 1;
            const float k2 = 2.0f * dot3(d, nn);
            const float3 x = make_float3(d.x - k2 * nn.x, d.y - k2 * nn.y, d.z - k2 * nn.z);
            const float l = sqrtf(dot3(x, x));
            RayHot R;
            R.d = make_float4(x.x / l, x.y / l, x.z / l, 0.0f);
            R.o = make_float4(hp.x, hp.y, hp.z, P.sdf ? nv.w : __int_as_float(sid));  // prev: surfel / cell
            R.l0 = make_float4(nn.x, nn.y, nn.z, 0.0f);
            R.l1 = make_float4(nn.x, nn.y, nn.z, 0.0f);
            W.ray[ray] = R;
            c.L = L + th;
            c.Ls = Ls + th;
            c.seg = c.seg + 1;
            const unsigned long long slot = agg_inc(&W.n_alive[b + 1]);
            next[slot] = ray;
            if (W.skey) W.skey[slot] = order_key(P, hp, make_float3(x.x / l, x.y / l, x.z / l));
        }
    }
}

// processing order for coherence (primary rays): key = (latitude band of `band` consecutive
// lattice points, azimuth of the ray); bands of ~sqrt(32 pi n) points make 32 consecutive
// slots a near-square patch of the sphere.  k_gen_primary then stores the rays in key order, so
// the wavefront's live list and its per-ray state stay in slot order (coalesced) and a warp's
// lanes trace neighbouring rays.  Ray ids, records and results do not change.
__global__ void k_order_keys(TP P, uint64_t n_batch, uint64_t j0, uint64_t band, unsigned* keys,
                             unsigned* vals) {
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_batch;
         j += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = (uint64_t)P.rank + (j0 + j) * (uint64_t)P.world;
        const float3 v = fib_dir(i, P.n_rays);
        const float a = atan2f(v.y, v.x);  // [-pi, pi]
        const unsigned q = (unsigned)fminf(65535.0f, fmaxf(0.0f, (a + 3.14159265f) * (65536.0f / 6.2831853f)));
        keys[j] = ((unsigned)(j / band) << 16) | q;
        vals[j] = (unsigned)j;
    }
}

// primary ray generation (A2): lattice index i = rank + j * world
// batch slots j in [0, n_batch) hold shard rays j0 + j
// perm (optional): slot j holds batch ray perm[j] (coherent order, k_order_keys)
__global__ void k_gen_primary(TP P, Wave W, uint64_t n_shard, uint64_t j0, const unsigned* perm) {
    const bool edges_on = P.n_edges > 0 && P.max_diff > 0;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_shard;
         j += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t jr = perm ? (uint64_t)perm[j] : j;
        const uint64_t i = (uint64_t)P.rank + (j0 + jr) * (uint64_t)P.world;
        const float3 d = fib_dir(i, P.n_rays);
        RayHot R;
        R.o = make_float4(P.tx, P.ty, P.tz, __int_as_float(-1));
        R.d = make_float4(d.x, d.y, d.z, 0.0f);
        R.l0 = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        R.l1 = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        W.ray[j] = R;
        RayCold& c = W.cold[j];
        c.L = 0.0f;
        c.Ls = 0.0f;
        c.kR = P.cRw;
        c.R0 = 0.0f;
        c.seg = 0;
        c.budget = P.max_refl;
        c.flags = edges_on ? 1 : 0;
        c.rid = i;
        c.h.n = 0;
        c.h.n_diff = 0;
        c.h.kinds = 0;
        c.h.s_edge = 0.0f;
        W.alive[0][j] = (unsigned)j;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) W.n_alive[0] = n_shard;
}

// primary rays with explicit lattice ids (nrt_debug_trace_rays): slot j traces ray ids[j]
// through the same TRACE/SHADE kernels; SHADE writes each segment's hit into P.hit_out
__global__ void k_gen_ids(TP P, Wave W, const uint64_t* ids, uint64_t n) {
    const int nseg = P.max_refl + 1;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
         j += (uint64_t)gridDim.x * blockDim.x) {
        const float3 d = fib_dir(ids[j], P.n_rays);
        RayHot R;
        R.o = make_float4(P.tx, P.ty, P.tz, __int_as_float(-1));
        R.d = make_float4(d.x, d.y, d.z, 0.0f);
        R.l0 = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        R.l1 = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        W.ray[j] = R;
        RayCold& c = W.cold[j];
        c.L = 0.0f;
        c.Ls = 0.0f;
        c.kR = P.cRw;
        c.R0 = 0.0f;
        c.seg = 0;
        c.budget = P.max_refl;
        c.flags = 0;
        c.rid = ids[j];
        c.h.n = 0;
        c.h.n_diff = 0;
        c.h.kinds = 0;
        c.h.s_edge = 0.0f;
        for (int k = 0; k < nseg; ++k) P.hit_out[j * nseg + k] = -2;  // not traced
        W.alive[0][j] = (unsigned)j;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) W.n_alive[0] = n;
}

// fan ray generation (A7, R15-R16): fan index f -> (event r, m); Eq. 14 lift
__global__ void k_gen_fans(TP P, Wave W, const nrt_event_rec* ev, int64_t n_ev,
                           const unsigned int* off, unsigned int total) {
    for (unsigned f = blockIdx.x * blockDim.x + threadIdx.x; f < total;
         f += gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = n_ev - 1;
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (off[mid] <= f) lo = mid;
            else hi = mid - 1;
        }
        const int64_t r = lo;
        const int m = (int)(f - off[r]);
        const nrt_event_rec& e = ev[r];
        const DevEdge& E = P.edges[e.edge];
        const FanGeo g = fan_geo(P, e);
        int n_refl = 0;
        for (int k = 0; k < e.n_hist; ++k)
            if (!((e.kinds >> k) & 1u)) n_refl++;
        int budget = P.max_refl - n_refl;
        if (budget < 0) continue;
        const double wedge = (double)E.n_exp * kPi;
        RayCold& c = W.cold[f];
        c.kR = (float)((double)P.c_R * (wedge / (double)g.M) * g.st);
        c.R0 = 0.5f * P.edge_bin;
        const float3 o = make_float3(E.a[0] + e.s * E.e[0], E.a[1] + e.s * E.e[1],
                                     E.a[2] + e.s * E.e[2]);
        Hist& h = c.h;
        h.n = e.n_hist;
        h.n_diff = e.n_diff;
        h.kinds = e.kinds;
        for (int k = 0; k < NRT_MAX_INT; ++k) {
            h.e[k].label = e.label[k];
            h.e[k].prim = e.prim[k];
            h.e[k].v[0] = e.v[k][0];
            h.e[k].v[1] = e.v[k][1];
            h.e[k].v[2] = e.v[k][2];
        }
        h.e[h.n].label = E.label;
        h.e[h.n].prim = e.edge;
        h.e[h.n].v[0] = o.x;
        h.e[h.n].v[1] = o.y;
        h.e[h.n].v[2] = o.z;
        h.kinds |= 1u << h.n;
        h.n++;
        h.n_diff++;
        h.s_edge = e.s;
        if (h.n + budget > NRT_MAX_INT) budget = NRT_MAX_INT - h.n;
        const double phi = (((double)m + 0.5) * wedge) / (double)g.M;
        double sp, cp;
        nrt_sincos(phi, &sp, &cp);
        float dir[3];
        for (int k = 0; k < 3; ++k) {
            const double x2 = cp * (double)E.t0[k] + sp * (double)E.n0[k];
            dir[k] = (float)(x2 * g.st + (double)E.e[k] * g.ct);
        }
        RayHot R;
        R.o = make_float4(o.x, o.y, o.z, __int_as_float(-1));
        R.d = make_float4(dir[0], dir[1], dir[2], 0.0f);
        R.l0 = make_float4(E.n0[0], E.n0[1], E.n0[2], 0.0f);
        R.l1 = make_float4(E.n1[0], E.n1[1], E.n1[2], 0.0f);
        W.ray[f] = R;
        c.L = e.L;
        c.Ls = 0.0f;
        c.seg = 0;
        c.budget = budget;
        c.flags = 2;
        c.rid = (1ull << 63) | ((uint64_t)r << 8) | (uint64_t)m;
        W.alive[0][agg_inc(&W.n_alive[0])] = f;
    }
}

TP make_tp(nrt_scene s, const LaunchArgs& a) {
    TP P{};
    P.cell = s->cell;
    P.rec = s->rec;
    P.sn = s->sn;
    P.label = s->label;
    P.ox = s->org[0];
    P.oy = s->org[1];
    P.oz = s->org[2];
    P.v = s->v;
    P.inv_v = s->inv_v;
    {
        const int md = std::max(s->dims[0], std::max(s->dims[1], s->dims[2]));
        P.ok_inv = 1.0f / (s->v * (float)((md + 63) / 64));
    }
    P.pad = s->pad;
    P.slack = fmaxf(s->slack, 4e-6f * fmaxf(fabsf(a.tx[0]), fmaxf(fabsf(a.tx[1]), fabsf(a.tx[2]))));
    P.nx = s->dims[0];
    P.ny = s->dims[1];
    P.nz = s->dims[2];
    P.tx = a.tx[0];
    P.ty = a.tx[1];
    P.tz = a.tx[2];
    P.rx = a.d_rx;
    P.n_rx = a.n_rx;
    P.n_rays = (uint64_t)a.n_rays;
    P.rank = a.desc.rank;
    P.world = a.desc.world;
    P.max_refl = a.max_refl;
    P.max_diff = a.max_diff;
    P.tau = a.desc.tau;
    P.cos_ex = cos_ex_of(a.desc.theta_ex_deg);
    P.cRw = cRw_of(a.desc.c_R, a.n_rays);
    P.b_e = s->r_max + a.desc.tau;
    P.edge_bin = a.desc.edge_bin;
    P.c_R = a.desc.c_R;
    P.dphi_deg = a.desc.dphi_deg;
    P.edges = s->edges;
    P.n_edges = s->n_edges;
    P.rxg_cell = a.rxg.cell;
    P.rxg_rx = a.rxg.rx;
    for (int k = 0; k < 3; ++k) {
        P.rxg_o[k] = a.rxg.o[k];
        P.rxg_n[k] = a.rxg.n[k];
        P.rxg_lo[k] = a.rxg.lo[k];
        P.rxg_hi[k] = a.rxg.hi[k];
    }
    P.rxg_v = a.rxg.v;
    P.rxg_inv = a.rxg.v > 0 ? 1.0f / a.rxg.v : 0.0f;
    P.rxg_tmax = a.rxg.tmax;
    P.shade_rx = a.rxg.cell ? 0 : a.n_rx;
    P.shade_edges = s->n_edges <= kShadeEdges ? s->n_edges : 0;
    if (a.desc.intersect == 1) {  // NEXT-1 (R40-R45): FP32 constants as the definition forms them
        P.sdf = 1;
        P.sdf_pts = s->sdf_pts;
        P.sdf_box = s->sdf_box;
        P.sdf_acell = s->sdf_acell;
        P.sdf_gcell = s->sdf_gcell;
        P.sdf_aref = s->sdf_aref;
        P.sdf_crange = s->sdf_crange;
        for (int k = 0; k < 3; ++k) {
            P.sg_o[k] = s->sdf_gorg[k];
            P.sg_n[k] = s->sdf_gdims[k];
            P.sd_n[k] = s->sdf_dims[k];
            P.sd_o[k] = s->sdf_org[k];
        }
        P.sn_p = s->sp;
        P.sdf_a = s->sdf_a;
        P.sdf_inv_a = 1.0f / s->sdf_a;
        P.sdf_half = 0.5f * (s->sdf_a * 1.7320508f);
        P.sdf_stop = 2.0f * P.sdf_half + s->sdf_pad;
        P.sdf_rs = a.desc.sdf_r_s;
        P.sdf_tsdf = a.desc.sdf_t_sdf;
        const float sigma = a.desc.sdf_xi * a.desc.sdf_r_s;
        P.sdf_sigma = sigma;
        P.sdf_inv = 1.0f / (2.0f * sigma * sigma);
    }
    return P;
}

int sm_count(int dev) {
    static int cached[64] = {0};
    if (dev >= 0 && dev < 64 && cached[dev]) return cached[dev];
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (dev >= 0 && dev < 64) cached[dev] = n;
    return n > 0 ? n : 148;
}

template <class K>
unsigned persistent_blocks(K kernel, int dev) {
    static int per_sm_cache[2] = {0, 0};
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 128, 0);
    (void)per_sm_cache;
    if (per_sm < 1) per_sm = 1;
    return (unsigned)(sm_count(dev) * per_sm);
}

}  // namespace

nrt_status rxgrid_build(nrt_scene s, const float* rx, int32_t n_rx, float rreg, RxGrid* g,
                        cudaStream_t st) {
    *g = RxGrid{};
    const char* e = getenv("NRT_RX_GRID_MIN");
    const int min_rx = e ? atoi(e) : NRT_SHADE_RX + 1;
    const char* ev = getenv("NRT_RX_GRID_V");
    const float v = ev ? (float)atof(ev) : 0.5f;
    // few receivers, or capture balls larger than the cells: the all-receivers loop is cheaper
    if (n_rx < min_rx || n_rx <= 0 || !(rreg <= 2.0f * v)) return NRT_OK;
    (void)s;
    const float reg = rreg * 1.001f + 1e-3f;  // registration radius with a float pad
    g->v = v;
    for (int a = 0; a < 3; ++a) {
        g->lo[a] = rx[a];
        g->hi[a] = rx[a];
    }
    for (int j = 0; j < n_rx; ++j)
        for (int a = 0; a < 3; ++a) {
            g->lo[a] = fminf(g->lo[a], rx[3 * j + a]);
            g->hi[a] = fmaxf(g->hi[a], rx[3 * j + a]);
        }
    for (int a = 0; a < 3; ++a) {
        g->o[a] = g->lo[a] - reg - v;
        g->n[a] = (int)ceilf((g->hi[a] + reg + v - g->o[a]) / v) + 1;
    }
    g->tmax = 1e30f;
    const int64_t nc = (int64_t)g->n[0] * g->n[1] * g->n[2];
    std::vector<std::vector<int>> bins(nc);
    for (int j = 0; j < n_rx; ++j) {
        int lo[3], hi[3];
        for (int a = 0; a < 3; ++a) {
            lo[a] = std::max(0, (int)floorf((rx[3 * j + a] - reg - g->o[a]) / v));
            hi[a] = std::min(g->n[a] - 1, (int)floorf((rx[3 * j + a] + reg - g->o[a]) / v));
        }
        for (int z = lo[2]; z <= hi[2]; ++z)
            for (int y = lo[1]; y <= hi[1]; ++y)
                for (int x = lo[0]; x <= hi[0]; ++x)
                    bins[x + (int64_t)g->n[0] * (y + (int64_t)g->n[1] * z)].push_back(j);
    }
    std::vector<uint2> cells(nc);
    std::vector<float4> srt;
    srt.reserve(n_rx);
    for (int64_t c = 0; c < nc; ++c) {
        cells[c].x = (unsigned)srt.size();
        for (int j : bins[c]) {
            float4 r;
            r.x = rx[3 * j];
            r.y = rx[3 * j + 1];
            r.z = rx[3 * j + 2];
            int jj = j;
            memcpy(&r.w, &jj, 4);
            srt.push_back(r);
        }
        cells[c].y = (unsigned)srt.size();
    }
    NRT_CUDA(cudaMallocAsync(&g->cell, nc * sizeof(uint2), st));
    NRT_CUDA(cudaMallocAsync(&g->rx, (srt.size() ? srt.size() : 1) * sizeof(float4), st));
    NRT_CUDA(cudaMemcpyAsync(g->cell, cells.data(), nc * sizeof(uint2), cudaMemcpyHostToDevice, st));
    if (srt.size())
        NRT_CUDA(cudaMemcpyAsync(g->rx, srt.data(), srt.size() * sizeof(float4), cudaMemcpyHostToDevice, st));
    NRT_CUDA(cudaStreamSynchronize(st));  // host vectors go out of scope
    return NRT_OK;
}

// largest capture radius of a launch (R12 / R16): L and the distance since an edge are bounded by
// (segments + 1) grid diagonals; after a diffraction kR = c_R (n pi / M)|sin theta| <= c_R dphi
void capture_radius_bounds(nrt_scene s, const LaunchArgs& a, float* r_primary, float* r_fan) {
    double d2 = 0;
    for (int k = 0; k < 3; ++k) d2 += (double)s->dims[k] * s->v * s->dims[k] * s->v;
    const double lmax = (a.max_refl + 2.0) * sqrt(d2) + 1.0;
    *r_primary = (float)(cRw_of(a.desc.c_R, a.n_rays) * lmax);
    *r_fan = (float)(a.desc.c_R * a.desc.dphi_deg * (kPi / 180.0) * lmax + 0.5 * a.desc.edge_bin);
}

void rxgrid_free(RxGrid* g, cudaStream_t st) {
    if (g->cell) cudaFreeAsync(g->cell, st);
    if (g->rx) cudaFreeAsync(g->rx, st);
    *g = RxGrid{};
}

// NRT_ORDER=0 disables the coherent primary-ray order (diagnostics)
static bool order_rays() {
    static const int on = [] {
        const char* e = getenv("NRT_ORDER");
        return e ? atoi(e) : 1;
    }();
    return on != 0;
}

static double host_ms_since(std::chrono::steady_clock::time_point t) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count();
}

struct Counters {
    unsigned long long raw_n, ev_n, bounces, tests, cells, nonempty;
    unsigned long long n_alive[kMaxIter + 1];
    unsigned long long ctr[kMaxIter];
};

static std::atomic<unsigned long long> g_hint_raw{0}, g_hint_ev{0}, g_hint_fan{0};
// rays in flight per wavefront batch (bounded wavefront state: ~440 B per ray in flight, so
// 2^26 rays hold ~30 GB of a 180 GB B200; measured on C5: 2^24 / 2^25 / 2^26 / 1e8 rays per
// batch -> 1280 / 1269 / 1235 / 1237 ms per step); NRT_BATCH overrides (A/B)
static uint64_t batch_rays() {
    if (const char* e = getenv("NRT_BATCH")) return strtoull(e, nullptr, 10);
    return 1ull << 26;
}
// reorder live lists of batches at least this long (NRT_SORT_MIN overrides: tests force the
// reorder path on small scenes)
static unsigned long long sort_min() {
    if (const char* e = getenv("NRT_SORT_MIN")) return strtoull(e, nullptr, 10);
    return 1ull << 15;
}

// wavefront buffers for up to `cap` rays (stream-ordered; freed by free_wave)
// Reorder each bounce's live list by (coarse cell, direction) only when the scene's records
// are well beyond L2 (measured: C5, 0.9 GB of records, trace -7 %; C2, 243 MB, no gain and
// +0.45 ms of sorts).  NRT_REORDER=0/1 forces it.
static bool reorder_on(nrt_scene s) {
    if (const char* e = getenv("NRT_REORDER")) return atoi(e) != 0;
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, s->device);
    return (double)s->nref * 32.0 > 4.0 * (double)l2;
}

static nrt_status alloc_wave(Wave& W, uint64_t cap, int dev, bool sdf, cudaStream_t st) {
    if (cap < 1) cap = 1;
    auto al = [](size_t b) { return (b + 255) / 256 * 256; };
    const size_t b_r = al(cap * sizeof(RayHot)), b_o = al(cap * sizeof(float4)),
                 b_c = al(cap * sizeof(RayCold)), b_a = al(cap * sizeof(unsigned));
    size_t b_t = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b_t, (unsigned*)nullptr, (unsigned*)nullptr,
                                    (unsigned*)nullptr, (unsigned*)nullptr, (int)cap, 0, 32, st);
    b_t = al(b_t);
    const size_t total = b_r + b_c + 2 * b_a + 3 * b_a + b_t + (sdf ? b_o : 0);
    char* p = (char*)ws_get(dev, total, st);
    if (!p) return set_error(NRT_E_NOMEM, "wavefront workspace of %zu bytes", total);
    {
        char* q = p + b_r + b_c + 2 * b_a;
        W.okey[0] = (unsigned*)q;
        W.okey[1] = (unsigned*)(q + b_a);
        W.oval = (unsigned*)(q + 2 * b_a);
        W.otmp = q + 3 * b_a;
        W.otmp_bytes = b_t;
        W.hitn = sdf ? (float4*)(q + 3 * b_a + b_t) : nullptr;
        W.skey = nullptr;  // per-bounce coherence reorder: see reorder_on()
    }
    W.slab = p;
    W.ray = (RayHot*)p;
    W.cold = (RayCold*)(p + b_r);
    W.alive[0] = (unsigned*)(p + b_r + b_c);
    W.alive[1] = (unsigned*)(p + b_r + b_c + b_a);
    return NRT_OK;
}
// returns the slab to the workspace cache once no queued kernel still reads it
static void free_wave(Wave& W, cudaStream_t st) {
    if (!W.slab) return;
    cudaStreamSynchronize(st);
    ws_put(W.slab);
    W.slab = nullptr;
}
struct WaveGuard {  // every exit path of a launch phase
    Wave* W;
    cudaStream_t st;
    ~WaveGuard() { free_wave(*W, st); }
};

// bounce loop: TRACE + SHADE per bounce; ms_kernel accumulates the TRACE kernels' time
static nrt_status run_bounces(const TP& P, Wave& W, uint64_t cap, int iters, int dev, bool counters,
                              float* ms_trace, cudaStream_t st) {
#if NRT_TRACE_COOP
#define NRT_K_TRACE k_trace_coop
#else
#define NRT_K_TRACE k_trace
#endif
    const unsigned tb = P.sdf ? (counters ? persistent_blocks(k_trace_sdf<true>, dev)
                                          : persistent_blocks(k_trace_sdf<false>, dev))
                              : (counters ? persistent_blocks(NRT_K_TRACE<true>, dev)
                                          : persistent_blocks(NRT_K_TRACE<false>, dev));
    const size_t shade_smem = (size_t)(P.shade_rx + P.shade_edges) * sizeof(float4);
    if (shade_smem > 48 * 1024)
        NRT_CUDA(cudaFuncSetAttribute(k_shade, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shade_smem));
    // SHADE: exactly one wave of resident blocks (its loop strides over the live list; a second,
    // partial wave only lengthened the tail); NRT_SHADE_BLOCKS overrides (blocks per SM)
    unsigned sb;
    {
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_shade, 128, shade_smem);
        if (const char* e = getenv("NRT_SHADE_BLOCKS")) per_sm = atoi(e);
        if (per_sm < 1) per_sm = 1;
        sb = (unsigned)sm_count(dev) * (unsigned)per_sm;
    }
    cudaEvent_t ev[3 * kMaxIter + 3];
    for (int i = 0; i < 3 * iters; ++i) cudaEventCreate(&ev[i]);
    unsigned long long last[3] = {0, 0, 0};
    if (counters && P.counters && getenv("NRT_BOUNCE_STATS")) {
        cudaMemcpyAsync(last, P.counters, sizeof(last), cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
    }
    for (int b = 0; b < iters; ++b) {
        cudaEventRecord(ev[3 * b], st);
        if (P.sdf) {
            if (counters) k_trace_sdf<true><<<tb, 128, 0, st>>>(P, W, b);
            else k_trace_sdf<false><<<tb, 128, 0, st>>>(P, W, b);
        } else if (counters) {
            NRT_K_TRACE<true><<<tb, 128, 0, st>>>(P, W, b);
        } else {
            NRT_K_TRACE<false><<<tb, 128, 0, st>>>(P, W, b);
        }
        ::nrt::count_launch();
        if (counters && P.counters && getenv("NRT_BOUNCE_STATS")) {  // diagnostics: per-bounce work
            unsigned long long c[3], na = 0;
            cudaMemcpyAsync(c, P.counters, sizeof(c), cudaMemcpyDeviceToHost, st);
            cudaMemcpyAsync(&na, W.n_alive + b, sizeof(na), cudaMemcpyDeviceToHost, st);
            cudaStreamSynchronize(st);
            fprintf(stderr, "[nrt] bounce %d: %llu segments, %.1f tests, %.1f cells, %.1f non-empty per segment\n", b, na,
                    (double)(c[0] - last[0]) / (na ? na : 1), (double)(c[1] - last[1]) / (na ? na : 1),
                    (double)(c[2] - last[2]) / (na ? na : 1));
            for (int q = 0; q < 3; ++q) last[q] = c[q];
        }
        cudaEventRecord(ev[3 * b + 1], st);
        k_shade<<<sb, 128, shade_smem, st>>>(P, W, b);
        ::nrt::count_launch();
        if (W.skey && b + 1 < iters && cap >= sort_min()) {
            // reorder the next live list by (coarse cell, direction): neighbouring lanes and
            // blocks then walk the same cells and share their records in L1/L2.  The count
            // stays on the device: entries past it are padded with the largest key and the
            // whole capacity is sorted (no host round trip inside the bounce loop)
            k_pad_keys<<<(unsigned)sm_count(dev) * 4, 256, 0, st>>>(W.skey, W.n_alive + b + 1, cap);
            ::nrt::count_launch();
            size_t tb = W.otmp_bytes;
            unsigned* nxt = W.alive[(b + 1) & 1];
            NRT_CUDA(cub::DeviceRadixSort::SortPairs(W.otmp, tb, W.skey, W.okey[1], nxt, W.oval, (int)cap,
                                                     0, 32, st));
            W.alive[(b + 1) & 1] = W.oval;
            W.oval = nxt;
        }
        cudaEventRecord(ev[3 * b + 2], st);
    }
    NRT_CUDA(cudaGetLastError());
    NRT_CUDA(cudaStreamSynchronize(st));
    float tot = 0, shade = 0;
    for (int b = 0; b < iters; ++b) {
        float ms = 0, ms2 = 0;
        cudaEventElapsedTime(&ms, ev[3 * b], ev[3 * b + 1]);
        cudaEventElapsedTime(&ms2, ev[3 * b + 1], ev[3 * b + 2]);
        tot += ms;
        shade += ms2;
    }
    if (getenv("NRT_PHASES")) fprintf(stderr, "[nrt] bounces: trace %.3f ms shade %.3f ms\n", tot, shade);
    for (int i = 0; i < 3 * iters; ++i) cudaEventDestroy(ev[i]);
    *ms_trace = tot;
    return NRT_OK;
}

nrt_status launch_primary(nrt_scene s, const LaunchArgs& a, nrt_coarse_rec** raw_out,
                          int64_t* n_raw, nrt_event_rec** ev_out, int64_t* n_ev,
                          uint64_t* bounces, KernelStats* stats, cudaStream_t st) {
    if (getenv("NRT_PHASES")) cudaStreamSynchronize(st);
    const auto t_start = std::chrono::steady_clock::now();
    TP P = make_tp(s, a);
    const uint64_t n_shard =
        a.n_rays > a.desc.rank ? ((uint64_t)a.n_rays - a.desc.rank + a.desc.world - 1) / a.desc.world
                               : 0;
    // capacities start from the largest counts any launch of this process needed (scene
    // handles are rebuilt often; a too-small buffer would re-run the whole launch)
    if (g_hint_raw.load() > s->hint_raw) s->hint_raw = g_hint_raw.load();
    if (g_hint_ev.load() > s->hint_ev) s->hint_ev = g_hint_ev.load();
    unsigned long long raw_cap = s->hint_raw + s->hint_raw / 4 + 1024;
    unsigned long long ev_cap = s->hint_ev + s->hint_ev / 4 + 1024;
    if (P.n_edges > 0 && P.max_diff > 0 && ev_cap < n_shard / 8) ev_cap = n_shard / 8;
    Counters* dc = nullptr;
    NRT_CUDA(cudaMallocAsync(&dc, sizeof(Counters), st));
    Wave W{};
    WaveGuard wg{&W, st};
    const uint64_t kBatch = batch_rays();
    NRT_TRY(alloc_wave(W, n_shard < kBatch ? n_shard : kBatch, s->device, P.sdf != 0, st));
    if (reorder_on(s)) W.skey = W.okey[0];
    if (getenv("NRT_PHASES")) {
        cudaStreamSynchronize(st);
        cudaMemPool_t pool;
        size_t res = 0, used = 0;
        cudaDeviceGetDefaultMemPool(&pool, s->device);
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &res);
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
        fprintf(stderr, "[nrt] wave alloc %.3f ms (pool reserved %.2f GB used %.2f GB)\n",
                host_ms_since(t_start), res / 1e9, used / 1e9);
    }
    W.n_alive = dc->n_alive;
    W.ctr = dc->ctr;
    nrt_coarse_rec* raw = nullptr;
    nrt_event_rec* ev = nullptr;
    Counters hc{};
    for (int attempt = 0; attempt < 3; ++attempt) {
        NRT_CUDA(cudaMallocAsync(&raw, raw_cap * sizeof(nrt_coarse_rec), st));
        NRT_CUDA(cudaMallocAsync(&ev, ev_cap * sizeof(nrt_event_rec), st));
        NRT_CUDA(cudaMemsetAsync(dc, 0, sizeof(Counters), st));
        P.raw = raw;
        P.raw_cap = raw_cap;
        P.raw_n = &dc->raw_n;
        P.ev = ev;
        P.ev_cap = ev_cap;
        P.ev_n = &dc->ev_n;
        P.bounces = &dc->bounces;
        P.counters = &dc->tests;
        // primary rays in batches of kBatch (bounded wavefront state: 290 B per ray in flight);
        // records, events and counters accumulate across batches
        stats->ms_kernel = 0.0f;
        for (uint64_t j0 = 0; j0 < n_shard; j0 += kBatch) {
            const uint64_t nb = n_shard - j0 < kBatch ? n_shard - j0 : kBatch;
            NRT_CUDA(cudaMemsetAsync(dc->n_alive, 0, sizeof(dc->n_alive) + sizeof(dc->ctr), st));
            unsigned gb = (unsigned)((nb + 255) / 256);
            if (gb > (unsigned)sm_count(s->device) * 16) gb = (unsigned)sm_count(s->device) * 16;
            const unsigned* perm = nullptr;
            if (order_rays()) {
                // coherent order: sorted (band, azimuth) keys -> permutation in alive[1] (free
                // until the first SHADE writes the next live list)
                uint64_t band = (uint64_t)sqrt(32.0 * kPi * (double)a.n_rays / (double)a.desc.world);
                if (band < 32) band = 32;
                int hi_bit = 16;
                while (hi_bit < 32 && ((nb / band) >> (hi_bit - 16))) ++hi_bit;
                k_order_keys<<<gb, 256, 0, st>>>(P, nb, j0, band, W.okey[0], W.oval);
                ::nrt::count_launch();
                size_t tb = W.otmp_bytes;
                NRT_CUDA(cub::DeviceRadixSort::SortPairs(W.otmp, tb, W.okey[0], W.okey[1], W.oval, W.alive[1],
                                                         (int)nb, 0, hi_bit, st));
                ::nrt::count_launch();
                perm = W.alive[1];
            }
            k_gen_primary<<<gb, 256, 0, st>>>(P, W, nb, j0, perm);
            ::nrt::count_launch();
            if (getenv("NRT_PHASES")) {
                cudaStreamSynchronize(st);
                fprintf(stderr, "[nrt] gen done %.3f ms\n", host_ms_since(t_start));
            }
            float ms = 0.0f;
            NRT_TRY(run_bounces(P, W, nb, a.max_refl + 1, s->device, a.desc.counters != 0, &ms, st));
            stats->ms_kernel += ms;
        }
        NRT_CUDA(cudaMemcpyAsync(&hc, dc, sizeof(hc), cudaMemcpyDeviceToHost, st));
        NRT_CUDA(cudaStreamSynchronize(st));
        stats->tests = hc.tests;
        stats->cells = hc.cells;
        stats->nonempty = hc.nonempty;
        if (hc.raw_n > s->hint_raw) s->hint_raw = hc.raw_n;
        if (hc.ev_n > s->hint_ev) s->hint_ev = hc.ev_n;
        if (hc.raw_n > g_hint_raw.load()) g_hint_raw.store(hc.raw_n);
        if (hc.ev_n > g_hint_ev.load()) g_hint_ev.store(hc.ev_n);
        if (getenv("NRT_PHASES"))
            fprintf(stderr, "[nrt] primary attempt %d: raw %llu/%llu events %llu/%llu\n", attempt,
                    hc.raw_n, raw_cap, hc.ev_n, ev_cap);
        if (hc.raw_n <= raw_cap && hc.ev_n <= ev_cap) break;
        cudaFreeAsync(raw, st);
        cudaFreeAsync(ev, st);
        raw_cap = hc.raw_n > raw_cap ? hc.raw_n : raw_cap;
        ev_cap = hc.ev_n > ev_cap ? hc.ev_n : ev_cap;
    }
    free_wave(W, st);
    cudaFreeAsync(dc, st);
    if (getenv("NRT_PHASES")) {
        cudaStreamSynchronize(st);
        fprintf(stderr, "[nrt] primary done %.3f ms\n", host_ms_since(t_start));
    }
    *raw_out = raw;
    *n_raw = (int64_t)hc.raw_n;
    *ev_out = ev;
    *n_ev = (int64_t)hc.ev_n;
    *bounces = hc.bounces;
    return NRT_OK;
}

nrt_status launch_fans(nrt_scene s, const LaunchArgs& a, const nrt_event_rec* ev, int64_t n_ev,
                       nrt_coarse_rec** raw_out, int64_t* n_raw, int64_t* n_fan_rays,
                       uint64_t* bounces, KernelStats* stats, cudaStream_t st) {
    *raw_out = nullptr;
    *n_raw = 0;
    *n_fan_rays = 0;
    *bounces = 0;
    if (n_ev <= 0) return NRT_OK;
    TP P = make_tp(s, a);
    unsigned int *cnt = nullptr, *off = nullptr;
    NRT_CUDA(cudaMallocAsync(&cnt, (n_ev + 1) * 4, st));
    NRT_CUDA(cudaMallocAsync(&off, (n_ev + 1) * 4, st));
    k_fan_count<<<(unsigned)((n_ev + 127) / 128), 128, 0, st>>>(P, ev, n_ev, cnt);
    ::nrt::count_launch();
    NRT_CUDA(cudaGetLastError());
    NRT_CUDA(cudaMemsetAsync(cnt + n_ev, 0, 4, st));
    size_t tb = 0;
    void* tmp = nullptr;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, off, n_ev + 1, st);
    NRT_CUDA(cudaMallocAsync(&tmp, tb, st));
    cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, off, n_ev + 1, st);
    cudaFreeAsync(tmp, st);
    unsigned int total = 0;
    NRT_CUDA(cudaMemcpyAsync(&total, off + n_ev, 4, cudaMemcpyDeviceToHost, st));
    NRT_CUDA(cudaStreamSynchronize(st));
    *n_fan_rays = total;
    Counters* dc = nullptr;
    NRT_CUDA(cudaMallocAsync(&dc, sizeof(Counters), st));
    if (g_hint_fan.load() > s->hint_fan) s->hint_fan = g_hint_fan.load();
    unsigned long long raw_cap = s->hint_fan + s->hint_fan / 4 + 1024;
    nrt_coarse_rec* raw = nullptr;
    Counters hc{};
    Wave W{};
    WaveGuard wg{&W, st};
    if (total > 0) NRT_TRY(alloc_wave(W, total, s->device, P.sdf != 0, st));
    if (total > 0 && reorder_on(s)) W.skey = W.okey[0];
    W.n_alive = dc->n_alive;
    W.ctr = dc->ctr;
    for (int attempt = 0; attempt < 3 && total > 0; ++attempt) {
        NRT_CUDA(cudaMallocAsync(&raw, raw_cap * sizeof(nrt_coarse_rec), st));
        NRT_CUDA(cudaMemsetAsync(dc, 0, sizeof(Counters), st));
        P.raw = raw;
        P.raw_cap = raw_cap;
        P.raw_n = &dc->raw_n;
        P.ev = nullptr;
        P.ev_cap = 0;
        P.ev_n = &dc->ev_n;
        P.bounces = &dc->bounces;
        P.counters = &dc->tests;
        unsigned gb = (total + 255) / 256;
        if (gb > (unsigned)sm_count(s->device) * 16) gb = (unsigned)sm_count(s->device) * 16;
        k_gen_fans<<<gb, 256, 0, st>>>(P, W, ev, n_ev, off, total);
        ::nrt::count_launch();
        // fans need at most max_refl + 1 segments (budget <= max_refl)
        NRT_TRY(run_bounces(P, W, total, a.max_refl + 1, s->device, a.desc.counters != 0,
                            &stats->ms_kernel, st));
        NRT_CUDA(cudaMemcpyAsync(&hc, dc, sizeof(hc), cudaMemcpyDeviceToHost, st));
        NRT_CUDA(cudaStreamSynchronize(st));
        stats->tests = hc.tests;
        stats->cells = hc.cells;
        stats->nonempty = hc.nonempty;
        if (hc.raw_n > s->hint_fan) s->hint_fan = hc.raw_n;
        if (hc.raw_n > g_hint_fan.load()) g_hint_fan.store(hc.raw_n);
        if (hc.raw_n <= raw_cap) break;
        cudaFreeAsync(raw, st);
        raw_cap = hc.raw_n;
    }
    free_wave(W, st);
    cudaFreeAsync(dc, st);
    cudaFreeAsync(cnt, st);
    cudaFreeAsync(off, st);
    *raw_out = raw;
    *n_raw = (int64_t)hc.raw_n;
    *bounces = hc.bounces;
    return NRT_OK;
}

// ---- NEXT-2 host side --------------------------------------------------------------------
// PCIE formation (R60) on the device: points sorted by (subvoxel, id); one thread per PCIE
__global__ void k_env_keys(const float4* sp, int64_t n, float ox, float oy, float oz, float a, int sd0, int sd1,
                           int sd2, int sv0, int sv1, unsigned* keys, unsigned* vals) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float4 p = sp[i];
    const int c0 = min(sd0 - 1, max(0, (int)floorf((p.x - ox) / a)));
    const int c1 = min(sd1 - 1, max(0, (int)floorf((p.y - oy) / a)));
    const int c2 = min(sd2 - 1, max(0, (int)floorf((p.z - oz) / a)));
    keys[i] = (unsigned)(c0 / 4 + sv0 * (c1 / 4 + sv1 * (c2 / 4)));
    vals[i] = (unsigned)i;
}
__global__ void k_env_pcie(const unsigned* subs, const unsigned* off, int64_t npc, const unsigned* ids, const float4* sp,
                           const int32_t* label, float ox, float oy, float oz, float S, int sv0, int sv1, EnvIE* out) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= npc) return;
    const unsigned s = subs[j];
    const int sb[3] = {(int)(s % (unsigned)sv0), (int)((s / (unsigned)sv0) % (unsigned)sv1),
                       (int)(s / ((unsigned)sv0 * (unsigned)sv1))};
    const float c[3] = {ox + ((float)sb[0] + 0.5f) * S, oy + ((float)sb[1] + 0.5f) * S, oz + ((float)sb[2] + 0.5f) * S};
    double sum[3] = {0.0, 0.0, 0.0};
    float bq = INFINITY;
    int lab = 0;
    const unsigned k0 = off[j], k1 = off[j + 1];
    for (unsigned k = k0; k < k1; ++k) {
        const unsigned id = ids[k];
        const float4 p = sp[id];
        sum[0] += (double)p.x;
        sum[1] += (double)p.y;
        sum[2] += (double)p.z;
        const float d[3] = {p.x - c[0], p.y - c[1], p.z - c[2]};
        const float q = (d[0] * d[0] + d[1] * d[1]) + d[2] * d[2];
        if (q < bq) {
            bq = q;
            lab = label[id];
        }
    }
    EnvIE I;
    const double cnt = (double)(k1 - k0);
    I.p[0] = (float)(sum[0] / cnt);
    I.p[1] = (float)(sum[1] / cnt);
    I.p[2] = (float)(sum[2] / cnt);
    I.kind = 0;
    I.label = lab;
    I.ref = (int)s;
    I.sub[0] = sb[0];
    I.sub[1] = sb[1];
    I.sub[2] = sb[2];
    I.s_edge = 0.0f;
    out[j] = I;
}

nrt_status launch_env(nrt_scene s, const LaunchArgs& a, nrt_coarse_rec** raw_out, int64_t* n_raw, uint64_t* rays,
                      float* ms_kernel, uint64_t* terms_out, cudaStream_t st) {
    *raw_out = nullptr;
    *n_raw = 0;
    *rays = 0;
    const TP P = make_tp(s, a);
    const int64_t n = s->n;
    const float A0 = s->sdf_a, V = 8.0f * A0, S = 4.0f * A0;
    int sd[3], sv[3], vd[3];
    for (int k = 0; k < 3; ++k) {
        sd[k] = s->sdf_dims[k];
        sv[k] = (sd[k] + 3) / 4;
        vd[k] = (sd[k] + 7) / 8;
    }
    const int64_t nsub = (int64_t)sv[0] * sv[1] * sv[2];
    // ---- PCIEs (device)
    std::vector<EnvIE> ies;
    {
        unsigned *k0 = nullptr, *k1 = nullptr, *v0 = nullptr, *v1 = nullptr, *uniq = nullptr, *cnt = nullptr,
                 *off = nullptr;
        int64_t* nr = nullptr;
        NRT_CUDA(cudaMallocAsync(&k0, n * 4, st));
        NRT_CUDA(cudaMallocAsync(&k1, n * 4, st));
        NRT_CUDA(cudaMallocAsync(&v0, n * 4, st));
        NRT_CUDA(cudaMallocAsync(&v1, n * 4, st));
        NRT_CUDA(cudaMallocAsync(&uniq, n * 4, st));
        NRT_CUDA(cudaMallocAsync(&cnt, (n + 1) * 4, st));
        NRT_CUDA(cudaMallocAsync(&off, (n + 1) * 4, st));
        NRT_CUDA(cudaMallocAsync(&nr, 8, st));
        const unsigned nb = (unsigned)((n + 255) / 256);
        k_env_keys<<<nb, 256, 0, st>>>(s->sp, n, s->sdf_org[0], s->sdf_org[1], s->sdf_org[2], A0, sd[0], sd[1], sd[2],
                                       sv[0], sv[1], k0, v0);
        ::nrt::count_launch();
        int bits = 1;
        while (((int64_t)1 << bits) < nsub) ++bits;
        cub::DoubleBuffer<unsigned> kb(k0, k1), vb(v0, v1);
        size_t tb = 0;
        void* tmp = nullptr;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, kb, vb, (int)n, 0, bits, st);
        NRT_CUDA(cudaMallocAsync(&tmp, tb, st));
        cub::DeviceRadixSort::SortPairs(tmp, tb, kb, vb, (int)n, 0, bits, st);
        cudaFreeAsync(tmp, st);
        tb = 0;
        cub::DeviceRunLengthEncode::Encode(nullptr, tb, kb.Current(), uniq, cnt, nr, (int64_t)n, st);
        NRT_CUDA(cudaMallocAsync(&tmp, tb, st));
        cub::DeviceRunLengthEncode::Encode(tmp, tb, kb.Current(), uniq, cnt, nr, (int64_t)n, st);
        cudaFreeAsync(tmp, st);
        int64_t npc = 0;
        NRT_CUDA(cudaMemcpyAsync(&npc, nr, 8, cudaMemcpyDeviceToHost, st));
        NRT_CUDA(cudaStreamSynchronize(st));
        NRT_CUDA(cudaMemsetAsync(cnt + npc, 0, 4, st));
        tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, off, (int)(npc + 1), st);
        NRT_CUDA(cudaMallocAsync(&tmp, tb, st));
        cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, off, (int)(npc + 1), st);
        cudaFreeAsync(tmp, st);
        EnvIE* d_pc = nullptr;
        NRT_CUDA(cudaMallocAsync(&d_pc, (npc > 0 ? npc : 1) * sizeof(EnvIE), st));
        k_env_pcie<<<(unsigned)((npc + 127) / 128), 128, 0, st>>>(uniq, off, npc, vb.Current(), s->sp, s->label,
                                                                    s->sdf_org[0], s->sdf_org[1], s->sdf_org[2], S,
                                                                    sv[0], sv[1], d_pc);
        ::nrt::count_launch();
        ies.resize(npc);
        NRT_CUDA(cudaMemcpyAsync(ies.data(), d_pc, npc * sizeof(EnvIE), cudaMemcpyDeviceToHost, st));
        NRT_CUDA(cudaStreamSynchronize(st));
        for (void* p : {(void*)k0, (void*)k1, (void*)v0, (void*)v1, (void*)uniq, (void*)cnt, (void*)off, (void*)nr,
                        (void*)d_pc})
            cudaFreeAsync(p, st);
    }
    const int npc = (int)ies.size();
    std::vector<int> pc_of_sub(nsub, -1);
    for (int j = 0; j < npc; ++j) pc_of_sub[ies[j].ref] = j;
    // ---- DEIEs and RXIEs (host, the definition's FP32 arithmetic)
    for (int j = 0; j < s->n_edges; ++j) {
        const DevEdge& E = s->h_edges[j];
        const float ev[3] = {E.b_[0] - E.a[0], E.b_[1] - E.a[1], E.b_[2] - E.a[2]};
        const float len = sqrtf((ev[0] * ev[0] + ev[1] * ev[1]) + ev[2] * ev[2]);
        std::vector<float> ts{0.0f};
        for (int k = 0; k < 3; ++k) {
            if (ev[k] == 0.0f) continue;
            const float lo = fminf(E.a[k], E.b_[k]), hi = fmaxf(E.a[k], E.b_[k]);
            const int64_t m0 = (int64_t)floorf((lo - s->sdf_org[k]) / S), m1 = (int64_t)floorf((hi - s->sdf_org[k]) / S) + 1;
            for (int64_t m = m0; m <= m1 && ts.size() < 4094; ++m) {
                const float t = ((s->sdf_org[k] + (float)m * S) - E.a[k]) / ev[k];
                if (t > 0.0f && t < 1.0f) ts.push_back(t);
            }
        }
        ts.push_back(1.0f);
        std::sort(ts.begin(), ts.end());
        for (size_t q = 0; q + 1 < ts.size(); ++q) {
            if (!(ts[q + 1] > ts[q])) continue;
            const float tm = 0.5f * (ts[q] + ts[q + 1]);
            EnvIE I{};
            for (int k = 0; k < 3; ++k) I.p[k] = E.a[k] + tm * ev[k];
            I.kind = 1;
            I.label = E.label;
            I.ref = j;
            I.s_edge = tm * len;
            ies.push_back(I);
        }
    }
    for (int j = 0; j < a.n_rx; ++j) {
        EnvIE I{};
        for (int k = 0; k < 3; ++k) I.p[k] = a.h_rx[3 * j + k];
        I.kind = 2;
        I.label = j;
        I.ref = j;
        ies.push_back(I);
    }
    for (size_t i = npc; i < ies.size(); ++i)
        for (int k = 0; k < 3; ++k) {
            int64_t c = (int64_t)floorf((ies[i].p[k] - s->sdf_org[k]) / S);
            if (c < 0) c = 0;
            if (c > sv[k] - 1) c = sv[k] - 1;
            ies[i].sub[k] = (int)c;
        }
    const int n_ie = (int)ies.size();
    // R61: voxel lists, march distances, cone
    const int nv = vd[0] * vd[1] * vd[2];
    std::vector<int> vstart(nv + 1, 0), vids(n_ie > 0 ? n_ie : 1), vox(n_ie > 0 ? n_ie : 1), march(nv);
    for (int i = 0; i < n_ie; ++i) {
        int v3[3];
        for (int k = 0; k < 3; ++k) v3[k] = std::min(ies[i].sub[k] / 2, vd[k] - 1);
        vox[i] = v3[0] + vd[0] * (v3[1] + vd[1] * v3[2]);
        vstart[vox[i] + 1]++;
    }
    for (int v = 0; v < nv; ++v) vstart[v + 1] += vstart[v];
    {
        std::vector<int> fill(nv, 0);
        for (int i = 0; i < n_ie; ++i) vids[vstart[vox[i]] + fill[vox[i]]++] = i;
    }
    std::vector<int> occ;
    for (int u = 0; u < nv; ++u)
        if (vstart[u + 1] > vstart[u]) occ.push_back(u);
    for (int v = 0; v < nv; ++v) {
        const int x = v % vd[0], y = (v / vd[0]) % vd[1], z = v / (vd[0] * vd[1]);
        int best = 1 << 20;
        for (int u : occ) {
            const int ux = u % vd[0], uy = (u / vd[0]) % vd[1], uz = u / (vd[0] * vd[1]);
            const int dd = std::max(std::abs(ux - x), std::max(std::abs(uy - y), std::abs(uz - z)));
            best = std::min(best, dd);
        }
        march[v] = best < 1 ? 1 : best;
    }
    const float dg[3] = {s->sdf_bmax[0] - s->sdf_org[0], s->sdf_bmax[1] - s->sdf_org[1], s->sdf_bmax[2] - s->sdf_org[2]};
    const float D = sqrtf((dg[0] * dg[0] + dg[1] * dg[1]) + dg[2] * dg[2]);
    EnvArgs A{};
    A.tan_c = V / D;
    A.sec_c = sqrtf(1.0f + A.tan_c * A.tan_c);
    for (int k = 0; k < 3; ++k) {
        A.vd[k] = vd[k];
        A.sv[k] = sv[k];
        A.sd[k] = sd[k];
        A.org[k] = s->sdf_org[k];
        A.tx[k] = a.tx[k];
    }
    A.V = V;
    A.S = S;
    A.a = A0;
    A.n_ie = n_ie;
    A.max_refl = a.max_refl;
    A.max_diff = a.max_diff;
    A.dphi_deg = a.desc.dphi_deg;
    A.rank = a.desc.rank;
    A.world = a.desc.world;
    // ---- upload
    EnvIE* d_ie = nullptr;
    int *d_pcs = nullptr, *d_vs = nullptr, *d_vi = nullptr, *d_m = nullptr;
    unsigned long long* ctr = nullptr;  // [raw_n, n_out, work, rays, terms]
    NRT_CUDA(cudaMallocAsync(&d_ie, (n_ie > 0 ? n_ie : 1) * sizeof(EnvIE), st));
    NRT_CUDA(cudaMallocAsync(&d_pcs, nsub * 4, st));
    NRT_CUDA(cudaMallocAsync(&d_vs, (nv + 1) * 4, st));
    NRT_CUDA(cudaMallocAsync(&d_vi, (n_ie > 0 ? n_ie : 1) * 4, st));
    NRT_CUDA(cudaMallocAsync(&d_m, nv * 4, st));
    NRT_CUDA(cudaMallocAsync(&ctr, 5 * 8, st));
    NRT_CUDA(cudaMemcpyAsync(d_ie, ies.data(), n_ie * sizeof(EnvIE), cudaMemcpyHostToDevice, st));
    NRT_CUDA(cudaMemcpyAsync(d_pcs, pc_of_sub.data(), nsub * 4, cudaMemcpyHostToDevice, st));
    NRT_CUDA(cudaMemcpyAsync(d_vs, vstart.data(), (nv + 1) * 4, cudaMemcpyHostToDevice, st));
    NRT_CUDA(cudaMemcpyAsync(d_vi, vids.data(), n_ie * 4, cudaMemcpyHostToDevice, st));
    NRT_CUDA(cudaMemcpyAsync(d_m, march.data(), nv * 4, cudaMemcpyHostToDevice, st));
    NRT_CUDA(cudaMemsetAsync(ctr, 0, 5 * 8, st));
    const bool counters = a.desc.counters != 0;
    A.terms = counters ? ctr + 4 : nullptr;
    A.ie = d_ie;
    A.pc_of_sub = d_pcs;
    A.vstart = d_vs;
    A.vids = d_vi;
    A.march = d_m;
    A.raw_n = ctr;
    A.n_out = ctr + 1;
    A.work = ctr + 2;
    A.rays = ctr + 3;
    // ---- levels
    unsigned long long raw_cap = 1 << 16, out_cap = 1 << 16;
    nrt_coarse_rec* raw = nullptr;
    NRT_CUDA(cudaMallocAsync(&raw, raw_cap * sizeof(nrt_coarse_rec), st));
    CRay *qin = nullptr, *qout = nullptr;
    unsigned long long n_in = 0;
    NRT_CUDA(cudaMallocAsync(&qout, out_cap * sizeof(CRay), st));
    const int sms = sm_count(s->device);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_env_prop<false>, 128, 0);
    if (per_sm < 1) per_sm = 1;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float tot = 0.0f;
    double ratio = 24.0;
    for (int level = 0; level <= NRT_MAX_INT; ++level) {
        if (level > 0 && n_in == 0) break;
        const unsigned long long items_done = level == 0 ? (unsigned long long)n_ie : n_in;
        unsigned long long h[4];
        NRT_CUDA(cudaMemcpyAsync(h, ctr, sizeof(h), cudaMemcpyDeviceToHost, st));
        NRT_CUDA(cudaStreamSynchronize(st));
        unsigned long long t5 = 0;
        NRT_CUDA(cudaMemcpyAsync(&t5, ctr + 4, 8, cudaMemcpyDeviceToHost, st));
        NRT_CUDA(cudaStreamSynchronize(st));
        const unsigned long long raw0 = h[0], rays0 = h[3], terms0 = t5;
        for (int attempt = 0; attempt < 4; ++attempt) {
            unsigned long long z[5] = {raw0, 0, 0, rays0, terms0};  // a re-run starts from the level's counts
            NRT_CUDA(cudaMemcpyAsync(ctr, z, 5 * 8, cudaMemcpyHostToDevice, st));
            A.raw = raw;
            A.raw_cap = raw_cap;
            A.out = qout;
            A.out_cap = out_cap;
            A.in = qin;
            A.n_in = n_in;
            const unsigned long long items = level == 0 ? (unsigned long long)n_ie : n_in;
            // grow the record buffer ahead of the level (a re-run costs the whole level)
            const unsigned long long rest = std::min<unsigned long long>(raw0 + 8 * items + 4096, 1ull << 25);
            if (attempt == 0 && raw_cap < rest) {
                nrt_coarse_rec* nr2 = nullptr;
                NRT_CUDA(cudaMallocAsync(&nr2, rest * sizeof(nrt_coarse_rec), st));
                if (raw0) NRT_CUDA(cudaMemcpyAsync(nr2, raw, raw0 * sizeof(nrt_coarse_rec), cudaMemcpyDeviceToDevice, st));
                cudaFreeAsync(raw, st);
                raw = nr2;
                raw_cap = rest;
                A.raw = raw;
                A.raw_cap = raw_cap;
            }
            // children of this level: the previous level's ratio (x 1.25), 24 at the start
            const unsigned long long est = std::min<unsigned long long>(
                (unsigned long long)(1.25 * ratio * (double)items) + 4096, 1ull << 26);
            if (attempt == 0 && out_cap < est && level < NRT_MAX_INT) {  // children: ~10-100 per item
                cudaFreeAsync(qout, st);
                out_cap = est;
                NRT_CUDA(cudaMallocAsync(&qout, out_cap * sizeof(CRay), st));
                A.out = qout;
                A.out_cap = out_cap;
            }
            unsigned blocks = (unsigned)std::min<unsigned long long>((unsigned long long)sms * per_sm, (items + 3) / 4);
            if (blocks < 1) blocks = 1;
            cudaEventRecord(e0, st);
            if (level == 0) {
                if (counters) k_env_tx<true><<<blocks, 128, 0, st>>>(P, A);
                else k_env_tx<false><<<blocks, 128, 0, st>>>(P, A);
            } else if (counters) {
                k_env_prop<true><<<blocks, 128, 0, st>>>(P, A);
            } else {
                k_env_prop<false><<<blocks, 128, 0, st>>>(P, A);
            }
            ::nrt::count_launch();
            cudaEventRecord(e1, st);
            NRT_CUDA(cudaGetLastError());
            NRT_CUDA(cudaMemcpyAsync(h, ctr, sizeof(h), cudaMemcpyDeviceToHost, st));
            NRT_CUDA(cudaStreamSynchronize(st));
            float ms = 0.0f;
            cudaEventElapsedTime(&ms, e0, e1);
            if (getenv("NRT_PHASES"))
                fprintf(stderr, "[nrt] cone level %d attempt %d: %llu items, %.3f ms, children %llu/%llu, records %llu/%llu\n",
                        level, attempt, items, ms, h[1], out_cap, h[0], raw_cap);
            if (h[0] <= raw_cap && h[1] <= out_cap) {
                tot += ms;
                break;
            }
            // overflow: grow and re-run this level (deterministic: the same inputs)
            if (h[0] > raw_cap) {
                nrt_coarse_rec* nr2 = nullptr;
                const unsigned long long cap2 = h[0] + h[0] / 2 + 1024;
                NRT_CUDA(cudaMallocAsync(&nr2, cap2 * sizeof(nrt_coarse_rec), st));
                NRT_CUDA(cudaMemcpyAsync(nr2, raw, raw0 * sizeof(nrt_coarse_rec), cudaMemcpyDeviceToDevice, st));
                cudaFreeAsync(raw, st);
                raw = nr2;
                raw_cap = cap2;
            }
            if (h[1] > out_cap) {
                cudaFreeAsync(qout, st);
                out_cap = h[1] + h[1] / 2 + 1024;
                NRT_CUDA(cudaMallocAsync(&qout, out_cap * sizeof(CRay), st));
            }
        }
        // the children become the next level's input
        if (items_done > 0 && h[1] > 0) ratio = (double)h[1] / (double)items_done;
        n_in = h[1];
        if (qin) cudaFreeAsync(qin, st);
        qin = qout;
        qout = nullptr;
        NRT_CUDA(cudaMallocAsync(&qout, out_cap * sizeof(CRay), st));
    }
    unsigned long long h[5];
    NRT_CUDA(cudaMemcpyAsync(h, ctr, sizeof(h), cudaMemcpyDeviceToHost, st));
    NRT_CUDA(cudaStreamSynchronize(st));
    *terms_out = h[4];
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    for (void* p : {(void*)d_ie, (void*)d_pcs, (void*)d_vs, (void*)d_vi, (void*)d_m, (void*)ctr, (void*)qin, (void*)qout})
        if (p) cudaFreeAsync(p, st);
    *raw_out = raw;
    *n_raw = (int64_t)h[0];
    *rays = h[3];
    *ms_kernel = tot;
    return NRT_OK;
}


// NEXT-4 host side: one warp per path of the shard j == rank (mod world); valid paths (or all,
// keep_invalid) -> R28 shortest per key, as the Gauss-Newton refinement's output
nrt_status refine_gd(nrt_scene s, nrt_paths coarse, const nrt_refine_desc* d, nrt_paths out, cudaStream_t st) {
    const int64_t n = coarse->n;
    out->n = 0;
    TP P{};
    P.label = s->label;
    P.edges = s->edges;
    P.n_edges = s->n_edges;
    P.sdf = 1;
    P.sdf_pts = s->sdf_pts;
    P.sdf_box = s->sdf_box;
    P.sdf_acell = s->sdf_acell;
    P.sdf_gcell = s->sdf_gcell;
    P.sdf_aref = s->sdf_aref;
    P.sdf_crange = s->sdf_crange;
    P.sn_p = s->sp;
    for (int k = 0; k < 3; ++k) {
        P.sg_o[k] = s->sdf_gorg[k];
        P.sg_n[k] = s->sdf_gdims[k];
        P.sd_n[k] = s->sdf_dims[k];
        P.sd_o[k] = s->sdf_org[k];
    }
    P.sdf_a = s->sdf_a;
    P.sdf_inv_a = 1.0f / s->sdf_a;
    P.sdf_half = 0.5f * (s->sdf_a * 1.7320508f);
    P.sdf_stop = 2.0f * P.sdf_half + s->sdf_pad;
    // FP32 parameters as the definition forms them (R50-R56)
    P.sdf_rs = (float)d->r_s;
    P.sdf_tsdf = (float)d->gd_t_sdf;
    const float sigma = (float)d->xi * (float)d->r_s;
    P.sdf_sigma = sigma;
    P.sdf_inv = 1.0f / (2.0f * sigma * sigma);
    P.tau = (float)d->tau;
    P.cos_ex = cos_ex_of((float)d->theta_ex_deg);
    GdArgs A{};
    A.in = (const nrt_coarse_rec*)coarse->d_rec;
    A.n_in = n;
    A.rank = d->rank;
    A.world = d->world;
    A.keep_invalid = d->keep_invalid;
    for (int k = 0; k < 3; ++k) A.tx[k] = coarse->tx[k];
    A.rho = d->gd_rho;
    A.alpha = (float)d->alpha;
    A.beta = (float)d->beta;
    A.delta = (float)d->delta;
    A.t_d = (float)d->gd_t_d;
    A.cos_ta = cos_ex_of((float)d->gd_t_a_deg);
    A.margin = 2.0f * sigma;
    const int64_t n_mine = n > d->rank ? (n - d->rank + d->world - 1) / d->world : 0;
    float* d_rx = nullptr;
    const size_t nrx = coarse->rx.size();
    NRT_CUDA(cudaMallocAsync(&d_rx, (nrx ? nrx : 3) * sizeof(float), st));
    if (nrx) NRT_CUDA(cudaMemcpyAsync(d_rx, coarse->rx.data(), nrx * sizeof(float), cudaMemcpyHostToDevice, st));
    A.rx = d_rx;
    nrt_refined_rec* o = nullptr;
    NRT_CUDA(cudaMallocAsync(&o, (size_t)(n_mine > 0 ? n_mine : 1) * sizeof(nrt_refined_rec), st));
    unsigned long long* ctr = nullptr;
    NRT_CUDA(cudaMallocAsync(&ctr, 3 * sizeof(unsigned long long), st));
    NRT_CUDA(cudaMemsetAsync(ctr, 0, 3 * sizeof(unsigned long long), st));
    A.out = o;
    A.n_ok = ctr;
    A.work = ctr + 1;
    A.terms = d->counters ? ctr + 2 : nullptr;
    const int dev = s->device;
    int per_sm = 0;
    if (d->counters) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_refine_gd<true>, 128, 0);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_refine_gd<false>, 128, 0);
    if (per_sm < 1) per_sm = 1;
    int64_t blocks = (int64_t)sm_count(dev) * per_sm;
    if (blocks > (n_mine + 3) / 4) blocks = (n_mine + 3) / 4;
    if (blocks < 1) blocks = 1;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
    if (n_mine > 0) {
        if (d->counters) k_refine_gd<true><<<(unsigned)blocks, 128, 0, st>>>(P, A);
        else k_refine_gd<false><<<(unsigned)blocks, 128, 0, st>>>(P, A);
        ::nrt::count_launch();
    }
    cudaEventRecord(e1, st);
    NRT_CUDA(cudaGetLastError());
    unsigned long long hctr[3] = {0, 0, 0};
    NRT_CUDA(cudaMemcpyAsync(hctr, ctr, sizeof(hctr), cudaMemcpyDeviceToHost, st));
    NRT_CUDA(cudaStreamSynchronize(st));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    out->info.ms_refine = ms;
    out->info.mls_value = hctr[2];  // Gaussian terms of the SDF evaluations (counters)
    cudaFreeAsync(d_rx, st);
    cudaFreeAsync(ctr, st);
    if (d->keep_invalid) {
        out->d_rec = o;
        out->n = n_mine;
    } else {
        nrt_refined_rec* u = nullptr;
        NRT_CUDA(cudaMallocAsync(&u, (size_t)(hctr[0] > 0 ? hctr[0] : 1) * sizeof(nrt_refined_rec), st));
        int64_t m = 0;
        NRT_TRY(dedupe_refined(o, (int64_t)hctr[0], u, &m, st));
        cudaFreeAsync(o, st);
        out->d_rec = u;
        out->n = m;
    }
    NRT_CUDA(cudaStreamSynchronize(st));
    out->info.n = out->n;
    out->info.n_raw = n_mine;
    return NRT_OK;
}

// per-segment hit ids of explicit primary rays, traced by the production wavefront (the same
// k_trace / k_shade launches, refill and reorder paths as nrt_launch); no records are emitted
nrt_status debug_trace(nrt_scene s, const LaunchArgs& a, const uint64_t* ids, int64_t n,
                       int64_t* hit_ids, cudaStream_t st) {
    if (n <= 0) return NRT_OK;
    TP P = make_tp(s, a);
    uint64_t* dids = nullptr;
    int64_t* dh = nullptr;
    const size_t nseg = (size_t)a.max_refl + 1;
    Counters* dc = nullptr;
    NRT_CUDA(cudaMallocAsync(&dc, sizeof(Counters), st));
    NRT_CUDA(cudaMemsetAsync(dc, 0, sizeof(Counters), st));
    NRT_CUDA(cudaMallocAsync(&dids, n * 8, st));
    NRT_CUDA(cudaMallocAsync(&dh, n * nseg * 8, st));
    NRT_CUDA(cudaMemcpyAsync(dids, ids, n * 8, cudaMemcpyHostToDevice, st));
    Wave W{};
    WaveGuard wg{&W, st};
    NRT_TRY(alloc_wave(W, (uint64_t)n, s->device, P.sdf != 0, st));
    if (reorder_on(s)) W.skey = W.okey[0];
    W.n_alive = dc->n_alive;
    W.ctr = dc->ctr;
    P.raw = nullptr;
    P.raw_cap = 0;
    P.raw_n = &dc->raw_n;
    P.ev = nullptr;
    P.ev_cap = 0;
    P.ev_n = &dc->ev_n;
    P.bounces = &dc->bounces;
    P.counters = &dc->tests;
    P.n_edges = 0;
    P.hit_out = dh;
    unsigned gb = (unsigned)((n + 255) / 256);
    if (gb > (unsigned)sm_count(s->device) * 16) gb = (unsigned)sm_count(s->device) * 16;
    k_gen_ids<<<gb, 256, 0, st>>>(P, W, dids, (uint64_t)n);
    ::nrt::count_launch();
    float ms = 0.0f;
    NRT_TRY(run_bounces(P, W, (uint64_t)n, a.max_refl + 1, s->device, false, &ms, st));
    NRT_CUDA(cudaGetLastError());
    NRT_CUDA(cudaMemcpyAsync(hit_ids, dh, n * nseg * 8, cudaMemcpyDeviceToHost, st));
    NRT_CUDA(cudaStreamSynchronize(st));
    free_wave(W, st);
    cudaFreeAsync(dids, st);
    cudaFreeAsync(dh, st);
    cudaFreeAsync(dc, st);
    return NRT_OK;
}

}  // namespace nrt
