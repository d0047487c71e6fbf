// launch.cu — A2-A7: Fibonacci ray generation, 3D-DDA nearest-surfel traversal, specular
// reflection, RX reception spheres, edge capture and Keller fans.
//
// Per ray, per segment, the hit is the lexicographic min (t, id) of the HIT predicate
// (R7-R9).  The grid walk only accelerates that argmin: every surfel is registered in all
// cells its padded disk AABB overlaps, and the walk stops only once best_t < t_exit - pad
// (DESIGN.md §6), so the result equals the brute-force definition for any voxel size.
// All FP32 arithmetic of the definition is done in the order DESIGN.md R3 fixes; the
// library is compiled with -fmad=false so no FMA contraction alters a rounding.
#include <cooperative_groups.h>

#include <cub/cub.cuh>

#include <cmath>
#include <cstring>

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
    const DevEdge* edges;
    int n_edges;
    // outputs
    nrt_coarse_rec* raw;
    unsigned long long raw_cap;
    unsigned long long* raw_n;
    nrt_event_rec* ev;
    unsigned long long ev_cap;
    unsigned long long* ev_n;
    unsigned long long* bounces;
    unsigned long long* counters;  // [tests, cells, nonempty cells] (instrumented build)
    int64_t* hit_out;  // debug: per-segment hit ids
};

__device__ __forceinline__ unsigned long long agg_inc(unsigned long long* ctr) {
    cg::coalesced_group g = cg::coalesced_threads();
    unsigned long long base = 0;
    if (g.thread_rank() == 0) base = atomicAdd(ctr, (unsigned long long)g.size());
    base = g.shfl(base, 0);
    return base + g.thread_rank();
}

// ---- A3: nearest surfel along (o, d) by 3D-DDA over the fine grid -----------------------
struct Cnt {
    unsigned long long tests = 0, cells = 0, nonempty = 0;
};

template <bool CNT>
__device__ int nearest(const TP& P, float3 o, float3 d, float3 l0, float3 l1, int prev,
                       float& t_out, Cnt& cnt) {
    float best_t = INFINITY;
    int best = -1;
    // grid entry (slab test); the walk only needs a conservative start
    const float gx1 = P.ox + P.nx * P.v, gy1 = P.oy + P.ny * P.v, gz1 = P.oz + P.nz * P.v;
    float ix_ = 1.0f / d.x, iy_ = 1.0f / d.y, iz_ = 1.0f / d.z;
    float t0 = 0.0f, t1 = INFINITY;
    {
        float a = (P.ox - o.x) * ix_, b = (gx1 - o.x) * ix_;
        if (d.x != 0.0f) { t0 = fmaxf(t0, fminf(a, b)); t1 = fminf(t1, fmaxf(a, b)); }
        else if (o.x < P.ox || o.x > gx1) t1 = -1.0f;
        a = (P.oy - o.y) * iy_; b = (gy1 - o.y) * iy_;
        if (d.y != 0.0f) { t0 = fmaxf(t0, fminf(a, b)); t1 = fminf(t1, fmaxf(a, b)); }
        else if (o.y < P.oy || o.y > gy1) t1 = -1.0f;
        a = (P.oz - o.z) * iz_; b = (gz1 - o.z) * iz_;
        if (d.z != 0.0f) { t0 = fmaxf(t0, fminf(a, b)); t1 = fminf(t1, fmaxf(a, b)); }
        else if (o.z < P.oz || o.z > gz1) t1 = -1.0f;
    }
    if (t0 > t1) {
        t_out = INFINITY;
        return -1;
    }
    float sx = o.x + t0 * d.x, sy = o.y + t0 * d.y, sz = o.z + t0 * d.z;
    int ix = min(P.nx - 1, max(0, (int)floorf((sx - P.ox) * P.inv_v)));
    int iy = min(P.ny - 1, max(0, (int)floorf((sy - P.oy) * P.inv_v)));
    int iz = min(P.nz - 1, max(0, (int)floorf((sz - P.oz) * P.inv_v)));
    const int stx = d.x > 0.0f ? 1 : -1, sty = d.y > 0.0f ? 1 : -1, stz = d.z > 0.0f ? 1 : -1;
    float tmx = d.x != 0.0f ? ((P.ox + (float)(ix + (stx > 0)) * P.v) - o.x) * ix_ : INFINITY;
    float tmy = d.y != 0.0f ? ((P.oy + (float)(iy + (sty > 0)) * P.v) - o.y) * iy_ : INFINITY;
    float tmz = d.z != 0.0f ? ((P.oz + (float)(iz + (stz > 0)) * P.v) - o.z) * iz_ : INFINITY;
    const float tau = P.tau, cex = P.cos_ex;
    for (;;) {
        const uint2 rg = __ldg(&P.cell[ix + P.nx * (iy + P.ny * iz)]);
        if (CNT) {
            cnt.cells++;
            cnt.tests += rg.y - rg.x;
            cnt.nonempty += rg.y > rg.x;
        }
        for (unsigned k = rg.x; k < rg.y; ++k) {
            const float4 A = __ldg(&P.rec[2 * k]);
            const float4 B = __ldg(&P.rec[2 * k + 1]);
            const int id = __float_as_int(B.w);
            const float wx = o.x - A.x, wy = o.y - A.y, wz = o.z - A.z;
            const float f0 = (wx * B.x + wy * B.y) + wz * B.z;
            const float dn = (d.x * B.x + d.y * B.y) + d.z * B.z;
            if (!(f0 * dn < 0.0f) || id == prev) continue;
            if (fabsf(f0) <= tau) {
                const float c0 = (B.x * l0.x + B.y * l0.y) + B.z * l0.z;
                const float c1 = (B.x * l1.x + B.y * l1.y) + B.z * l1.z;
                if (fabsf(c0) >= cex || fabsf(c1) >= cex) continue;
            }
            const float t = (-f0) / dn;
            if (t > best_t) continue;
            const float hx = o.x + t * d.x, hy = o.y + t * d.y, hz = o.z + t * d.z;
            const float qx = hx - A.x, qy = hy - A.y, qz = hz - A.z;
            const float qq = (qx * qx + qy * qy) + qz * qz;
            if (qq <= A.w && (t < best_t || id < best)) {
                best_t = t;
                best = id;
            }
        }
        const float te = fminf(tmx, fminf(tmy, tmz));
        if (best_t < te - P.pad) break;
        if (tmx <= tmy && tmx <= tmz) {
            ix += stx;
            if (ix < 0 || ix >= P.nx) break;
            tmx = ((P.ox + (float)(ix + (stx > 0)) * P.v) - o.x) * ix_;
        } else if (tmy <= tmz) {
            iy += sty;
            if (iy < 0 || iy >= P.ny) break;
            tmy = ((P.oy + (float)(iy + (sty > 0)) * P.v) - o.y) * iy_;
        } else {
            iz += stz;
            if (iz < 0 || iz >= P.nz) break;
            tmz = ((P.oz + (float)(iz + (stz > 0)) * P.v) - o.z) * iz_;
        }
    }
    t_out = best_t;
    return best;
}

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
        c.label[k] = on ? h.label[k] : 0;
        c.prim[k] = on ? h.prim[k] : 0u;
        c.v[k][0] = on ? h.v[k][0] : 0.0f;
        c.v[k][1] = on ? h.v[k][1] : 0.0f;
        c.v[k][2] = on ? h.v[k][2] : 0.0f;
    }
    c.s_edge = h.s_edge;
    c.L = L;
    c.ray_id = ray_id;
    P.raw[slot] = c;
}

// ---- A5: RX reception spheres (R12 / R16) ---------------------------------------------
__device__ void rx_captures(const TP& P, const Hist& h, float3 o, float3 d, float t_hit, float L,
                            float Ls, float kR, float R0, bool after_diff, uint64_t ray_id) {
    for (int j = 0; j < P.n_rx; ++j) {
        const float x0 = P.rx[3 * j], x1 = P.rx[3 * j + 1], x2 = P.rx[3 * j + 2];
        const float wx = x0 - o.x, wy = x1 - o.y, wz = x2 - o.z;
        const float tj = (wx * d.x + wy * d.y) + wz * d.z;
        if (!(tj > 0.0f && tj < t_hit)) continue;
        const float px = wx - tj * d.x, py = wy - tj * d.y, pz = wz - tj * d.z;
        const float pp = (px * px + py * py) + pz * pz;
        const float R = after_diff ? kR * (Ls + tj) + R0 : kR * (L + tj);
        if (!(pp <= R * R)) continue;
        write_record(P, h, j, L + tj, ray_id);
    }
}

// ---- A6: edge capture -> diffraction events (R13) --------------------------------------
__device__ void edge_captures(const TP& P, const Hist& h, float3 o, float3 d, float t_hit,
                              float L, uint64_t ray_id) {
    for (int j = 0; j < P.n_edges; ++j) {
        const DevEdge& E = P.edges[j];
        const float b = (d.x * E.e[0] + d.y * E.e[1]) + d.z * E.e[2];
        const float w0x = o.x - E.a[0], w0y = o.y - E.a[1], w0z = o.z - E.a[2];
        const float den = 1.0f - b * b;
        if (!(den > 1e-12f)) continue;
        const float de = (E.e[0] * w0x + E.e[1] * w0y) + E.e[2] * w0z;
        const float dd = (d.x * w0x + d.y * w0y) + d.z * w0z;
        const float te = (b * de - dd) / den;
        const float s = (de - b * dd) / den;
        if (!(s >= 0.0f && s <= E.len)) continue;
        if (!(te > 0.0f && te < t_hit + P.b_e)) continue;
        const float pcx = o.x + te * d.x, pcy = o.y + te * d.y, pcz = o.z + te * d.z;
        const float pex = E.a[0] + s * E.e[0], pey = E.a[1] + s * E.e[1], pez = E.a[2] + s * E.e[2];
        const float dx = pcx - pex, dy = pcy - pey, dz = pcz - pez;
        const float dist2 = (dx * dx + dy * dy) + dz * dz;
        const float R = P.cRw * (L + te);
        if (!(dist2 <= R * R)) continue;
        unsigned long long slot = agg_inc(P.ev_n);
        if (slot >= P.ev_cap) continue;
        nrt_event_rec e;
        e.n_hist = h.n;
        e.n_diff = h.n_diff;
        e.kinds = (uint16_t)h.kinds;
        e.pad_ = 0;
#pragma unroll
        for (int k = 0; k < NRT_MAX_INT; ++k) {
            bool on = k < h.n;
            e.label[k] = on ? h.label[k] : 0;
            e.prim[k] = on ? h.prim[k] : 0u;
            e.v[k][0] = on ? h.v[k][0] : 0.0f;
            e.v[k][1] = on ? h.v[k][1] : 0.0f;
            e.v[k][2] = on ? h.v[k][2] : 0.0f;
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
}

// ---- C.1 step 2: one ray (primary or fan) --------------------------------------------
template <bool CNT>
__device__ void trace(const TP& P, Hist& h, float3 o, float3 d, float L, int budget,
                      bool allow_edges, float3 l0, float3 l1, bool after_diff, float kR, float R0,
                      uint64_t ray_id, unsigned long long& bounces, int64_t* hit_out, Cnt& cnt) {
    float Ls = 0.0f;
    int prev = -1;
    for (int seg = 0; seg <= budget; ++seg) {
        float th;
        const int s = nearest<CNT>(P, o, d, l0, l1, prev, th, cnt);
        ++bounces;
        if (hit_out) hit_out[seg] = s;
        rx_captures(P, h, o, d, th, L, Ls, kR, R0, after_diff, ray_id);
        if (allow_edges && h.n_diff < P.max_diff && h.n < NRT_MAX_INT)
            edge_captures(P, h, o, d, th, L, ray_id);
        if (s < 0 || seg == budget) break;
        // A4: reflect (d' = d - (2 d.n) n, normalised)
        const float3 hp = make_float3(o.x + th * d.x, o.y + th * d.y, o.z + th * d.z);
        const float4 nv = __ldg(&P.sn[s]);
        const float3 n = make_float3(nv.x, nv.y, nv.z);
        h.label[h.n] = __ldg(&P.label[s]);
        h.prim[h.n] = (uint32_t)s;
        h.v[h.n][0] = hp.x;
        h.v[h.n][1] = hp.y;
        h.v[h.n][2] = hp.z;
        h.n++;
        const float k2 = 2.0f * dot3(d, n);
        const float3 x = make_float3(d.x - k2 * n.x, d.y - k2 * n.y, d.z - k2 * n.z);
        const float l = sqrtf(dot3(x, x));
        d = make_float3(x.x / l, x.y / l, x.z / l);
        o = hp;
        L = L + th;
        Ls = Ls + th;
        l0 = n;
        l1 = n;
        prev = s;
    }
}

__device__ __forceinline__ void flush_counts(const TP& P, unsigned long long bounces, const Cnt& c,
                                             bool cnt_on) {
    for (int off = 16; off > 0; off >>= 1) bounces += __shfl_down_sync(0xffffffffu, bounces, off);
    if ((threadIdx.x & 31) == 0) atomicAdd(P.bounces, bounces);
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

template <bool CNT>
__global__ void __launch_bounds__(128) k_primary(TP P, uint64_t n_shard) {
    unsigned long long bounces = 0;
    Cnt cnt;
    const float3 z3 = make_float3(0.0f, 0.0f, 0.0f);
    const bool edges_on = P.n_edges > 0 && P.max_diff > 0;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_shard;
         j += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = (uint64_t)P.rank + j * (uint64_t)P.world;
        Hist h;
        h.n = 0;
        h.n_diff = 0;
        h.kinds = 0;
        h.s_edge = 0.0f;
        const float3 d = fib_dir(i, P.n_rays);
        trace<CNT>(P, h, make_float3(P.tx, P.ty, P.tz), d, 0.0f, P.max_refl, edges_on, z3, z3,
                   false, P.cRw, 0.0f, i, bounces, nullptr, cnt);
    }
    flush_counts(P, bounces, cnt, CNT);
}

__global__ void k_debug(TP P, const uint64_t* ids, int64_t n) {
    int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    unsigned long long b = 0;
    Hist h;
    h.n = 0;
    h.n_diff = 0;
    h.kinds = 0;
    h.s_edge = 0.0f;
    const float3 z3 = make_float3(0.0f, 0.0f, 0.0f);
    int64_t* out = P.hit_out + q * (P.max_refl + 1);
    for (int k = 0; k <= P.max_refl; ++k) out[k] = -2;
    Cnt cnt;
    trace<false>(P, h, make_float3(P.tx, P.ty, P.tz), fib_dir(ids[q], P.n_rays), 0.0f, P.max_refl,
                 false, z3, z3, false, P.cRw, 0.0f, ids[q], b, out, cnt);
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

template <bool CNT>
__global__ void __launch_bounds__(128) k_fans(TP P, const nrt_event_rec* ev, int64_t n_ev,
                                              const unsigned int* off, unsigned int total) {
    unsigned long long bounces = 0;
    Cnt cnt;
    for (unsigned f = blockIdx.x * blockDim.x + threadIdx.x; f < total;
         f += gridDim.x * blockDim.x) {
        // event r: last r with off[r] <= f
        int64_t lo = 0, hi = n_ev - 1;
        while (lo < hi) {
            int64_t mid = (lo + hi + 1) >> 1;
            if (off[mid] <= f) lo = mid;
            else hi = mid - 1;
        }
        const int64_t r = lo;
        const int m = (int)(f - off[r]);
        const nrt_event_rec& e = ev[r];
        const DevEdge& E = P.edges[e.edge];
        const FanGeo g = fan_geo(P, e);
        const double wedge = (double)E.n_exp * kPi;
        const float kR = (float)((double)P.c_R * (wedge / (double)g.M) * g.st);
        const float R0 = 0.5f * P.edge_bin;
        const float3 o = make_float3(E.a[0] + e.s * E.e[0], E.a[1] + e.s * E.e[1],
                                     E.a[2] + e.s * E.e[2]);
        Hist h;
        h.n = e.n_hist;
        h.n_diff = e.n_diff;
        h.kinds = e.kinds;
        for (int k = 0; k < NRT_MAX_INT; ++k) {
            h.label[k] = e.label[k];
            h.prim[k] = e.prim[k];
            h.v[k][0] = e.v[k][0];
            h.v[k][1] = e.v[k][1];
            h.v[k][2] = e.v[k][2];
        }
        h.label[h.n] = E.label;
        h.prim[h.n] = e.edge;
        h.v[h.n][0] = o.x;
        h.v[h.n][1] = o.y;
        h.v[h.n][2] = o.z;
        h.kinds |= 1u << h.n;
        h.n++;
        h.n_diff++;
        h.s_edge = e.s;
        int n_refl = 0;
        for (int k = 0; k < e.n_hist; ++k)
            if (!((e.kinds >> k) & 1u)) n_refl++;
        int budget = P.max_refl - n_refl;
        if (budget < 0) continue;
        if (h.n + budget > NRT_MAX_INT) budget = NRT_MAX_INT - h.n;
        const double phi = (((double)m + 0.5) * wedge) / (double)g.M;
        double sp, cp;
        nrt_sincos(phi, &sp, &cp);
        float dir[3];
        for (int k = 0; k < 3; ++k) {
            const double x2 = cp * (double)E.t0[k] + sp * (double)E.n0[k];
            dir[k] = (float)(x2 * g.st + (double)E.e[k] * g.ct);
        }
        const uint64_t rid = (1ull << 63) | ((uint64_t)r << 8) | (uint64_t)m;
        trace<CNT>(P, h, o, make_float3(dir[0], dir[1], dir[2]), e.L, budget, false,
                   make_float3(E.n0[0], E.n0[1], E.n0[2]), make_float3(E.n1[0], E.n1[1], E.n1[2]),
                   true, kR, R0, rid, bounces, nullptr, cnt);
    }
    flush_counts(P, bounces, cnt, CNT);
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
    P.pad = s->pad;
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

}  // namespace

struct Counters {
    unsigned long long raw_n, ev_n, bounces, tests, cells, nonempty;
};

nrt_status launch_primary(nrt_scene s, const LaunchArgs& a, nrt_coarse_rec** raw_out,
                          int64_t* n_raw, nrt_event_rec** ev_out, int64_t* n_ev,
                          uint64_t* bounces, KernelStats* stats, cudaStream_t st) {
    TP P = make_tp(s, a);
    const uint64_t n_shard =
        a.n_rays > a.desc.rank ? ((uint64_t)a.n_rays - a.desc.rank + a.desc.world - 1) / a.desc.world
                               : 0;
    unsigned long long raw_cap = 1 << 16, ev_cap = 1 << 14;
    Counters* dc = nullptr;
    NRT_CUDA(cudaMallocAsync(&dc, sizeof(Counters), st));
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
        const int sms = sm_count(s->device);
        uint64_t blocks = (n_shard + 127) / 128;
        const uint64_t maxb = (uint64_t)sms * 16;
        if (blocks > maxb) blocks = maxb;
        if (blocks < 1) blocks = 1;
        P.counters = &dc->tests;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, st);
        if (a.desc.counters) k_primary<true><<<(unsigned)blocks, 128, 0, st>>>(P, n_shard);
        else k_primary<false><<<(unsigned)blocks, 128, 0, st>>>(P, n_shard);
        ::nrt::count_launch();
        cudaEventRecord(e1, st);
        NRT_CUDA(cudaGetLastError());
        NRT_CUDA(cudaMemcpyAsync(&hc, dc, sizeof(hc), cudaMemcpyDeviceToHost, st));
        NRT_CUDA(cudaStreamSynchronize(st));
        cudaEventElapsedTime(&stats->ms_kernel, e0, e1);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        stats->tests = hc.tests;
        stats->cells = hc.cells;
        stats->nonempty = hc.nonempty;
        if (hc.raw_n <= raw_cap && hc.ev_n <= ev_cap) break;
        cudaFreeAsync(raw, st);
        cudaFreeAsync(ev, st);
        raw_cap = hc.raw_n > raw_cap ? hc.raw_n : raw_cap;
        ev_cap = hc.ev_n > ev_cap ? hc.ev_n : ev_cap;
    }
    cudaFreeAsync(dc, st);
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
    k_fan_count<<<(unsigned)((n_ev + 127) / 128), 128, 0, st>>>(P, ev, n_ev, cnt); ::nrt::count_launch();
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
    unsigned long long raw_cap = 1 << 16;
    nrt_coarse_rec* raw = nullptr;
    Counters hc{};
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
        const int sms = sm_count(s->device);
        uint64_t blocks = (total + 127) / 128;
        if (blocks > (uint64_t)sms * 16) blocks = (uint64_t)sms * 16;
        P.counters = &dc->tests;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, st);
        if (a.desc.counters) k_fans<true><<<(unsigned)blocks, 128, 0, st>>>(P, ev, n_ev, off, total);
        else k_fans<false><<<(unsigned)blocks, 128, 0, st>>>(P, ev, n_ev, off, total);
        ::nrt::count_launch();
        cudaEventRecord(e1, st);
        NRT_CUDA(cudaGetLastError());
        NRT_CUDA(cudaMemcpyAsync(&hc, dc, sizeof(hc), cudaMemcpyDeviceToHost, st));
        NRT_CUDA(cudaStreamSynchronize(st));
        cudaEventElapsedTime(&stats->ms_kernel, e0, e1);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        stats->tests = hc.tests;
        stats->cells = hc.cells;
        stats->nonempty = hc.nonempty;
        if (hc.raw_n <= raw_cap) break;
        cudaFreeAsync(raw, st);
        raw_cap = hc.raw_n;
    }
    cudaFreeAsync(dc, st);
    cudaFreeAsync(cnt, st);
    cudaFreeAsync(off, st);
    *raw_out = raw;
    *n_raw = (int64_t)hc.raw_n;
    *bounces = hc.bounces;
    return NRT_OK;
}

nrt_status debug_trace(nrt_scene s, const LaunchArgs& a, const uint64_t* ids, int64_t n,
                       int64_t* hit_ids, cudaStream_t st) {
    if (n <= 0) return NRT_OK;
    TP P = make_tp(s, a);
    uint64_t* dids = nullptr;
    int64_t* dh = nullptr;
    Counters* dc = nullptr;
    const size_t nseg = (size_t)a.max_refl + 1;
    NRT_CUDA(cudaMallocAsync(&dids, n * 8, st));
    NRT_CUDA(cudaMallocAsync(&dh, n * nseg * 8, st));
    NRT_CUDA(cudaMallocAsync(&dc, sizeof(Counters), st));
    NRT_CUDA(cudaMemsetAsync(dc, 0, sizeof(Counters), st));
    NRT_CUDA(cudaMemcpyAsync(dids, ids, n * 8, cudaMemcpyHostToDevice, st));
    P.raw = nullptr;
    P.raw_cap = 0;
    P.raw_n = &dc->raw_n;
    P.ev_n = &dc->ev_n;
    P.bounces = &dc->bounces;
    P.counters = &dc->tests;
    P.hit_out = dh;
    k_debug<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(P, dids, n); ::nrt::count_launch();
    NRT_CUDA(cudaGetLastError());
    NRT_CUDA(cudaMemcpyAsync(hit_ids, dh, n * nseg * 8, cudaMemcpyDeviceToHost, st));
    NRT_CUDA(cudaStreamSynchronize(st));
    cudaFreeAsync(dids, st);
    cudaFreeAsync(dh, st);
    cudaFreeAsync(dc, st);
    return NRT_OK;
}

}  // namespace nrt
