// refine.cu — A9-A10: batched path refinement, one warp per coarse path (FP64).
//
// The refined path is the root of the residual of DESIGN.md §5 (readings R18-R28):
//   reflection k: r_k = [g.u, g.v, f_sdf] with the MLS surface of Eqs. 1-4 over
//     the same-label surfels within 4 sigma (sigma = xi r_s), normals oriented by the
//     seed normal (Eq. 3 + R20), basis (u, v) of the MLS normal, g the Eq. 9-10 vector;
//   diffraction k: r_k = g.e (Eq. 11, I_k = a + t_k e, Eq. 8).
// reached by damped Gauss-Newton with a central-difference Jacobian (h = 1e-7), step
// -(J^T J + lam I)^-1 J^T r, Armijo backtracking (Eq. 12 form, R24), converged at |D|_inf <
// tol.  Then validity (R25): on-edge, same side, support, FP64 visibility; delay = L/c (R26).
//
// B200 mapping: a warp owns a path.  Per reflection vertex the warp gathers once the
// candidate surfels (same label, within Rq + M of a gather centre) from the fine grid into a
// per-warp scratch list; every MLS evaluation then streams that list with lanes splitting the
// candidates and a butterfly reduction of the 7 FP64 sums.  The small dense algebra lives in
// per-warp shared memory.  Shadow rays walk the same grid with the warp splitting each cell.
#include <cub/cub.cuh>

#include <cmath>
#include <cstdio>

#include "internal.cuh"

namespace nrt {

namespace {

constexpr int kWarps = 4;               // warps (paths in flight) per block
constexpr int kMaxDim = 3 * NRT_MAX_INT;
constexpr int kCap = 2048;              // candidate ids per vertex per warp slot
constexpr double kC = 299792458.0;
constexpr double kH = 1e-7;             // central-difference step (m)

struct RP {
    // grid (as in launch.cu)
    const uint2* cell;
    const float4* rec;
    const float4* sp;  // (p, r)
    const float4* sn;  // (n, label bits)
    float ox, oy, oz, v, inv_v, pad;
    int nx, ny, nz;
    const DevEdge* edges;
    // problem
    const nrt_coarse_rec* in;
    int64_t n_in;
    int rank, world;
    double tx[3];
    const float* rx;
    double sigma, rq, rg, tau, cos_ex, tol, alpha, beta;
    int max_iter;
    // outputs
    nrt_refined_rec* out;       // [n_in] (keep_invalid order) or compacted
    unsigned long long* n_out;
    int keep_invalid;
    // scratch
    unsigned* cand;             // [slots][NRT_MAX_INT][kCap]
    int slots;
    unsigned long long* work;   // path counter
};

struct Vtx {  // per-vertex gather state (warp-uniform)
    double c[3];
    int n;
    bool over;  // candidate list overflowed -> direct grid scan
};

struct WarpSmem {
    double J[kMaxDim * kMaxDim];
    double A[kMaxDim * kMaxDim];
    double r[kMaxDim], rp[kMaxDim], rm[kMaxDim], b[kMaxDim], z[kMaxDim], zt[kMaxDim];
    double pb[NRT_MAX_INT][3], nb[NRT_MAX_INT][3];  // MLS cache at z
    double pbx[3], nbx[3];                           // MLS at a perturbed vertex
    int ok;
};

__device__ __forceinline__ double ddot(const double a[3], const double b[3]) {
    return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
}

__device__ __forceinline__ double wsum(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

struct Path {
    int n, dim;
    int kind[NRT_MAX_INT];
    int32_t label[NRT_MAX_INT];
    uint32_t prim[NRT_MAX_INT];
    int col[NRT_MAX_INT];
    double nseed[NRT_MAX_INT][3];
    double ea[NRT_MAX_INT][3], ee[NRT_MAX_INT][3], elen[NRT_MAX_INT];
    double rxp[3];
};

// ---- candidate gather: home-cell records of the label within rg of c (superset of every
// neighbourhood the GN iterations evaluate while |x - c| <= rg - rq)
__device__ void gather(const RP& P, int32_t label, const double c[3], unsigned* list, Vtx& V,
                       int lane) {
    V.c[0] = c[0];
    V.c[1] = c[1];
    V.c[2] = c[2];
    V.over = false;
    const float lo[3] = {(float)(c[0] - P.rg), (float)(c[1] - P.rg), (float)(c[2] - P.rg)};
    const float hi[3] = {(float)(c[0] + P.rg), (float)(c[1] + P.rg), (float)(c[2] + P.rg)};
    int i0 = max(0, (int)floorf((lo[0] - P.ox) * P.inv_v)), i1 = min(P.nx - 1, (int)floorf((hi[0] - P.ox) * P.inv_v));
    int j0 = max(0, (int)floorf((lo[1] - P.oy) * P.inv_v)), j1 = min(P.ny - 1, (int)floorf((hi[1] - P.oy) * P.inv_v));
    int k0 = max(0, (int)floorf((lo[2] - P.oz) * P.inv_v)), k1 = min(P.nz - 1, (int)floorf((hi[2] - P.oz) * P.inv_v));
    const int nxr = i1 - i0 + 1, nyr = j1 - j0 + 1, nzr = k1 - k0 + 1;
    const int ncells = (nxr > 0 && nyr > 0 && nzr > 0) ? nxr * nyr * nzr : 0;
    const double rg2 = P.rg * P.rg;
    int count = 0;
    for (int base = 0; base < ncells; base += 32) {
        const int q = base + lane;
        unsigned mine[48];
        int nm = 0;
        bool spill = false;
        if (q < ncells) {
            const int ci = i0 + q % nxr, cj = j0 + (q / nxr) % nyr, ck = k0 + q / (nxr * nyr);
            const uint2 rg = __ldg(&P.cell[ci + P.nx * (cj + P.ny * ck)]);
            if (rg.y > rg.x) {
                for (unsigned k = rg.x; k < rg.y; ++k) {
                    const float4 A = __ldg(&P.rec[2 * k]);
                    const float4 B = __ldg(&P.rec[2 * k + 1]);
                    const unsigned id = __float_as_uint(B.w);
                    const float4 nv = __ldg(&P.sn[id]);
                    if (__float_as_int(nv.w) != label) continue;
                    // home cell of p: count each surfel once
                    const int hx = (int)floorf((A.x - P.ox) * P.inv_v), hy = (int)floorf((A.y - P.oy) * P.inv_v),
                              hz = (int)floorf((A.z - P.oz) * P.inv_v);
                    if (hx != ci || hy != cj || hz != ck) continue;
                    const double dx = (double)A.x - c[0], dy = (double)A.y - c[1], dz = (double)A.z - c[2];
                    if (dx * dx + dy * dy + dz * dz > rg2) continue;
                    if (nm < 48) mine[nm++] = id;
                    else spill = true;
                }
            }
        }
        // warp-ordered append (deterministic for a given grid)
        int pre = nm;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(0xffffffffu, pre, o);
            if (lane >= o) pre += t;
        }
        const int tot = __shfl_sync(0xffffffffu, pre, 31);
        const int start = count + pre - nm;
        for (int m = 0; m < nm; ++m)
            if (start + m < kCap) list[start + m] = mine[m];
        count += tot;
        if (__any_sync(0xffffffffu, spill)) V.over = true;
    }
    if (count > kCap) V.over = true;
    V.n = count < kCap ? count : kCap;
    __syncwarp();
}

// MLS (Eqs. 1-4) at x: sums over the cached candidates (or a direct scan on overflow)
__device__ bool mls(const RP& P, const Path& D, int k, const double x[3], const unsigned* list,
                    const Vtx& V, double pb[3], double nb[3], int lane) {
    const double inv2s2 = 1.0 / (2.0 * P.sigma * P.sigma);
    const double r2 = (4.0 * P.sigma) * (4.0 * P.sigma);
    double W = 0, Px = 0, Py = 0, Pz = 0, Nx = 0, Ny = 0, Nz = 0;
    const double* ns = D.nseed[k];
    for (int j = lane; j < V.n; j += 32) {
        const unsigned id = list[j];
        const float4 pa = __ldg(&P.sp[id]);
        const float4 na = __ldg(&P.sn[id]);
        const double p0 = pa.x, p1 = pa.y, p2 = pa.z;
        const double d0 = p0 - x[0], d1 = p1 - x[1], d2 = p2 - x[2];
        const double dd = (d0 * d0 + d1 * d1) + d2 * d2;
        if (dd > r2) continue;
        const double w = exp(-dd * inv2s2);
        const double n0 = na.x, n1 = na.y, n2 = na.z;
        const double sg = ((n0 * ns[0] + n1 * ns[1]) + n2 * ns[2]) < 0.0 ? -1.0 : 1.0;
        W += w;
        Px += w * p0;
        Py += w * p1;
        Pz += w * p2;
        Nx += w * sg * n0;
        Ny += w * sg * n1;
        Nz += w * sg * n2;
    }
    W = wsum(W);
    Px = wsum(Px);
    Py = wsum(Py);
    Pz = wsum(Pz);
    Nx = wsum(Nx);
    Ny = wsum(Ny);
    Nz = wsum(Nz);
    if (!(W > 0.0)) return false;
    pb[0] = Px / W;
    pb[1] = Py / W;
    pb[2] = Pz / W;
    nb[0] = Nx / W;
    nb[1] = Ny / W;
    nb[2] = Nz / W;
    const double l = sqrt(ddot(nb, nb));
    if (!(l > 0.0)) return false;
    nb[0] /= l;
    nb[1] /= l;
    nb[2] /= l;
    return true;
}

__device__ void basis(const double n[3], double u[3], double v[3]) {
    const double m0 = fabs(n[0]), m1 = fabs(n[1]), m2 = fabs(n[2]);
    int k = 0;
    if (m1 < m0) k = 1;
    if (m2 < (k == 0 ? m0 : m1)) k = 2;
    const double ax[3] = {k == 0 ? 1.0 : 0.0, k == 1 ? 1.0 : 0.0, k == 2 ? 1.0 : 0.0};
    u[0] = n[1] * ax[2] - n[2] * ax[1];
    u[1] = n[2] * ax[0] - n[0] * ax[2];
    u[2] = n[0] * ax[1] - n[1] * ax[0];
    const double l = sqrt(ddot(u, u));
    u[0] /= l;
    u[1] /= l;
    u[2] /= l;
    v[0] = n[1] * u[2] - n[2] * u[1];
    v[1] = n[2] * u[0] - n[0] * u[2];
    v[2] = n[0] * u[1] - n[1] * u[0];
}

__device__ __forceinline__ void vpoint(const RP& P, const Path& D, const double* z, int k, double x[3]) {
    if (k < 0) {
        x[0] = P.tx[0];
        x[1] = P.tx[1];
        x[2] = P.tx[2];
    } else if (k >= D.n) {
        x[0] = D.rxp[0];
        x[1] = D.rxp[1];
        x[2] = D.rxp[2];
    } else if (D.kind[k] == 0) {
        const double* zk = z + D.col[k];
        x[0] = zk[0];
        x[1] = zk[1];
        x[2] = zk[2];
    } else {
        const double t = z[D.col[k]];
        x[0] = D.ea[k][0] + t * D.ee[k][0];
        x[1] = D.ea[k][1] + t * D.ee[k][1];
        x[2] = D.ea[k][2] + t * D.ee[k][2];
    }
}

// MLS of vertex k at x, re-gathering when x left the safe ball of the gather centre
__device__ bool vertex_mls(const RP& P, const Path& D, int k, const double x[3], unsigned* list,
                           Vtx& V, double pb[3], double nb[3], int lane) {
    const double dx = x[0] - V.c[0], dy = x[1] - V.c[1], dz = x[2] - V.c[2];
    if (sqrt(dx * dx + dy * dy + dz * dz) > P.rg - P.rq || V.over) gather(P, D.label[k], x, list, V, lane);
    if (V.over) return false;  // neighbourhood larger than the scratch: reported as NO_SUPPORT
    return mls(P, D, k, x, list, V, pb, nb, lane);
}

// residual components of vertex k (writes r[col..]), given its MLS (reflection)
__device__ bool vertex_residual(const RP& P, const Path& D, const double* z, int k, const double* pb,
                                const double* nb, double* r) {
    double x[3], a[3], c[3];
    vpoint(P, D, z, k, x);
    vpoint(P, D, z, k - 1, a);
    vpoint(P, D, z, k + 1, c);
    const double va[3] = {x[0] - a[0], x[1] - a[1], x[2] - a[2]};
    const double vb[3] = {x[0] - c[0], x[1] - c[1], x[2] - c[2]};
    const double la = sqrt(ddot(va, va)), lb = sqrt(ddot(vb, vb));
    if (!(la > 0.0 && lb > 0.0)) return false;
    const double g[3] = {va[0] / la + vb[0] / lb, va[1] / la + vb[1] / lb, va[2] / la + vb[2] / lb};
    double* rk = r + D.col[k];
    if (D.kind[k] == 0) {
        double u[3], v[3];
        basis(nb, u, v);
        const double xp[3] = {x[0] - pb[0], x[1] - pb[1], x[2] - pb[2]};
        rk[0] = ddot(g, u);
        rk[1] = ddot(g, v);
        rk[2] = ddot(xp, nb);
    } else {
        rk[0] = ddot(g, D.ee[k]);
    }
    return true;
}

// full residual at z (MLS of every reflection vertex recomputed; cache updated)
__device__ bool residual_all(const RP& P, const Path& D, const double* z, double* r, unsigned* lists,
                             Vtx* V, double (*pb)[3], double (*nb)[3], int lane) {
    for (int k = 0; k < D.n; ++k) {
        if (D.kind[k] != 0) continue;
        double x[3];
        vpoint(P, D, z, k, x);
        if (!vertex_mls(P, D, k, x, lists + (size_t)k * kCap, V[k], pb[k], nb[k], lane)) return false;
    }
    for (int k = 0; k < D.n; ++k)
        if (!vertex_residual(P, D, z, k, pb[k], nb[k], r)) return false;
    return true;
}

__device__ double sq(const double* r, int m) {
    double s = 0;
    for (int i = 0; i < m; ++i) s += r[i] * r[i];
    return s;
}

// FP64 occlusion of segment x0 -> x1 (R25 d): warp walks the grid cells the segment crosses
__device__ bool occluded(const RP& P, const double x0[3], const double x1[3], const double* lam0,
                         int n0, const double* lam1, int n1, int lane) {
    const double dv[3] = {x1[0] - x0[0], x1[1] - x0[1], x1[2] - x0[2]};
    const double len = sqrt(ddot(dv, dv));
    const double d[3] = {dv[0] / len, dv[1] / len, dv[2] / len};
    const float of[3] = {(float)x0[0], (float)x0[1], (float)x0[2]};
    const float df[3] = {(float)d[0], (float)d[1], (float)d[2]};
    const float g0[3] = {P.ox, P.oy, P.oz};
    const int dims[3] = {P.nx, P.ny, P.nz};
    int ic[3];
    float tm[3], inv[3];
    for (int a = 0; a < 3; ++a) {
        ic[a] = min(dims[a] - 1, max(0, (int)floorf((of[a] - g0[a]) * P.inv_v)));
        inv[a] = 1.0f / df[a];
        tm[a] = df[a] != 0.0f ? ((g0[a] + (float)(ic[a] + (df[a] > 0.0f)) * P.v) - of[a]) * inv[a] : INFINITY;
    }
    const float tend = (float)len + P.pad;
    for (;;) {
        const uint2 rg = __ldg(&P.cell[ic[0] + P.nx * (ic[1] + P.ny * ic[2])]);
        bool hit = false;
        if (rg.y > rg.x) {
            for (unsigned k = rg.x + lane; k < rg.y; k += 32) {
                const float4 A = __ldg(&P.rec[2 * k]);
                const float4 B = __ldg(&P.rec[2 * k + 1]);
                const double p[3] = {A.x, A.y, A.z}, n[3] = {B.x, B.y, B.z};
                const double r = A.w;
                const double w[3] = {x0[0] - p[0], x0[1] - p[1], x0[2] - p[2]};
                const double f0 = ddot(w, n), dn = ddot(d, n);
                if (!(f0 * dn < 0.0)) continue;
                const double t = -f0 / dn;
                if (!(t < len)) continue;
                const double h[3] = {x0[0] + t * d[0] - p[0], x0[1] + t * d[1] - p[1], x0[2] + t * d[2] - p[2]};
                if (!(ddot(h, h) <= r * r)) continue;
                bool ex = false;
                if (fabs(f0) <= P.tau)
                    for (int q = 0; q < n0; ++q)
                        if (fabs(ddot(n, lam0 + 3 * q)) >= P.cos_ex) ex = true;
                const double w1[3] = {x1[0] - p[0], x1[1] - p[1], x1[2] - p[2]};
                const double f1 = ddot(w1, n);
                if (!ex && fabs(f1) <= P.tau)
                    for (int q = 0; q < n1; ++q)
                        if (fabs(ddot(n, lam1 + 3 * q)) >= P.cos_ex) ex = true;
                if (!ex) hit = true;
            }
        }
        if (__any_sync(0xffffffffu, hit)) return true;
        int a = 0;
        if (tm[1] < tm[a]) a = 1;
        if (tm[2] < tm[a]) a = 2;
        if (tm[a] > tend) return false;
        ic[a] += df[a] > 0.0f ? 1 : -1;
        if (ic[a] < 0 || ic[a] >= dims[a]) return false;
        tm[a] = ((g0[a] + (float)(ic[a] + (df[a] > 0.0f)) * P.v) - of[a]) * inv[a];
    }
}

__device__ bool supported(const RP& P, int32_t label, const double x[3], const unsigned* list,
                          const Vtx& V, int lane) {
    bool s = false;
    for (int j = lane; j < V.n; j += 32) {
        const unsigned id = list[j];
        const float4 pa = __ldg(&P.sp[id]);
        const float4 na = __ldg(&P.sn[id]);
        const double w[3] = {x[0] - pa.x, x[1] - pa.y, x[2] - pa.z};
        const double n[3] = {na.x, na.y, na.z};
        const double r = pa.w;
        if (fabs(ddot(w, n)) <= P.tau && ddot(w, w) <= r * r + P.tau * P.tau) s = true;
    }
    return __any_sync(0xffffffffu, s);
}

__global__ void __launch_bounds__(32 * kWarps) k_refine(RP P) {
    __shared__ WarpSmem smem[kWarps];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpSmem& S = smem[wid];
    const int slot = blockIdx.x * kWarps + wid;
    unsigned* lists = P.cand + (size_t)slot * NRT_MAX_INT * kCap;
    const int64_t n_mine = P.n_in > P.rank ? (P.n_in - P.rank + P.world - 1) / P.world : 0;
    for (;;) {
        unsigned long long q = 0;
        if (lane == 0) q = atomicAdd(P.work, 1ull);
        q = __shfl_sync(0xffffffffu, q, 0);
        if ((int64_t)q >= n_mine) break;
        const int64_t pi = P.rank + (int64_t)q * P.world;
        const nrt_coarse_rec& c = P.in[pi];
        // ---- set up the unknowns at the coarse seed
        Path D;
        D.n = c.n_int;
        int m = 0;
        for (int a = 0; a < 3; ++a) D.rxp[a] = (double)P.rx[3 * (size_t)c.rx + a];
        for (int k = 0; k < D.n; ++k) {
            D.kind[k] = (c.kinds >> k) & 1u;
            D.label[k] = c.label[k];
            D.prim[k] = c.prim[k];
            D.col[k] = m;
            if (D.kind[k] == 0) {
                const float4 nv = __ldg(&P.sn[c.prim[k]]);
                D.nseed[k][0] = nv.x;
                D.nseed[k][1] = nv.y;
                D.nseed[k][2] = nv.z;
                if (lane == 0)
                    for (int a = 0; a < 3; ++a) S.z[m + a] = c.v[k][a];
                m += 3;
            } else {
                const DevEdge& E = P.edges[c.prim[k]];
                for (int a = 0; a < 3; ++a) D.ea[k][a] = E.a[a];
                m += 1;
            }
        }
        D.dim = m;
        // diffraction: unit direction and length in FP64 from the f32 endpoints a, b
        for (int k = 0; k < D.n; ++k) {
            if (D.kind[k] == 0) continue;
            const DevEdge& E = P.edges[c.prim[k]];
            const double ev[3] = {(double)E.b_[0] - E.a[0], (double)E.b_[1] - E.a[1], (double)E.b_[2] - E.a[2]};
            const double l = sqrt(ddot(ev, ev));
            for (int a = 0; a < 3; ++a) D.ee[k][a] = ev[a] / l;
            D.elen[k] = l;
            const double w[3] = {c.v[k][0] - D.ea[k][0], c.v[k][1] - D.ea[k][1], c.v[k][2] - D.ea[k][2]};
            if (lane == 0) S.z[D.col[k]] = ddot(w, D.ee[k]);
        }
        __syncwarp();
        Vtx V[NRT_MAX_INT];
        for (int k = 0; k < D.n; ++k) {
            if (D.kind[k] != 0) continue;
            const double x[3] = {S.z[D.col[k]], S.z[D.col[k] + 1], S.z[D.col[k] + 2]};
            gather(P, D.label[k], x, lists + (size_t)k * kCap, V[k], lane);
        }
        int status = NRT_REF_NO_CONVERGE, it = 0;
        double pbk[3], nbk[3];
        if (m == 0) status = NRT_REF_OK;
        else if (!residual_all(P, D, S.z, S.r, lists, V, S.pb, S.nb, lane)) status = NRT_REF_NO_SUPPORT;
        else {
            for (it = 1; it <= P.max_iter; ++it) {
                // ---- Jacobian by central differences; only the perturbed vertex's MLS moves
                bool ok = true;
                for (int j = 0; j < m && ok; ++j) {
                    int k = 0;
                    while (k + 1 < D.n && D.col[k + 1] <= j) ++k;
                    for (int sgn = 0; sgn < 2 && ok; ++sgn) {
                        double* rr = sgn == 0 ? S.rp : S.rm;
                        __syncwarp();
                        const double zj = S.z[j];
                        double zz[kMaxDim];
                        for (int i = 0; i < m; ++i) zz[i] = S.z[i];
                        zz[j] = sgn == 0 ? zj + kH : zj - kH;
                        if (D.kind[k] == 0) {
                            double x[3];
                            vpoint(P, D, zz, k, x);
                            ok = vertex_mls(P, D, k, x, lists + (size_t)k * kCap, V[k], pbk, nbk, lane);
                        }
                        for (int q2 = 0; q2 < D.n && ok; ++q2) {
                            const bool mine = q2 == k && D.kind[k] == 0;
                            ok = vertex_residual(P, D, zz, q2, mine ? pbk : S.pb[q2], mine ? nbk : S.nb[q2], rr);
                        }
                        (void)rr;
                    }
                    if (ok && lane == 0)
                        for (int i = 0; i < m; ++i) S.J[i * m + j] = (S.rp[i] - S.rm[i]) / (2.0 * kH);
                    __syncwarp();
                }
                if (!ok) {
                    status = NRT_REF_NO_SUPPORT;
                    break;
                }
                // ---- normal equations + Cholesky (lane 0; m <= 24)
                int solved = 1;
                double dmax = 0;
                if (lane == 0) {
                    double tr = 0;
                    for (int i = 0; i < m; ++i) {
                        for (int j = 0; j < m; ++j) {
                            double s = 0;
                            for (int q2 = 0; q2 < m; ++q2) s += S.J[q2 * m + i] * S.J[q2 * m + j];
                            S.A[i * m + j] = s;
                        }
                        tr += S.A[i * m + i];
                        double s = 0;
                        for (int q2 = 0; q2 < m; ++q2) s += S.J[q2 * m + i] * S.r[q2];
                        S.b[i] = -s;
                    }
                    const double lam = 1e-12 * tr / m;
                    for (int i = 0; i < m; ++i) S.A[i * m + i] += lam;
                    for (int j = 0; j < m && solved; ++j) {
                        double d = S.A[j * m + j];
                        for (int k = 0; k < j; ++k) d -= S.A[j * m + k] * S.A[j * m + k];
                        if (!(d > 0.0)) {
                            solved = 0;
                            break;
                        }
                        d = sqrt(d);
                        S.A[j * m + j] = d;
                        for (int i = j + 1; i < m; ++i) {
                            double s = S.A[i * m + j];
                            for (int k = 0; k < j; ++k) s -= S.A[i * m + k] * S.A[j * m + k];
                            S.A[i * m + j] = s / d;
                        }
                    }
                    if (solved) {
                        for (int i = 0; i < m; ++i) {
                            double s = S.b[i];
                            for (int k = 0; k < i; ++k) s -= S.A[i * m + k] * S.b[k];
                            S.b[i] = s / S.A[i * m + i];
                        }
                        for (int i = m - 1; i >= 0; --i) {
                            double s = S.b[i];
                            for (int k = i + 1; k < m; ++k) s -= S.A[k * m + i] * S.b[k];
                            S.b[i] = s / S.A[i * m + i];
                        }
                        for (int i = 0; i < m; ++i) dmax = fmax(dmax, fabs(S.b[i]));
                    }
                }
                solved = __shfl_sync(0xffffffffu, solved, 0);
                dmax = __shfl_sync(0xffffffffu, dmax, 0);
                __syncwarp();
                if (!solved) {
                    status = NRT_REF_DEGENERATE;
                    break;
                }
                if (dmax < P.tol) {  // converged: take the (tiny) full step
                    if (lane == 0)
                        for (int i = 0; i < m; ++i) S.zt[i] = S.z[i] + S.b[i];
                    __syncwarp();
                    double pbs[NRT_MAX_INT][3], nbs[NRT_MAX_INT][3];
                    for (int k = 0; k < D.n; ++k)
                        for (int a = 0; a < 3; ++a) {
                            pbs[k][a] = S.pb[k][a];
                            nbs[k][a] = S.nb[k][a];
                        }
                    __syncwarp();
                    if (residual_all(P, D, S.zt, S.rp, lists, V, pbs, nbs, lane)) {
                        __syncwarp();
                        if (lane == 0)
                            for (int i = 0; i < m; ++i) {
                                S.z[i] = S.zt[i];
                                S.r[i] = S.rp[i];
                            }
                    }
                    status = NRT_REF_OK;
                    __syncwarp();
                    break;
                }
                const double f0 = sq(S.r, m);
                double gam = 1.0;
                bool acc = false;
                while (gam > 1e-12) {
                    if (lane == 0)
                        for (int i = 0; i < m; ++i) S.zt[i] = S.z[i] + gam * S.b[i];
                    __syncwarp();
                    double pbs[NRT_MAX_INT][3], nbs[NRT_MAX_INT][3];
                    const bool okr = residual_all(P, D, S.zt, S.rp, lists, V, pbs, nbs, lane);
                    __syncwarp();
                    if (okr && sq(S.rp, m) <= (1.0 - 2.0 * P.alpha * gam) * f0) {
                        if (lane == 0)
                            for (int i = 0; i < m; ++i) {
                                S.z[i] = S.zt[i];
                                S.r[i] = S.rp[i];
                            }
                        for (int k = 0; k < D.n; ++k)
                            for (int a = 0; a < 3; ++a) {
                                S.pb[k][a] = pbs[k][a];
                                S.nb[k][a] = nbs[k][a];
                            }
                        acc = true;
                        __syncwarp();
                        break;
                    }
                    gam *= P.beta;
                }
                if (!acc) {
                    status = NRT_REF_NO_CONVERGE;
                    break;
                }
            }
            if (it > P.max_iter) it = P.max_iter;
        }
        __syncwarp();
        // ---- final residual, gradient norm, validity
        double I[NRT_MAX_INT + 2][3];
        for (int k = -1; k <= D.n; ++k) vpoint(P, D, S.z, k, I[k + 1]);
        double gsq = 0, rmax = 0;
        if (status == NRT_REF_OK && m > 0) {
            double pbs[NRT_MAX_INT][3], nbs[NRT_MAX_INT][3];
            __syncwarp();
            if (!residual_all(P, D, S.z, S.rp, lists, V, pbs, nbs, lane)) status = NRT_REF_NO_SUPPORT;
            else {
                for (int k = 0; k < D.n; ++k)
                    for (int a = 0; a < 3; ++a) {
                        S.nb[k][a] = nbs[k][a];
                    }
                for (int k = 0; k < D.n; ++k) {
                    const double* rk = S.rp + D.col[k];
                    gsq += D.kind[k] == 0 ? rk[0] * rk[0] + rk[1] * rk[1] : rk[0] * rk[0];
                }
                for (int i = 0; i < m; ++i) S.r[i] = S.rp[i];
            }
        }
        for (int i = 0; i < m; ++i) rmax = fmax(rmax, fabs(S.r[i]));
        if (status == NRT_REF_OK)
            for (int k = 0; k < D.n; ++k)
                if (D.kind[k] == 1) {
                    const double t = S.z[D.col[k]];
                    if (!(t >= 0.0 && t <= D.elen[k])) status = NRT_REF_OFF_EDGE;
                }
        if (status == NRT_REF_OK)
            for (int k = 0; k < D.n; ++k)
                if (D.kind[k] == 0) {
                    const double a[3] = {I[k][0] - I[k + 1][0], I[k][1] - I[k + 1][1], I[k][2] - I[k + 1][2]};
                    const double b[3] = {I[k + 2][0] - I[k + 1][0], I[k + 2][1] - I[k + 1][1], I[k + 2][2] - I[k + 1][2]};
                    const double sa = ddot(a, S.nb[k]), sb = ddot(b, S.nb[k]);
                    if (!((sa > 0 && sb > 0) || (sa < 0 && sb < 0))) status = NRT_REF_WRONG_SIDE;
                }
        if (status == NRT_REF_OK)
            for (int k = 0; k < D.n; ++k)
                if (D.kind[k] == 0 && status == NRT_REF_OK) {
                    // the support query may need a wider list than the GN ball: re-gather here
                    const double dx = I[k + 1][0] - V[k].c[0], dy = I[k + 1][1] - V[k].c[1], dz = I[k + 1][2] - V[k].c[2];
                    if (sqrt(dx * dx + dy * dy + dz * dz) > P.rg - P.rq || V[k].over)
                        gather(P, D.label[k], I[k + 1], lists + (size_t)k * kCap, V[k], lane);
                    if (V[k].over || !supported(P, D.label[k], I[k + 1], lists + (size_t)k * kCap, V[k], lane))
                        status = NRT_REF_NO_SUPPORT;
                }
        if (status == NRT_REF_OK) {
            for (int j = 0; j <= D.n && status == NRT_REF_OK; ++j) {
                double l0[6], l1[6];
                int n0 = 0, n1 = 0;
                if (j >= 1) {
                    const int k = j - 1;
                    if (D.kind[k] == 0) {
                        for (int a = 0; a < 3; ++a) l0[a] = S.nb[k][a];
                        n0 = 1;
                    } else {
                        const DevEdge& E = P.edges[D.prim[k]];
                        for (int a = 0; a < 3; ++a) {
                            l0[a] = E.n0[a];
                            l0[3 + a] = E.n1[a];
                        }
                        n0 = 2;
                    }
                }
                if (j + 1 <= D.n) {
                    const int k = j;
                    if (D.kind[k] == 0) {
                        for (int a = 0; a < 3; ++a) l1[a] = S.nb[k][a];
                        n1 = 1;
                    } else {
                        const DevEdge& E = P.edges[D.prim[k]];
                        for (int a = 0; a < 3; ++a) {
                            l1[a] = E.n0[a];
                            l1[3 + a] = E.n1[a];
                        }
                        n1 = 2;
                    }
                }
                if (occluded(P, I[j], I[j + 1], l0, n0, l1, n1, lane)) status = NRT_REF_OCCLUDED;
            }
        }
        // ---- output
        if (lane == 0 && (P.keep_invalid || status == NRT_REF_OK)) {
            nrt_refined_rec o;
            memset(&o, 0, sizeof(o));
            o.rx = c.rx;
            o.n_int = c.n_int;
            o.n_diff = c.n_diff;
            o.kinds = c.kinds;
            for (int k = 0; k < NRT_MAX_INT; ++k) {
                o.label[k] = c.label[k];
                o.prim[k] = c.prim[k];
            }
            o.ray_id = c.ray_id;
            double L = 0;
            for (int j = 0; j <= D.n; ++j) {
                const double s3[3] = {I[j + 1][0] - I[j][0], I[j + 1][1] - I[j][1], I[j + 1][2] - I[j][2]};
                L += sqrt(ddot(s3, s3));
            }
            o.L = L;
            o.delay = L / kC;
            for (int k = 0; k < D.n; ++k)
                for (int a = 0; a < 3; ++a) o.v[k][a] = I[k + 1][a];
            const double d0[3] = {I[1][0] - I[0][0], I[1][1] - I[0][1], I[1][2] - I[0][2]};
            const double dl[3] = {I[D.n][0] - I[D.n + 1][0], I[D.n][1] - I[D.n + 1][1], I[D.n][2] - I[D.n + 1][2]};
            const double l0 = sqrt(ddot(d0, d0)), ll = sqrt(ddot(dl, dl));
            o.aod_az = (float)(atan2(d0[1], d0[0]) * 180.0 / kPi);
            o.aod_el = (float)(asin(fmax(-1.0, fmin(1.0, d0[2] / l0))) * 180.0 / kPi);
            o.aoa_az = (float)(atan2(dl[1], dl[0]) * 180.0 / kPi);
            o.aoa_el = (float)(asin(fmax(-1.0, fmin(1.0, dl[2] / ll))) * 180.0 / kPi);
            for (int k = 0; k < D.n; ++k) {
                const double din[3] = {I[k + 1][0] - I[k][0], I[k + 1][1] - I[k][1], I[k + 1][2] - I[k][2]};
                const double l = sqrt(ddot(din, din));
                const double c2 = D.kind[k] == 0 ? fabs(ddot(din, S.nb[k])) / l : ddot(din, D.ee[k]) / l;
                o.inc[k] = (float)(acos(fmax(-1.0, fmin(1.0, c2))) * 180.0 / kPi);
            }
            o.status = status;
            o.iters = it;
            o.resid = m ? rmax : 0.0;
            o.gradsq = gsq;
            const unsigned long long at = P.keep_invalid ? (unsigned long long)q : atomicAdd(P.n_out, 1ull);
            P.out[at] = o;
        }
        __syncwarp();
    }
}

}  // namespace

nrt_status refine(nrt_scene s, nrt_paths coarse, const nrt_refine_desc* d, nrt_paths out,
                  cudaStream_t st) {
    const int64_t n = coarse->n;
    out->n = 0;
    RP P{};
    P.cell = s->cell;
    P.rec = s->rec;
    P.sp = s->sp;
    P.sn = s->sn;
    P.ox = s->org[0];
    P.oy = s->org[1];
    P.oz = s->org[2];
    P.v = s->v;
    P.inv_v = s->inv_v;
    P.pad = s->pad;
    P.nx = s->dims[0];
    P.ny = s->dims[1];
    P.nz = s->dims[2];
    P.edges = s->edges;
    P.in = (const nrt_coarse_rec*)coarse->d_rec;
    P.n_in = n;
    P.rank = d->rank;
    P.world = d->world;
    for (int a = 0; a < 3; ++a) P.tx[a] = coarse->tx[a];
    P.sigma = d->xi * d->r_s;
    P.tau = d->tau;
    {
        double sn_, cs;
        nrt_sincos(d->theta_ex_deg * (kPi / 180.0), &sn_, &cs);
        P.cos_ex = cs;
    }
    P.rq = fmax(4.0 * P.sigma, (double)s->r_max + d->tau);
    P.rg = P.rq + fmax(0.05, 2.0 * P.sigma);
    P.tol = d->tol_m;
    P.alpha = d->alpha;
    P.beta = d->beta;
    P.max_iter = d->max_iter;
    P.keep_invalid = d->keep_invalid;
    const int64_t n_mine = n > d->rank ? (n - d->rank + d->world - 1) / d->world : 0;
    float* d_rx = nullptr;
    const size_t nrx = coarse->rx.size();
    NRT_CUDA(cudaMallocAsync(&d_rx, (nrx ? nrx : 3) * sizeof(float), st));
    if (nrx) NRT_CUDA(cudaMemcpyAsync(d_rx, coarse->rx.data(), nrx * sizeof(float), cudaMemcpyHostToDevice, st));
    P.rx = d_rx;
    nrt_refined_rec* o = nullptr;
    NRT_CUDA(cudaMallocAsync(&o, (size_t)(n_mine > 0 ? n_mine : 1) * sizeof(nrt_refined_rec), st));
    unsigned long long* ctr = nullptr;
    NRT_CUDA(cudaMallocAsync(&ctr, 2 * sizeof(unsigned long long), st));
    NRT_CUDA(cudaMemsetAsync(ctr, 0, 2 * sizeof(unsigned long long), st));
    P.out = o;
    P.n_out = ctr;
    P.work = ctr + 1;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_refine, 32 * kWarps, 0);
    if (per_sm < 1) per_sm = 1;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s->device);
    int64_t blocks = (int64_t)sms * per_sm;
    const int64_t need = (n_mine + kWarps - 1) / kWarps;
    if (blocks > need) blocks = need;
    if (blocks < 1) blocks = 1;
    P.slots = (int)blocks * kWarps;
    NRT_CUDA(cudaMallocAsync(&P.cand, (size_t)P.slots * NRT_MAX_INT * kCap * sizeof(unsigned), st));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
    if (n_mine > 0) {
        k_refine<<<(unsigned)blocks, 32 * kWarps, 0, st>>>(P);
        ::nrt::count_launch();
    }
    cudaEventRecord(e1, st);
    NRT_CUDA(cudaGetLastError());
    unsigned long long n_ok = 0;
    NRT_CUDA(cudaMemcpyAsync(&n_ok, ctr, sizeof(n_ok), cudaMemcpyDeviceToHost, st));
    NRT_CUDA(cudaStreamSynchronize(st));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    out->info.ms_refine = ms;
    cudaFreeAsync(P.cand, st);
    cudaFreeAsync(d_rx, st);
    cudaFreeAsync(ctr, st);
    if (d->keep_invalid) {
        out->d_rec = o;
        out->n = n_mine;
    } else {
        // R28: shortest per key among the valid paths
        nrt_refined_rec* u = nullptr;
        NRT_CUDA(cudaMallocAsync(&u, (size_t)(n_ok > 0 ? n_ok : 1) * sizeof(nrt_refined_rec), st));
        int64_t m = 0;
        NRT_TRY(dedupe_refined(o, (int64_t)n_ok, u, &m, st));
        cudaFreeAsync(o, st);
        out->d_rec = u;
        out->n = m;
    }
    NRT_CUDA(cudaStreamSynchronize(st));
    out->info.n = out->n;
    out->info.n_raw = n_mine;
    return NRT_OK;
}

}  // namespace nrt
