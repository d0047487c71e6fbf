// refine.cu — A9-A10: batched path refinement (FP64), one thread block (NW warps) per path.
//
// The refined path is the root of the residual of DESIGN.md §5 (readings R18-R28):
//   reflection k: r_k = [g.u, g.v, f_sdf] with the MLS surface of Eqs. 1-4 over
//     the same-label surfels within 4 sigma (sigma = xi r_s), normals oriented by the
//     seed normal (Eq. 3 + R20), basis (u, v) of the MLS normal, g the Eq. 9-10 vector;
//   diffraction k: r_k = g.e (Eq. 11, I_k = a + t_k e, Eq. 8).
// reached by damped Gauss-Newton with a central-difference Jacobian (h = 1e-7), step
// -(J^T J + lam I)^-1 J^T r, Armijo backtracking (Eq. 12 form, R24), converged at |D|_inf <
// tol, stalled (NO_CONVERGE, R23b) once an accepted step |gamma D|_inf < tol.  Then validity
// (R25): on-edge, same side, support, FP64 visibility; delay = L/c (R26).
//
// B200 mapping.  Refinement is latency-bound (a few thousand small solves), so
// one block of NW warps works on one path and spreads the independent pieces of each GN
// iteration over its warps:
//   * the 2m perturbed residuals of the Jacobian (column j on warp j mod NW);
//   * the backtracking trials: warp w evaluates gamma = beta^(round*NW + w), and the block
//     accepts the first trial (in sequence order) that passes Armijo — exactly the step the
//     sequential loop would take;
//   * the MLS sums inside a warp: lanes split the candidates, butterfly-reduce 7 FP64 sums.
// Per reflection vertex the block gathers once (from the fine grid, home-cell dedupe, same
// label, within rg of a gather centre) the candidate surfels into SHARED memory; an MLS
// point farther than rg - rq from its centre falls back to a direct grid scan (same set).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "internal.cuh"

namespace nrt {

namespace {

#ifndef NRT_REFINE_WARPS
#define NRT_REFINE_WARPS 8
#endif
constexpr int NW = NRT_REFINE_WARPS;      // warps per path
#ifndef NRT_MLS_ILP
#define NRT_MLS_ILP 1
#endif
constexpr int kMaxDim = 3 * NRT_MAX_INT;
constexpr int kCapS = 768;                // shared-memory candidates per reflection vertex
constexpr double kC = 299792458.0;
constexpr double kH = 1e-7;               // central-difference step (m)

struct RP {
    const uint2* cell;
    const float4* rec;
    const float4* sp;  // (p, r)
    const float4* sn;  // (n, label bits)
    float ox, oy, oz, v, inv_v, pad;
    int nx, ny, nz;
    const uint2* hcell;   // home grid (each surfel once)
    const float4* hrec;
    float inv_hv;
    int hx, hy, hz;
    const DevEdge* edges;
    const nrt_coarse_rec* in;
    int64_t n_in;
    int rank, world;
    double tx[3];
    const float* rx;
    double sigma, rq, rg, tau, cos_ex, tol, alpha, beta;
    int max_iter, nv_max;  // nv_max: reflection vertices with shared candidate storage
    nrt_refined_rec* out;
    unsigned long long* n_out;
    int keep_invalid;
    unsigned long long* work;
    long long* cycles;  // optional per-path latency (NRT_REFINE_TIMING diagnostics)
};

struct Path {
    int n, dim;
    int kind[NRT_MAX_INT];
    int32_t label[NRT_MAX_INT];
    uint32_t prim[NRT_MAX_INT];
    int col[NRT_MAX_INT];
    int slot[NRT_MAX_INT];  // shared candidate slot of a reflection vertex (-1: none)
    double nseed[NRT_MAX_INT][3];
    double ea[NRT_MAX_INT][3], ee[NRT_MAX_INT][3], elen[NRT_MAX_INT];
    double rxp[3];
};

struct Vtx {
    double c[3];
    int n;       // candidates in shared memory
    int direct;  // 1: no usable list (overflow) -> direct scans
};

struct Trial {  // one warp's residual evaluation result
    double r[kMaxDim];
    double pb[NRT_MAX_INT][3], nb[NRT_MAX_INT][3];
    double f;
    int ok;
};

struct Smem {
    Path D;  // the path being refined (one copy per block)
    double J[kMaxDim * kMaxDim];
    union {
        struct {
            double A[kMaxDim * kMaxDim];  // normal equations (solve phase)
            Trial tr[NW];                 // residual evaluations (line search, checks)
        };
        double Rpm[2 * kMaxDim * kMaxDim];  // perturbed residuals, row 2j (+h), 2j+1 (-h)
    };
    double z[kMaxDim], r[kMaxDim], b[kMaxDim];
    double pb[NRT_MAX_INT][3], nb[NRT_MAX_INT][3];
    double zw[NW][kMaxDim];  // per-warp trial point
    double I[NRT_MAX_INT + 2][3];
    Vtx V[NRT_MAX_INT];
    int flag[NW];
    int okv[NRT_MAX_INT];
    int vstat;
    int vflag[2 * NRT_MAX_INT + 1];  // validity: support failures [0, n), occlusions [n, 2n+1)
    double nbv[NRT_MAX_INT][3];      // final MLS normals (validity)
    double gsq, rmax;
    double dval;
    unsigned long long q;
};
static_assert(sizeof(double) * kMaxDim * kMaxDim + sizeof(Trial) * NW >=
                  sizeof(double) * 2 * kMaxDim * kMaxDim,
              "Rpm must not spill past A + tr");

__device__ __forceinline__ double ddot(const double a[3], const double b[3]) {
    return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
}
__device__ __forceinline__ double wsum(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// candidate storage of slot s: p (xyz) and n (xyz) as floats, kCapS entries
__device__ __forceinline__ float* cand_ptr(float* cand, int s) { return cand + (size_t)s * kCapS * 6; }

typedef cub::BlockScan<int, 32 * NW> BlockScanT;

__device__ unsigned long long g_dbg[16];  // diagnostics (NRT_REFINE_TIMING): MLS list/direct, LS rounds, gathers

// home-grid cell range of the axis-aligned box [c - R, c + R] (clamped)
struct Box {
    int i0, i1, j0, j1, k0, k1;
};
__device__ __forceinline__ Box home_box(const RP& P, const double c[3], double R) {
    Box b;
    b.i0 = max(0, (int)floorf(((float)(c[0] - R) - P.ox) * P.inv_hv));
    b.i1 = min(P.hx - 1, (int)floorf(((float)(c[0] + R) - P.ox) * P.inv_hv));
    b.j0 = max(0, (int)floorf(((float)(c[1] - R) - P.oy) * P.inv_hv));
    b.j1 = min(P.hy - 1, (int)floorf(((float)(c[1] + R) - P.oy) * P.inv_hv));
    b.k0 = max(0, (int)floorf(((float)(c[2] - R) - P.oz) * P.inv_hv));
    b.k1 = min(P.hz - 1, (int)floorf(((float)(c[2] + R) - P.oz) * P.inv_hv));
    return b;
}

// ---- one warp visits every surfel of the home cells of box B: f(home record index) is called
// by the lane that owns the record (32 cell headers per round trip, warp prefix sum of the
// counts, lanes stride over the flattened records).
template <class F>
__device__ __forceinline__ void scan_box(const RP& P, const Box& B, int lane, F&& f) {
    const int nxr = B.i1 - B.i0 + 1, nyr = B.j1 - B.j0 + 1, nzr = B.k1 - B.k0 + 1;
    const int ncells = (nxr > 0 && nyr > 0 && nzr > 0) ? nxr * nyr * nzr : 0;
    for (int base = 0; base < ncells; base += 32) {
        const int q0 = base + lane;
        unsigned s0 = 0, cnt = 0;
        if (q0 < ncells) {
            const int ci = B.i0 + q0 % nxr, cj = B.j0 + (q0 / nxr) % nyr, ck = B.k0 + q0 / (nxr * nyr);
            const uint2 rg = __ldg(&P.hcell[ci + P.hx * (cj + P.hy * ck)]);
            if (rg.y > rg.x) {
                s0 = rg.x;
                cnt = rg.y - rg.x;
            }
        }
        unsigned incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const unsigned total = __shfl_sync(0xffffffffu, incl, 31);
        for (unsigned g0 = 0; g0 < total; g0 += 32) {  // warp-uniform trip count
            const unsigned g = g0 + lane;
            int lo = 0;  // owner lane: first lane whose inclusive prefix exceeds g
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const unsigned pm = __shfl_sync(0xffffffffu, incl, lo + step - 1);
                if (pm <= g) lo += step;
            }
            const unsigned excl = __shfl_sync(0xffffffffu, incl - cnt, lo);
            const unsigned st = __shfl_sync(0xffffffffu, s0, lo);
            if (g < total) f(st + (g - excl));
        }
    }
}

// ---- block-cooperative gather of the label's surfels within rg of c from the home grid.
// Deterministic order: home cells in linear order, each round of blockDim cells compacted by a
// block prefix sum (so the MLS sums, hence the results, are bitwise reproducible).
__device__ void gather(const RP& P, int32_t label, const double c[3], float* list, Vtx& V,
                       int* counter, typename BlockScanT::TempStorage& scan) {
    const int tid = threadIdx.x;
    if (tid == 0) {
        V.c[0] = c[0];
        V.c[1] = c[1];
        V.c[2] = c[2];
        *counter = 0;
        if (P.cycles) atomicAdd(&g_dbg[3], 1ull);
    }
    __syncthreads();
    const Box B = home_box(P, c, P.rg);
    const int nxr = B.i1 - B.i0 + 1, nyr = B.j1 - B.j0 + 1, nzr = B.k1 - B.k0 + 1;
    const int ncells = (nxr > 0 && nyr > 0 && nzr > 0) ? nxr * nyr * nzr : 0;
    const double rg2 = P.rg * P.rg;
    auto match = [&](unsigned k, float4& A, float4& nv) {
        A = __ldg(&P.hrec[2 * k]);
        const double dx = (double)A.x - c[0], dy = (double)A.y - c[1], dz = (double)A.z - c[2];
        if (dx * dx + dy * dy + dz * dz > rg2) return false;
        nv = __ldg(&P.hrec[2 * k + 1]);
        return __float_as_int(nv.w) == label;
    };
    for (int base = 0; base < ncells; base += blockDim.x) {
        const int q = base + tid;
        uint2 rg = make_uint2(0, 0);
        int cnt = 0;
        if (q < ncells) {
            const int ci = B.i0 + q % nxr, cj = B.j0 + (q / nxr) % nyr, ck = B.k0 + q / (nxr * nyr);
            rg = __ldg(&P.hcell[ci + P.hx * (cj + P.hy * ck)]);
            for (unsigned k = rg.x; k < rg.y; ++k) {
                float4 A, nv;
                cnt += match(k, A, nv);
            }
        }
        int off = 0, tot = 0;
        BlockScanT(scan).ExclusiveSum(cnt, off, tot);
        const int start = *counter;
        if (cnt)
            for (unsigned k = rg.x, w = 0; k < rg.y; ++k) {
                float4 A, nv;
                if (!match(k, A, nv)) continue;
                const int at = start + off + (int)w++;
                if (at < kCapS) {
                    float* e = list + 6 * at;
                    e[0] = A.x;
                    e[1] = A.y;
                    e[2] = A.z;
                    e[3] = nv.x;
                    e[4] = nv.y;
                    e[5] = nv.z;
                }
            }
        __syncthreads();
        if (tid == 0) *counter = start + tot;
        __syncthreads();
    }
    if (tid == 0) {
        V.direct = *counter > kCapS;
        V.n = V.direct ? 0 : *counter;
    }
    __syncthreads();
}

// ---- MLS (Eqs. 1-4) at x, one warp.  From the shared list when x lies in the safe ball of
// the gather centre, else by a direct scan of the home grid (same set, another order).
__device__ bool mls(const RP& P, const Path& D, int k, const double x[3], const float* list,
                    const Vtx& V, double pb[3], double nb[3], int lane) {
    const double inv2s2 = 1.0 / (2.0 * P.sigma * P.sigma);
    const double r2 = (4.0 * P.sigma) * (4.0 * P.sigma);
    const double* ns = D.nseed[k];
    double W = 0, Px = 0, Py = 0, Pz = 0, Nx = 0, Ny = 0, Nz = 0;
    const double dxc = x[0] - V.c[0], dyc = x[1] - V.c[1], dzc = x[2] - V.c[2];
    const bool use_list = !V.direct && sqrt(dxc * dxc + dyc * dyc + dzc * dzc) <= P.rg - P.rq;
    if (P.cycles && lane == 0) atomicAdd(&g_dbg[use_list ? 0 : 1], 1ull);
    const long long t_mls0 = P.cycles ? clock64() : 0;
    auto acc = [&](double p0, double p1, double p2, double n0, double n1, double n2) {
        const double d0 = p0 - x[0], d1 = p1 - x[1], d2 = p2 - x[2];
        const double dd = (d0 * d0 + d1 * d1) + d2 * d2;
        if (dd > r2) return;
        const double w = exp(-dd * inv2s2);
        const double sg = ((n0 * ns[0] + n1 * ns[1]) + n2 * ns[2]) < 0.0 ? -1.0 : 1.0;
        W += w;
        Px += w * p0;
        Py += w * p1;
        Pz += w * p2;
        Nx += w * sg * n0;
        Ny += w * sg * n1;
        Nz += w * sg * n2;
    };
    if (use_list) {
        // NRT_MLS_ILP candidates per lane and round (1 measured fastest: FP64 issue, not exp
        // latency, bounds the loop); each lane adds its candidates j = lane, lane + 32, ... in
        // that order, and a candidate outside 4 sigma adds w = 0 (every sum bitwise unchanged)
        const int n = V.n;
        for (int j0 = lane; j0 < n; j0 += 32 * NRT_MLS_ILP) {
            double wv[NRT_MLS_ILP], sgv[NRT_MLS_ILP];
            float e[NRT_MLS_ILP][6];
#pragma unroll
            for (int u = 0; u < NRT_MLS_ILP; ++u) {
                const int j = j0 + 32 * u;
                for (int a = 0; a < 6; ++a) e[u][a] = j < n ? list[6 * j + a] : 0.0f;
                const double d0 = (double)e[u][0] - x[0], d1 = (double)e[u][1] - x[1], d2 = (double)e[u][2] - x[2];
                const double dd = (d0 * d0 + d1 * d1) + d2 * d2;
                const double w = exp(-dd * inv2s2);
                wv[u] = (j < n && dd <= r2) ? w : 0.0;
                sgv[u] = (((double)e[u][3] * ns[0] + (double)e[u][4] * ns[1]) + (double)e[u][5] * ns[2]) < 0.0 ? -1.0 : 1.0;
            }
#pragma unroll
            for (int u = 0; u < NRT_MLS_ILP; ++u) {
                const double w = wv[u], sg = sgv[u];
                W += w;
                Px += w * (double)e[u][0];
                Py += w * (double)e[u][1];
                Pz += w * (double)e[u][2];
                Nx += w * sg * (double)e[u][3];
                Ny += w * sg * (double)e[u][4];
                Nz += w * sg * (double)e[u][5];
            }
        }
    } else {
        const int32_t label = D.label[k];
        scan_box(P, home_box(P, x, 4.0 * P.sigma), lane, [&](unsigned q) {
            const float4 A = __ldg(&P.hrec[2 * q]);
            const double d0 = (double)A.x - x[0], d1 = (double)A.y - x[1], d2 = (double)A.z - x[2];
            if ((d0 * d0 + d1 * d1) + d2 * d2 > r2) return;
            const float4 nv = __ldg(&P.hrec[2 * q + 1]);
            if (__float_as_int(nv.w) != label) return;
            acc(A.x, A.y, A.z, nv.x, nv.y, nv.z);
        });
    }
    W = wsum(W);
    if (P.cycles && lane == 0) atomicAdd(&g_dbg[use_list ? 4 : 5], (unsigned long long)(clock64() - t_mls0));
    if (P.cycles && lane == 0 && !use_list && !(W > 0.0)) {
        atomicAdd(&g_dbg[12], 1ull);
        atomicAdd(&g_dbg[13], (unsigned long long)(clock64() - t_mls0));
    }
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

// one warp: full residual at z into T (MLS of every reflection vertex recomputed)
__device__ void residual_all(const RP& P, const Path& D, const double* z, const float* cand,
                             const Vtx* V, Trial& T, int lane) {
    bool ok = true;
    double pb[3], nb[3];
    for (int k = 0; k < D.n && ok; ++k) {
        if (D.kind[k] != 0) continue;
        double x[3];
        vpoint(P, D, z, k, x);
        ok = mls(P, D, k, x, cand_ptr(const_cast<float*>(cand), D.slot[k]), V[D.slot[k]], pb, nb, lane);
        if (ok && lane == 0)
            for (int a = 0; a < 3; ++a) {
                T.pb[k][a] = pb[a];
                T.nb[k][a] = nb[a];
            }
    }
    __syncwarp();
    // vertex residuals in parallel (lane k -> vertex k), then |r|^2 in index order on lane 0
    bool okv = true;
    if (ok && lane < D.n) okv = vertex_residual(P, D, z, lane, T.pb[lane], T.nb[lane], T.r);
    ok = ok && __all_sync(0xffffffffu, okv);
    __syncwarp();
    if (ok && lane == 0) {
        double f = 0;
        for (int i = 0; i < D.dim; ++i) f += T.r[i] * T.r[i];
        T.f = f;
    }
    if (lane == 0) T.ok = ok;
    __syncwarp();
}

// whole block: the same residual as residual_all, with the MLS of reflection vertex k on warp
// (k mod NW) — every MLS sum is formed exactly as in residual_all (one warp, same lanes, same
// order), so T is bitwise the same; the vertex residuals then run on warp 0.  Ends synced.
__device__ void residual_coop(const RP& P, const Path& D, const double* z, const float* cand,
                              const Vtx* V, Trial& T, int* okv_s, int wid, int lane) {
    for (int k = wid; k < D.n; k += NW) {
        int ok = 1;
        if (D.kind[k] == 0) {
            double x[3], pb[3], nb[3];
            vpoint(P, D, z, k, x);
            ok = mls(P, D, k, x, cand_ptr(const_cast<float*>(cand), D.slot[k]), V[D.slot[k]], pb, nb, lane);
            if (ok && lane == 0)
                for (int a = 0; a < 3; ++a) {
                    T.pb[k][a] = pb[a];
                    T.nb[k][a] = nb[a];
                }
        }
        if (lane == 0) okv_s[k] = ok;
    }
    __syncthreads();
    if (wid == 0) {
        bool ok = true;
        for (int k = 0; k < D.n; ++k) ok = ok && okv_s[k];
        bool okv = true;
        if (ok && lane < D.n) okv = vertex_residual(P, D, z, lane, T.pb[lane], T.nb[lane], T.r);
        ok = ok && __all_sync(0xffffffffu, okv);
        __syncwarp();
        if (ok && lane == 0) {
            double f = 0;
            for (int i = 0; i < D.dim; ++i) f += T.r[i] * T.r[i];
            T.f = f;
        }
        if (lane == 0) T.ok = ok;
    }
    __syncthreads();
}

// FP64 occlusion of segment x0 -> x1 (R25 d), one warp.  The segment's t-range [0, len + pad]
// is cut into 32 equal pieces and lane j walks the grid cells of piece j by 3D-DDA (so the
// dependent header loads form 32 short chains instead of one long one); each round, every lane
// stops at its next non-empty cell and the warp tests the union of those cells' records
// together (flattened over the lanes, consecutive lanes on consecutive records).  The pieces'
// cells cover the cells the whole-segment walk visits (a piece starts in the cell holding its
// first point; boundary rounding is covered by the registration pad), and each
// record test is the exact per-record predicate, so the any-hit answer is the same.
__device__ bool occluded(const RP& P, const double x0[3], const double x1[3], const double* lam0,
                         int n0, const double* lam1, int n1, int lane) {
    const double dv[3] = {x1[0] - x0[0], x1[1] - x0[1], x1[2] - x0[2]};
    const double len = sqrt(ddot(dv, dv));
    const double d[3] = {dv[0] / len, dv[1] / len, dv[2] / len};
    const float of[3] = {(float)x0[0], (float)x0[1], (float)x0[2]};
    const float df[3] = {(float)d[0], (float)d[1], (float)d[2]};
    const float g0[3] = {P.ox, P.oy, P.oz};
    const int dims[3] = {P.nx, P.ny, P.nz};
    const float tend = (float)len + P.pad;
    const float piece = tend * (1.0f / 32.0f);
    const float ts = (float)lane * piece, te = lane == 31 ? tend : (float)(lane + 1) * piece;
    int ic[3];
    float tm[3], inv[3];
    for (int a = 0; a < 3; ++a) {
        const float pa = of[a] + ts * df[a];
        ic[a] = min(dims[a] - 1, max(0, (int)floorf((pa - g0[a]) * P.inv_v)));
        inv[a] = 1.0f / df[a];
        tm[a] = df[a] != 0.0f ? ((g0[a] + (float)(ic[a] + (df[a] > 0.0f)) * P.v) - of[a]) * inv[a] : INFINITY;
    }
    bool walking = true;
    for (;;) {
        // advance this lane to its next non-empty cell (the cell it stands in first)
        uint2 rg = make_uint2(0, 0);
        while (walking) {
            rg = __ldg(&P.cell[ic[0] + P.nx * (ic[1] + P.ny * ic[2])]);
            if (rg.y > rg.x) break;
            int a = 0;
            if (tm[1] < tm[a]) a = 1;
            if (tm[2] < tm[a]) a = 2;
            if (tm[a] > te) {
                walking = false;
                break;
            }
            ic[a] += df[a] > 0.0f ? 1 : -1;
            if (ic[a] < 0 || ic[a] >= dims[a]) {
                walking = false;
                break;
            }
            tm[a] = ((g0[a] + (float)(ic[a] + (df[a] > 0.0f)) * P.v) - of[a]) * inv[a];
        }
        const unsigned cnt = walking ? rg.y - rg.x : 0u;
        unsigned incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const unsigned total = __shfl_sync(0xffffffffu, incl, 31);
        if (total == 0) return false;  // no lane has a cell left
        bool hit = false;
        for (unsigned g0i = 0; g0i < total; g0i += 32) {
            const unsigned g = g0i + lane;
            int lo = 0;  // owner lane: first lane whose inclusive prefix exceeds g
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const unsigned pm = __shfl_sync(0xffffffffu, incl, lo + step - 1);
                if (pm <= g) lo += step;
            }
            const unsigned excl = __shfl_sync(0xffffffffu, incl - cnt, lo);
            const unsigned st = __shfl_sync(0xffffffffu, rg.x, lo);
            if (g < total) {
                const unsigned k = st + (g - excl);
                const float4 A = __ldg(&P.rec[2 * k]);
                const float4 B = __ldg(&P.rec[2 * k + 1]);
                const double p[3] = {A.x, A.y, A.z}, n[3] = {B.x, B.y, B.z};
                const double r = A.w;
                const double w[3] = {x0[0] - p[0], x0[1] - p[1], x0[2] - p[2]};
                const double f0 = ddot(w, n), dn = ddot(d, n);
                if (f0 * dn < 0.0) {
                    const double t = -f0 / dn;
                    const double h[3] = {x0[0] + t * d[0] - p[0], x0[1] + t * d[1] - p[1], x0[2] + t * d[2] - p[2]};
                    if (t < len && ddot(h, h) <= r * r) {
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
            }
        }
        if (__any_sync(0xffffffffu, hit)) return true;
        // step past the tested cell
        if (walking) {
            int a = 0;
            if (tm[1] < tm[a]) a = 1;
            if (tm[2] < tm[a]) a = 2;
            if (tm[a] > te) {
                walking = false;
            } else {
                ic[a] += df[a] > 0.0f ? 1 : -1;
                if (ic[a] < 0 || ic[a] >= dims[a]) walking = false;
                else tm[a] = ((g0[a] + (float)(ic[a] + (df[a] > 0.0f)) * P.v) - of[a]) * inv[a];
            }
        }
    }
}

// support (R25 c) over every same-label surfel near x (home grid, one warp)
__device__ bool supported(const RP& P, int32_t label, const double x[3], int lane) {
    bool s = false;
    const double lim2 = P.rq * P.rq;
    scan_box(P, home_box(P, x, P.rq), lane, [&](unsigned q) {
        if (s) return;
        const float4 A = __ldg(&P.hrec[2 * q]);
        const double w[3] = {x[0] - A.x, x[1] - A.y, x[2] - A.z};
        if (ddot(w, w) > lim2) return;
        const float4 nv = __ldg(&P.hrec[2 * q + 1]);
        if (__float_as_int(nv.w) != label) return;
        const double n[3] = {nv.x, nv.y, nv.z};
        const double r = A.w;
        if (fabs(ddot(w, n)) <= P.tau && ddot(w, w) <= r * r + P.tau * P.tau) s = true;
    });
    return __any_sync(0xffffffffu, s);
}

// Two register budgets of the same kernel: MINB = 3 resident blocks per SM (80 registers) is
// the throughput regime (many paths: C4/C5), MINB = 2 (128 registers, no spills) the latency
// regime (few paths, a tail of long GN runs: C2).  Measured: C2 refine -4.6 % with 2,
// C4 +12 % with 2.  refine() picks by the number of paths.
#ifndef NRT_LAT_MINB
#define NRT_LAT_MINB 2  // resident blocks per SM in the latency regime
#endif
template <int MINB>
__global__ void __launch_bounds__(32 * NW, MINB) k_refine(RP P) {
    extern __shared__ __align__(16) unsigned char dyn[];
    Smem& S = *reinterpret_cast<Smem*>(dyn);
    float* cand = reinterpret_cast<float*>(dyn + ((sizeof(Smem) + 15) & ~size_t(15)));
    __shared__ int counter;
    __shared__ typename BlockScanT::TempStorage scan;
    const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
    const int64_t n_mine = P.n_in > P.rank ? (P.n_in - P.rank + P.world - 1) / P.world : 0;
    for (;;) {
        const long long t_start = clock64();
        if (tid == 0) S.q = atomicAdd(P.work, 1ull);
        __syncthreads();
        const unsigned long long q = S.q;
        __syncthreads();
        if ((int64_t)q >= n_mine) break;
        // hand out the paths from the end of the key order (most interactions first) so the
        // expensive ones do not start last
        const int64_t jq = n_mine - 1 - (int64_t)q;
        const int64_t pi = P.rank + jq * P.world;
        const nrt_coarse_rec& c = P.in[pi];
        // ---- the path and its unknowns at the coarse seed (shared, built by thread 0)
        Path& D = S.D;
        if (tid == 0) {
            D.n = c.n_int;
            int m0 = 0, nslot = 0;
            for (int a = 0; a < 3; ++a) D.rxp[a] = (double)P.rx[3 * (size_t)c.rx + a];
            for (int k = 0; k < D.n; ++k) {
                D.kind[k] = (c.kinds >> k) & 1u;
                D.label[k] = c.label[k];
                D.prim[k] = c.prim[k];
                D.col[k] = m0;
                D.slot[k] = -1;
                if (D.kind[k] == 0) {
                    const float4 nv = __ldg(&P.sn[c.prim[k]]);
                    D.nseed[k][0] = nv.x;
                    D.nseed[k][1] = nv.y;
                    D.nseed[k][2] = nv.z;
                    D.slot[k] = nslot++;
                    m0 += 3;
                } else {
                    const DevEdge& E = P.edges[c.prim[k]];
                    const double ev[3] = {(double)E.b_[0] - E.a[0], (double)E.b_[1] - E.a[1], (double)E.b_[2] - E.a[2]};
                    const double l = sqrt(ddot(ev, ev));
                    for (int a = 0; a < 3; ++a) {
                        D.ea[k][a] = E.a[a];
                        D.ee[k][a] = ev[a] / l;
                    }
                    D.elen[k] = l;
                    m0 += 1;
                }
            }
            D.dim = m0;
        }
        __syncthreads();
        const int m = D.dim;
        // no state of the block's previous path survives (residual and MLS point/normal of a
        // path whose first residual is undefined are reported as zero)
        for (int e = tid; e < 3 * NRT_MAX_INT; e += blockDim.x) {
            (&S.pb[0][0])[e] = 0.0;
            (&S.nb[0][0])[e] = 0.0;
            S.r[e] = 0.0;
        }
        if (tid == 0)
            for (int k = 0; k < D.n; ++k) {
                if (D.kind[k] == 0) {
                    for (int a = 0; a < 3; ++a) S.z[D.col[k] + a] = c.v[k][a];
                } else {
                    const double w[3] = {c.v[k][0] - D.ea[k][0], c.v[k][1] - D.ea[k][1], c.v[k][2] - D.ea[k][2]};
                    S.z[D.col[k]] = ddot(w, D.ee[k]);
                }
            }
        __syncthreads();
        for (int k = 0; k < D.n; ++k) {
            if (D.kind[k] != 0) continue;
            const double x[3] = {S.z[D.col[k]], S.z[D.col[k] + 1], S.z[D.col[k] + 2]};
            if (D.slot[k] < P.nv_max) {
                gather(P, D.label[k], x, cand_ptr(cand, D.slot[k]), S.V[D.slot[k]], &counter, scan);
            } else if (tid == 0) {
                // no shared slot (more reflections than provisioned): direct scans
                S.V[D.slot[k]].direct = 1;
                S.V[D.slot[k]].n = 0;
            }
        }
        __syncthreads();
        int status = NRT_REF_NO_CONVERGE, it = 0;
        if (m == 0) {
            status = NRT_REF_OK;
        } else {
            if (wid == 0) residual_all(P, D, S.z, cand, S.V, S.tr[0], lane);
            __syncthreads();
            if (!S.tr[0].ok) status = NRT_REF_NO_SUPPORT;
            else {
                if (tid == 0) {
                    for (int i = 0; i < m; ++i) S.r[i] = S.tr[0].r[i];
                    for (int k = 0; k < D.n; ++k)
                        for (int a = 0; a < 3; ++a) {
                            S.pb[k][a] = S.tr[0].pb[k][a];
                            S.nb[k][a] = S.tr[0].nb[k][a];
                        }
                }
                __syncthreads();
                if (P.cycles && tid == 0) atomicAdd(&g_dbg[6], (unsigned long long)(clock64() - t_start));
                for (it = 1; it <= P.max_iter; ++it) {
                    long long tph = clock64();
                    auto phase = [&](int slot) {
                        if (P.cycles && tid == 0) {
                            const long long t = clock64();
                            atomicAdd(&g_dbg[slot], (unsigned long long)(t - tph));
                            tph = t;
                        }
                    };
                    // keep every vertex inside the safe ball of its candidate list: re-centre
                    // the gather when the iterate drifted more than half the margin
                    for (int k = 0; k < D.n; ++k) {
                        if (D.kind[k] != 0 || D.slot[k] >= P.nv_max) continue;
                        const Vtx& V = S.V[D.slot[k]];
                        const double* x = S.z + D.col[k];
                        const double dx = x[0] - V.c[0], dy = x[1] - V.c[1], dz = x[2] - V.c[2];
                        if (V.direct || sqrt(dx * dx + dy * dy + dz * dz) > 0.5 * (P.rg - P.rq)) {
                            const double xc[3] = {x[0], x[1], x[2]};
                            __syncthreads();
                            gather(P, D.label[k], xc, cand_ptr(cand, D.slot[k]), S.V[D.slot[k]], &counter, scan);
                        }
                    }
                    phase(8);
                    // ---- Jacobian: the 2m perturbed residuals (task t = 2j + sign) spread over
                    // the warps (only vertex k's MLS moves), then J = (r+ - r-) / 2h by the block
                    if (tid < NW) S.flag[tid] = 1;
                    __syncthreads();
                    for (int t = wid; t < 2 * m; t += NW) {
                        const int j = t >> 1, sgn = t & 1;
                        int k = 0;
                        while (k + 1 < D.n && D.col[k + 1] <= j) ++k;
                        double* zz = S.zw[wid];
                        if (lane < m) zz[lane] = S.z[lane];
                        __syncwarp();
                        if (lane == 0) zz[j] = sgn == 0 ? S.z[j] + kH : S.z[j] - kH;
                        __syncwarp();
                        bool okj = true;
                        double pbk[3] = {0, 0, 0}, nbk[3] = {0, 0, 0};
                        if (D.kind[k] == 0) {
                            double x[3];
                            vpoint(P, D, zz, k, x);
                            okj = mls(P, D, k, x, cand_ptr(cand, D.slot[k]), S.V[D.slot[k]], pbk, nbk, lane);
                        }
                        // only vertices k-1, k, k+1 see unknown j; the rest keep r(z)
                        double* rr = S.Rpm + t * kMaxDim;
                        bool okv = true;
                        if (okj && lane < D.n) {
                            const int q2 = lane;
                            if (q2 >= k - 1 && q2 <= k + 1) {
                                const bool mine = q2 == k && D.kind[k] == 0;
                                okv = vertex_residual(P, D, zz, q2, mine ? pbk : S.pb[q2], mine ? nbk : S.nb[q2], rr);
                            } else {
                                const int c0 = D.col[q2], c1 = q2 + 1 < D.n ? D.col[q2 + 1] : m;
                                for (int i = c0; i < c1; ++i) rr[i] = S.r[i];
                            }
                        }
                        okj = okj && __all_sync(0xffffffffu, okv);
                        if (!okj && lane == 0) S.flag[wid] = 0;
                        __syncwarp();
                    }
                    __syncthreads();
                    bool okJ = true;
                    for (int w = 0; w < NW; ++w) okJ = okJ && S.flag[w];
                    if (!okJ) {
                        status = NRT_REF_NO_SUPPORT;
                        break;
                    }
                    for (int e = tid; e < m * m; e += blockDim.x) {
                        const int i = e / m, j = e % m;
                        S.J[i * m + j] = (S.Rpm[(2 * j) * kMaxDim + i] - S.Rpm[(2 * j + 1) * kMaxDim + i]) / (2.0 * kH);
                    }
                    __syncthreads();
                    phase(9);
                    // ---- normal equations (whole block) + Cholesky solve (warp 0), m <= 24
                    for (int e = tid; e < m * m + m; e += blockDim.x) {
                        if (e < m * m) {
                            const int i = e / m, j = e % m;
                            double s = 0;
                            for (int q2 = 0; q2 < m; ++q2) s += S.J[q2 * m + i] * S.J[q2 * m + j];
                            S.A[i * m + j] = s;
                        } else {
                            const int i = e - m * m;
                            double s = 0;
                            for (int q2 = 0; q2 < m; ++q2) s += S.J[q2 * m + i] * S.r[q2];
                            S.b[i] = -s;
                        }
                    }
                    __syncthreads();
                    if (wid == 0) {
                        double tr = 0;
                        for (int i = 0; i < m; ++i) tr += S.A[i * m + i];
                        const double lam = 1e-12 * tr / m;
                        if (lane < m) S.A[lane * m + lane] += lam;
                        __syncwarp();
                        // Gauss-Jordan on the SPD system, lane i owning row i: no pivoting is
                        // needed (the pivots are the squared Cholesky diagonals, so a pivot <= 0
                        // is exactly the Cholesky failure -> DEGENERATE); each elimination step
                        // is one division per lane plus independent row updates
                        int solved = 1;
                        double* Ai = S.A + lane * m;
                        for (int k = 0; k < m; ++k) {
                            const double pk = S.A[k * m + k];
                            if (!(pk > 0.0)) {
                                solved = 0;
                                break;
                            }
                            const double* Ak = S.A + k * m;
                            const double bk = S.b[k];
                            double fi = 0.0;
                            if (lane < m && lane != k) fi = Ai[k] / pk;
                            __syncwarp();
                            if (lane < m && lane != k) {
                                for (int j = k + 1; j < m; ++j) Ai[j] -= fi * Ak[j];
                                Ai[k] = 0.0;
                                S.b[lane] -= fi * bk;
                            }
                            __syncwarp();
                        }
                        double dmax = 0;
                        if (solved) {
                            double di = 0.0;
                            if (lane < m) {
                                di = S.b[lane] / Ai[lane];
                                S.b[lane] = di;
                            }
                            dmax = fabs(di);
                            for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
                        }
                        __syncwarp();
                        if (lane == 0) S.dval = solved ? dmax : -1.0;
                    }
                    __syncthreads();
                    const double dmax = S.dval;
                    if (dmax < 0.0) {
                        status = NRT_REF_DEGENERATE;
                        break;
                    }
                    if (dmax < P.tol) {  // converged: take the (tiny) full step
                        if (wid == 0) {
                            double* zt = S.zw[0];
                            if (lane < m) zt[lane] = S.z[lane] + S.b[lane];
                            __syncwarp();
                            residual_all(P, D, zt, cand, S.V, S.tr[0], lane);
                            if (S.tr[0].ok && lane < m) S.z[lane] = zt[lane];
                        }
                        status = NRT_REF_OK;
                        __syncthreads();
                        break;
                    }
                    phase(10);
                    // ---- backtracking: NW trials per round, first accepted in sequence order
                    const double f0 = [&] {
                        double s = 0;
                        for (int i = 0; i < m; ++i) s += S.r[i] * S.r[i];
                        return s;
                    }();
                    int accepted = -1;
                    double gacc = 0.0;  // accepted gamma (block-uniform)
                    // trial 0 (gamma = 1, accepted in most iterations) by the whole block, the
                    // vertices' MLS spread over the warps; then rounds of NW trials, warp w
                    // evaluating gamma = beta^(1 + round NW + w)
                    if (wid == 0 && lane < m) S.zw[0][lane] = S.z[lane] + 1.0 * S.b[lane];
                    __syncthreads();
                    residual_coop(P, D, S.zw[0], cand, S.V, S.tr[0], S.okv, wid, lane);
                    if (S.tr[0].ok && S.tr[0].f <= (1.0 - 2.0 * P.alpha * 1.0) * f0) {
                        if (tid < m) {
                            S.z[tid] = S.zw[0][tid];
                            S.r[tid] = S.tr[0].r[tid];
                        } else if (tid >= 32 && tid < 32 + 3 * D.n) {
                            const int k = (tid - 32) / 3, a = (tid - 32) % 3;
                            S.pb[k][a] = S.tr[0].pb[k][a];
                            S.nb[k][a] = S.tr[0].nb[k][a];
                        }
                        accepted = 0;
                        gacc = 1.0;
                    }
                    __syncthreads();
                    for (int round = 0; accepted < 0; ++round) {
                        if (P.cycles && tid == 0) atomicAdd(&g_dbg[2], 1ull);
                        double gam = 1.0;
                        for (int e = 0; e < 1 + round * NW + wid; ++e) gam *= P.beta;
                        const bool live = gam > 1e-12;
                        if (live) {
                            double* zt = S.zw[wid];
                            if (lane < m) zt[lane] = S.z[lane] + gam * S.b[lane];
                            __syncwarp();
                            residual_all(P, D, zt, cand, S.V, S.tr[wid], lane);
                            if (lane == 0)
                                S.flag[wid] = S.tr[wid].ok && S.tr[wid].f <= (1.0 - 2.0 * P.alpha * gam) * f0;
                        } else if (lane == 0) {
                            S.flag[wid] = 2;  // exhausted
                        }
                        __syncthreads();
                        int first = -1;
                        bool exhausted = false;
                        for (int w = 0; w < NW; ++w) {
                            if (S.flag[w] == 2) {
                                exhausted = true;
                                break;
                            }
                            if (S.flag[w] == 1) {
                                first = w;
                                break;
                            }
                        }
                        if (first >= 0) {
                            double gm = 1.0;  // the sequential loop's gamma, same products
                            for (int e = 0; e < 1 + round * NW + first; ++e) gm *= P.beta;
                            gacc = gm;
                            if (tid < m) {
                                S.z[tid] = S.z[tid] + gm * S.b[tid];
                                S.r[tid] = S.tr[first].r[tid];
                            } else if (tid >= 32 && tid < 32 + 3 * D.n) {
                                const int k = (tid - 32) / 3, a = (tid - 32) % 3;
                                S.pb[k][a] = S.tr[first].pb[k][a];
                                S.nb[k][a] = S.tr[first].nb[k][a];
                            }
                            accepted = first;
                        } else if (exhausted) {
                            accepted = NW;  // sentinel: failed
                        }
                        __syncthreads();
                    }
                    phase(11);
                    if (accepted == NW) {
                        status = NRT_REF_NO_CONVERGE;
                        break;
                    }
                    if (gacc * dmax < P.tol) {  // R23b: stalled at a non-root
                        status = NRT_REF_NO_CONVERGE;
                        break;
                    }
                }
                if (it > P.max_iter) it = P.max_iter;
            }
        }
        __syncthreads();
        const long long t_valid = clock64();
        // ---- final residual, gradient norm, validity.  Warp 0: residual, on-edge, same side;
        // then the support tests (one per reflection vertex) and the shadow rays (one per
        // segment) run on separate warps; the status is the first failing check in R25 order.
        if (wid == 0) {
            double (*I)[3] = S.I;
            if (lane <= D.n + 1) vpoint(P, D, S.z, lane - 1, I[lane]);
            __syncwarp();
            double gsq = 0, rmax = 0;
            Trial& T = S.tr[0];
            if (status == NRT_REF_OK && m > 0) {
                residual_all(P, D, S.z, cand, S.V, T, lane);
                if (!T.ok) status = NRT_REF_NO_SUPPORT;
                else {
                    for (int k = 0; k < D.n; ++k) {
                        const double* rk = T.r + D.col[k];
                        gsq += D.kind[k] == 0 ? rk[0] * rk[0] + rk[1] * rk[1] : rk[0] * rk[0];
                    }
                    for (int i = 0; i < m; ++i) rmax = fmax(rmax, fabs(T.r[i]));
                }
            } else {
                for (int i = 0; i < m; ++i) rmax = fmax(rmax, fabs(S.r[i]));
            }
            const double (*nbf)[3] = (status == NRT_REF_OK && m > 0) ? T.nb : S.nb;
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
                        const double sa = ddot(a, nbf[k]), sb = ddot(b, nbf[k]);
                        if (!((sa > 0 && sb > 0) || (sa < 0 && sb < 0))) status = NRT_REF_WRONG_SIDE;
                    }
            if (lane < 3 * D.n) S.nbv[lane / 3][lane % 3] = nbf[lane / 3][lane % 3];
            if (lane == 0) {
                S.vstat = status;
                S.gsq = gsq;
                S.rmax = rmax;
            }
        }
        __syncthreads();
        status = S.vstat;
        if (status == NRT_REF_OK) {
            const double (*I)[3] = S.I;
            const double (*nbf)[3] = S.nbv;
            for (int t = wid; t < 2 * D.n + 1; t += NW) {
                if (t < D.n) {  // support of reflection vertex t (R25 c)
                    const int k = t;
                    const bool ok = D.kind[k] != 0 || supported(P, D.label[k], I[k + 1], lane);
                    if (lane == 0) S.vflag[t] = ok ? 0 : 1;
                    continue;
                }
                const int j = t - D.n;  // shadow ray of segment j (R25 d)
                double l0[6], l1[6];
                int n0 = 0, n1 = 0;
                if (j >= 1) {
                    const int k = j - 1;
                    if (D.kind[k] == 0) {
                        for (int a = 0; a < 3; ++a) l0[a] = nbf[k][a];
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
                        for (int a = 0; a < 3; ++a) l1[a] = nbf[k][a];
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
                const bool occ = occluded(P, I[j], I[j + 1], l0, n0, l1, n1, lane);
                if (lane == 0) S.vflag[t] = occ ? 1 : 0;
            }
        }
        __syncthreads();
        if (wid == 0) {
            double (*I)[3] = S.I;
            const double (*nbf)[3] = S.nbv;
            const double gsq = S.gsq, rmax = S.rmax;
            if (status == NRT_REF_OK) {
                for (int k = 0; k < D.n; ++k)
                    if (S.vflag[k]) status = NRT_REF_NO_SUPPORT;
                if (status == NRT_REF_OK)
                    for (int j = 0; j <= D.n; ++j)
                        if (S.vflag[D.n + j]) status = NRT_REF_OCCLUDED;
            }
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
                    const double c2 = D.kind[k] == 0 ? fabs(ddot(din, nbf[k])) / l : ddot(din, D.ee[k]) / l;
                    o.inc[k] = (float)(acos(fmax(-1.0, fmin(1.0, c2))) * 180.0 / kPi);
                }
                o.status = status;
                o.iters = it;
                o.resid = m ? rmax : 0.0;
                o.gradsq = gsq;
                if (P.cycles) {
                    P.cycles[jq] = clock64() - t_start;
                    atomicAdd(&g_dbg[7], (unsigned long long)(clock64() - t_valid));
                }
                const unsigned long long at = P.keep_invalid ? (unsigned long long)jq : atomicAdd(P.n_out, 1ull);
                P.out[at] = o;
            }
        }
        __syncthreads();
    }
}

// select flags (nrt_refine_desc.select): 1 keeps paths without a diffraction, 2 with one
// (f may be null: sel = 0 keeps everything); nrefl_max = max reflections of a kept path
__global__ void k_select_flags(const nrt_coarse_rec* in, int64_t n, int sel, unsigned char* f,
                               int* nrefl_max) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const bool keep = sel == 0 || (in[i].n_diff > 0) == (sel == 2);
    if (f) f[i] = keep;
    if (keep) atomicMax(nrefl_max, (int)in[i].n_int - (int)in[i].n_diff);
}

}  // namespace

#ifndef NRT_REFINE_ENTRY
#define NRT_REFINE_ENTRY refine
#endif
nrt_status NRT_REFINE_ENTRY(nrt_scene s, nrt_paths coarse, const nrt_refine_desc* d, nrt_paths out,
                            cudaStream_t st) {
#if NRT_REFINE_WARPS == 8
    {  // latency regime (few paths, set by a tail of long GN runs): the 12-warp build of this
       // file (refine_nw12.cu) — per-path results do not depend on the warp count
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s->device);
        const int64_t mine = coarse->n / (d->world > 0 ? d->world : 1);
        const char* e = getenv("NRT_REFINE_NW12");
        if (e ? atoi(e) != 0 : mine < (int64_t)sms * 3 * 8) return refine_nw12(s, coarse, d, out, st);
    }
#endif
    int64_t n = coarse->n;
    out->n = 0;
    const nrt_coarse_rec* in = (const nrt_coarse_rec*)coarse->d_rec;
    nrt_coarse_rec* sel_buf = nullptr;
    // reflection vertices per path bound the shared candidate slots; a launch handle knows its
    // max_refl, an imported or filtered set is scanned
    int nrefl = coarse->max_refl > 0 ? coarse->max_refl : -1;
    if ((d->select != 0 || nrefl < 0) && n > 0) {  // order-preserving compaction of the selected kind
        unsigned char* flags = nullptr;
        int64_t* d_ns = nullptr;
        int* d_nr = nullptr;
        void* tmp = nullptr;
        size_t tb = 0;
        cub::DeviceSelect::Flagged(nullptr, tb, in, (unsigned char*)nullptr, (nrt_coarse_rec*)nullptr,
                                   (int64_t*)nullptr, n, st);
        if (d->select != 0) {
            NRT_CUDA(cudaMallocAsync(&sel_buf, n * sizeof(nrt_coarse_rec), st));
            NRT_CUDA(cudaMallocAsync(&flags, n, st));
            NRT_CUDA(cudaMallocAsync(&tmp, tb, st));
        }
        NRT_CUDA(cudaMallocAsync(&d_ns, sizeof(int64_t) + sizeof(int), st));
        d_nr = (int*)(d_ns + 1);
        NRT_CUDA(cudaMemsetAsync(d_ns, 0, sizeof(int64_t) + sizeof(int), st));
        k_select_flags<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(in, n, d->select, flags, d_nr);
        ::nrt::count_launch();
        if (d->select != 0) cub::DeviceSelect::Flagged(tmp, tb, in, flags, sel_buf, d_ns, n, st);
        struct {
            int64_t ns;
            int nr;
        } h{0, 0};
        NRT_CUDA(cudaMemcpyAsync(&h, d_ns, sizeof(int64_t) + sizeof(int), cudaMemcpyDeviceToHost, st));
        NRT_CUDA(cudaStreamSynchronize(st));
        cudaFreeAsync(flags, st);
        cudaFreeAsync(d_ns, st);
        cudaFreeAsync(tmp, st);
        if (d->select != 0) {
            in = sel_buf;
            n = h.ns;
        }
        nrefl = h.nr;
    }
    struct SelGuard {
        nrt_coarse_rec* p;
        cudaStream_t st;
        ~SelGuard() {
            if (p) cudaFreeAsync(p, st);
        }
    } sel_guard{sel_buf, st};
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
    P.hcell = s->hcell;
    P.hrec = s->hrec;
    P.inv_hv = s->inv_hv;
    P.hx = s->hdims[0];
    P.hy = s->hdims[1];
    P.hz = s->hdims[2];
    P.edges = s->edges;
    P.in = in;
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
    // gather margin: iterates may drift half of it before a re-gather; 1.5 sigma keeps the
    // lists of dense clouds (RR: 5e4 /m^2) within kCapS while sparse ones re-gather rarely
    P.rg = P.rq + (getenv("NRT_REFINE_MARGIN") ? atof(getenv("NRT_REFINE_MARGIN")) : fmax(0.01, 1.5 * P.sigma));
    P.tol = d->tol_m;
    P.alpha = d->alpha;
    P.beta = d->beta;
    P.max_iter = d->max_iter;
    P.keep_invalid = d->keep_invalid;
    // shared candidate slots: one per reflection vertex of the longest path (<= max_refl)
    int nv = nrefl < 1 ? 1 : nrefl > NRT_MAX_INT ? NRT_MAX_INT : nrefl;
    P.nv_max = nv;
    const size_t smem = ((sizeof(Smem) + 15) & ~size_t(15)) + (size_t)nv * kCapS * 6 * sizeof(float);
    const int64_t n_mine = n > d->rank ? (n - d->rank + d->world - 1) / d->world : 0;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s->device);
    // latency regime: fewer paths than ~8 rounds of the throughput grid
#if NRT_REFINE_WARPS == 8
    const bool latency = getenv("NRT_REFINE_MINB") ? atoi(getenv("NRT_REFINE_MINB")) == 2
                                                   : n_mine < (int64_t)sms * 3 * 8;
#else
    const bool latency = true;  // the wide build serves the latency regime only
#endif
#if NRT_REFINE_WARPS == 8
    void (*kern)(RP) = latency ? k_refine<NRT_LAT_MINB> : k_refine<3>;
#else
    void (*kern)(RP) = k_refine<NRT_LAT_MINB>;
    (void)latency;
#endif
    NRT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    NRT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
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
    const bool timing = getenv("NRT_REFINE_TIMING") != nullptr && d->keep_invalid;
    if (timing) {
        NRT_CUDA(cudaMallocAsync(&P.cycles, (size_t)(n_mine > 0 ? n_mine : 1) * 8, st));
        NRT_CUDA(cudaMemsetAsync(P.cycles, 0, (size_t)(n_mine > 0 ? n_mine : 1) * 8, st));
        const unsigned long long zero[16] = {};
        NRT_CUDA(cudaMemcpyToSymbolAsync(g_dbg, zero, sizeof(zero), 0, cudaMemcpyHostToDevice, st));
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * NW, smem);
    if (per_sm < 1) per_sm = 1;
    if (d->blocks_per_sm > 0 && d->blocks_per_sm < per_sm) per_sm = d->blocks_per_sm;
    int64_t blocks = (int64_t)sms * per_sm;
    if (blocks > n_mine) blocks = n_mine;
    if (blocks < 1) blocks = 1;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
    if (n_mine > 0) {
        kern<<<(unsigned)blocks, 32 * NW, smem, st>>>(P);
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
    cudaFreeAsync(d_rx, st);
    cudaFreeAsync(ctr, st);
    if (timing) {
        std::vector<long long> cyc(n_mine > 0 ? n_mine : 1);
        std::vector<nrt_refined_rec> rr(n_mine > 0 ? n_mine : 1);
        cudaMemcpy(cyc.data(), P.cycles, n_mine * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(rr.data(), o, n_mine * sizeof(nrt_refined_rec), cudaMemcpyDeviceToHost);
        std::vector<int64_t> ix(n_mine);
        for (int64_t i = 0; i < n_mine; ++i) ix[i] = i;
        std::sort(ix.begin(), ix.end(), [&](int64_t a, int64_t b) { return cyc[a] > cyc[b]; });
        long long tot = 0;
        for (int64_t i = 0; i < n_mine; ++i) tot += cyc[i];
        fprintf(stderr, "[nrt] refine: %lld paths, sum %.3g cycles, blocks %lld\n", (long long)n_mine,
                (double)tot, (long long)blocks);
        unsigned long long dbg[16];
        cudaMemcpyFromSymbol(dbg, g_dbg, sizeof(dbg));
        fprintf(stderr, "[nrt]   block cycles: prologue %.3g regather %.3g jacobian %.3g solve %.3g linesearch %.3g validity %.3g\n",
                (double)dbg[6], (double)dbg[8], (double)dbg[9], (double)dbg[10], (double)dbg[11], (double)dbg[7]);
        fprintf(stderr, "[nrt]   mls list %llu direct %llu, ls rounds %llu, gathers %llu\n", dbg[0], dbg[1],
                dbg[2], dbg[3]);
        fprintf(stderr, "[nrt]   avg cycles: mls list %.0f direct %.0f\n", (double)dbg[4] / (dbg[0] + 1),
                (double)dbg[5] / (dbg[1] + 1));
        fprintf(stderr, "[nrt]   direct MLS with an empty neighbourhood: %llu (%.3g cycles)\n", dbg[12],
                (double)dbg[13]);
        for (int64_t i = 0; i < n_mine && i < 12; ++i)
            fprintf(stderr, "[nrt]   path %lld: %.3g cycles, n_int %d, iters %d, status %d\n",
                    (long long)ix[i], (double)cyc[ix[i]], rr[ix[i]].n_int, rr[ix[i]].iters,
                    rr[ix[i]].status);
        cudaFree(P.cycles);
    }
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
