// refine.cu — A9-A10: batched path refinement (FP64).
//
// The refined path is the root of the residual of DESIGN.md §5 (readings R18-R28, R37):
//   reflection k: r_k = [g.u, g.v, f_sdf] with the MLS surface of Eqs. 1-4 over
//     the same-label surfels within 4 sigma (sigma = xi r_s), normals oriented by the
//     seed normal (Eq. 3 + R20), basis (u, v) of the MLS normal, g the Eq. 9-10 vector;
//   diffraction k: r_k = g.e (Eq. 11, I_k = a + t_k e, Eq. 8).
// reached by damped Gauss-Newton with the analytic Jacobian (R37: chain rule through g, the MLS
// point and normal and the basis), step -(J^T J + lam I)^-1 J^T r, Armijo backtracking (Eq. 12
// form, R24), converged at |D|_inf < tol, stalled (NO_CONVERGE, R23b) once an accepted step
// |gamma D|_inf < tol.  Then validity (R25): on-edge, same side, support, FP64 visibility;
// delay = L/c (R26), angles (R27).
//
// B200 mapping.  Two kernels over the same device functions (the same arithmetic):
//   * k_refine_w, ONE WARP PER PATH (BJ "one warp per path running Gauss-Newton"), the
//     throughput regime (1e4-1e6 paths): no block barrier; the derivative MLS passes, the
//     backtracking trials (in sequence, each stopping at its first undefined vertex or once its
//     partial sum of squares exceeds the Armijo bound) and the validity checks all on the warp;
//   * k_refine_b, ONE BLOCK OF NW WARPS PER PATH, the latency regime (few paths; the kernel time
//     is the longest GN runs): vertices' MLS over the warps, NW speculative trials per round.
// Per reflection vertex the warp/block keeps a candidate list in global scratch (L2-resident):
// the label's surfels within 4 sigma + mw of a gather centre as FP64 SoA with the Eq. 3
// orientation folded in; an MLS point farther than mw from the centre scans the home grid's
// cell rows directly (same set).  MLS sums: lanes split the candidates, butterfly reduce.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "internal.cuh"

namespace nrt {

namespace {

#ifndef NRT_REFINE_NW
#define NRT_REFINE_NW 12
#endif
constexpr int NW = NRT_REFINE_NW;  // warps per path of the block kernel (latency regime)
constexpr int kMaxDim = 3 * NRT_MAX_INT;
constexpr double kC = 299792458.0;

struct RP {
    const uint2* cell;
    const float4* rec;
    const float4* sp;  // (p, r)
    const float4* sn;  // (n, label bits)
    float ox, oy, oz, v, inv_v, pad;
    int nx, ny, nz;
    const uint2* hcell;    // home grid (each surfel once)
    const float4* hrec;
    const unsigned* hoff;  // home-cell record offsets (cell rows are contiguous ranges)
    float inv_hv;
    int hx, hy, hz;
    const DevEdge* edges;
    const nrt_coarse_rec* in;
    int64_t n_in;
    int rank, world;
    double tx[3];
    const float* rx;
    double sigma, rq, tau, cos_ex, tol, alpha, beta;
    int max_iter, nv_max;  // nv_max: candidate-list slots (reflection vertices) per path
    double mw;             // list margin: radius 4 sigma + mw, used while the vertex is within mw
    int capw;              // candidates per list
    nrt_refined_rec* out;
    unsigned long long* n_out;
    int keep_invalid;
    unsigned long long* work;
    long long* cycles;  // optional per-path latency (NRT_REFINE_TIMING diagnostics)
    unsigned long long* mls_cnt;  // optional [value, deriv] neighbourhood terms evaluated
};

struct Path {
    int n, dim;
    int kind[NRT_MAX_INT];
    int32_t label[NRT_MAX_INT];
    uint32_t prim[NRT_MAX_INT];
    int col[NRT_MAX_INT];
    int slot[NRT_MAX_INT];  // candidate-list slot of a reflection vertex
    double nseed[NRT_MAX_INT][3];
    double ea[NRT_MAX_INT][3], ee[NRT_MAX_INT][3], elen[NRT_MAX_INT];
    double rxp[3];
};

struct Vtx {
    double c[3];
    int n;       // candidates in the list
    int direct;  // 1: no usable list (overflow) -> direct scans
};

struct Trial {  // one residual evaluation
    double r[kMaxDim];
    double pb[NRT_MAX_INT][3], nb[NRT_MAX_INT][3];
    double f;
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

__device__ unsigned long long g_dbg[16];  // diagnostics (NRT_REFINE_TIMING)

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

// exp(x) for the Gaussian weights of Eq. 4 (x <= 0), table-driven: x = (32 k' + j) ln2/32 + r,
// exp(x) = 2^k' 2^(j/32) exp(r), |r| <= ln2/64, exp(r) by a degree-6 Taylor polynomial
// (truncation 4e-18 relative); about 2 ulp, like the library exp (results are compared with a
// tolerance), at 12 FP64 operations instead of the library's range-checked 18 plus
// constant materialisation.  2^(j/32) in shared memory (s_exp2), filled by init_exp2().
__shared__ double s_exp2[32];
__constant__ double c_exp2[32] = {  // 2^(j/32), correctly rounded (computed at 200 bits)
    1.0, 1.0218971486541166, 1.0442737824274138, 1.0671404006768237,
    1.0905077326652577, 1.1143867425958924, 1.1387886347566916, 1.1637248587775775,
    1.189207115002721, 1.215247359980469, 1.241857812073484, 1.2690509571917332,
    1.2968395546510096, 1.3252366431597413, 1.3542555469368927, 1.383909881963832,
    1.4142135623730951, 1.4451808069770467, 1.4768261459394993, 1.5091644275934228,
    1.5422108254079407, 1.5759808451078865, 1.6104903319492543, 1.645755478153965,
    1.681792830507429, 1.718619298122478, 1.7562521603732995, 1.7947090750031072,
    1.8340080864093424, 1.8741676341103, 1.9152065613971474, 1.9571441241754002,
};
__device__ __forceinline__ void init_exp2() {
    if (threadIdx.x < 32) s_exp2[threadIdx.x] = c_exp2[threadIdx.x];
}
__device__ __forceinline__ double exp_neg(double x) {
    x = fmax(x, -700.0);
    const double t = fma(x, 46.166241308446828, 6755399441055744.0);  // x 32/ln2 + 1.5 2^52
    const double kf = t - 6755399441055744.0;                          // round(x 32/ln2)
    const int k = __double2loint(t);
    double r = fma(kf, -0.021660849392498290, x);                      // Cody-Waite, ln2/32 hi
    r = fma(kf, -7.2470212932696856e-19, r);                           // and lo
    double q = 1.0 / 720.0;
    q = fma(q, r, 1.0 / 120.0);
    q = fma(q, r, 1.0 / 24.0);
    q = fma(q, r, 1.0 / 6.0);
    q = fma(q, r, 0.5);
    q = fma(q, r, 1.0);                                                // exp(r) = 1 + r q
    const double tj = s_exp2[k & 31];
    const double w = fma(tj * r, q, tj);
    return __hiloint2double(__double2hiint(w) + ((k >> 5) << 20), __double2loint(w));
}

// list element type: the surfel inputs are float, so float storage is exact (the conversion to
// double happens at use); NRT_LIST_F64=1 stores them pre-converted (twice the L2 footprint;
// measured: no faster)
#if defined(NRT_LIST_F64) && NRT_LIST_F64
typedef double lst_t;
#else
typedef float lst_t;
#endif

// candidate list of one reflection vertex in the warp kernel's global scratch: SoA,
// rows (p.x, p.y, p.z, s n.x, s n.y, s n.z) of capw entries, s = sgn(n . n_seed) folded in at
// gather time (the Eq. 3 + R20 orientation is fixed per vertex), so an MLS evaluation does no
// float->double conversion and no orientation test.
__device__ __forceinline__ lst_t* wlist(lst_t* cand, int slot, int capw) {
    return cand + (size_t)slot * 6 * capw;
}

// warp gather of the label's surfels within 4 sigma + mw of c (home cells in linear order,
// records of a cell in order, compacted by a warp prefix sum over rounds of 32 cells)
__device__ __noinline__ void gather_w(const RP& P, int32_t label, const double ns[3], const double c[3],
                                      lst_t* list, Vtx& V, int lane) {
    if (lane == 0) {
        V.c[0] = c[0];
        V.c[1] = c[1];
        V.c[2] = c[2];
        if (P.cycles) atomicAdd(&g_dbg[3], 1ull);
    }
    const double rl = 4.0 * P.sigma + P.mw;
    const Box B = home_box(P, c, rl);
    const int nxr = B.i1 - B.i0 + 1, nyr = B.j1 - B.j0 + 1, nzr = B.k1 - B.k0 + 1;
    const int ncells = (nxr > 0 && nyr > 0 && nzr > 0) ? nxr * nyr * nzr : 0;
    const double rl2 = rl * rl;
    auto match = [&](unsigned k, float4& A, float4& nv) {
        A = __ldg(&P.hrec[2 * k]);
        const double dx = (double)A.x - c[0], dy = (double)A.y - c[1], dz = (double)A.z - c[2];
        if ((dx * dx + dy * dy) + dz * dz > rl2) return false;
        nv = __ldg(&P.hrec[2 * k + 1]);
        return __float_as_int(nv.w) == label;
    };
    const int cap = P.capw;
    int count = 0;
    for (int base = 0; base < ncells; base += 32) {
        const int q = base + lane;
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
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const int tot = __shfl_sync(0xffffffffu, incl, 31);
        if (cnt)
            for (unsigned k = rg.x, w = 0; k < rg.y; ++k) {
                float4 A, nv;
                if (!match(k, A, nv)) continue;
                const int at = count + (incl - cnt) + (int)w++;
                if (at < cap) {
                    const double n0 = nv.x, n1 = nv.y, n2 = nv.z;
                    const double sg = ((n0 * ns[0] + n1 * ns[1]) + n2 * ns[2]) < 0.0 ? -1.0 : 1.0;
                    list[at] = A.x;
                    list[cap + at] = A.y;
                    list[2 * cap + at] = A.z;
                    list[3 * cap + at] = sg * n0;
                    list[4 * cap + at] = sg * n1;
                    list[5 * cap + at] = sg * n2;
                }
            }
        count += tot;
    }
    if (lane == 0) {
        V.direct = count > cap;
        V.n = V.direct ? 0 : count;
    }
    __syncwarp();
}

// MLS (Eqs. 1-4) at x, one warp: from the vertex's FP64 list when x lies within mw of its
// gather centre (the list then holds every label surfel within 4 sigma of x), else by a direct
// scan of the home grid.  Two candidates per lane per round (independent exp chains).
__device__ __noinline__ bool mls_w(const RP& P, const Path& D, int k, const double x[3], const lst_t* list,
                                   const Vtx& V, double pb[3], double nb[3], int lane) {
    const double inv2s2 = 1.0 / (2.0 * P.sigma * P.sigma);
    const double r2 = (4.0 * P.sigma) * (4.0 * P.sigma);
    double W = 0, Px = 0, Py = 0, Pz = 0, Nx = 0, Ny = 0, Nz = 0;
    const double dxc = x[0] - V.c[0], dyc = x[1] - V.c[1], dzc = x[2] - V.c[2];
    const bool use_list = !V.direct && sqrt(dxc * dxc + dyc * dyc + dzc * dzc) <= P.mw;
    if (P.cycles && lane == 0) atomicAdd(&g_dbg[use_list ? 0 : 1], 1ull);
    const long long t_mls0 = P.cycles ? clock64() : 0;
    unsigned terms = 0;  // neighbourhood members within 4 sigma evaluated by this lane
    if (use_list) {
        const int n = V.n, cap = P.capw;
        const double x0 = x[0], x1 = x[1], x2 = x[2];
        for (int j = lane; j < n; j += 64) {
            const int j2 = j + 32;
            const bool has2 = j2 < n;
            const double a0 = list[j], a1 = list[cap + j], a2 = list[2 * cap + j];
            const double b0 = has2 ? list[j2] : 0.0, b1 = has2 ? list[cap + j2] : 0.0,
                         b2 = has2 ? list[2 * cap + j2] : 0.0;
            const double da0 = a0 - x0, da1 = a1 - x1, da2 = a2 - x2;
            const double db0 = b0 - x0, db1 = b1 - x1, db2 = b2 - x2;
            const double dda = (da0 * da0 + da1 * da1) + da2 * da2;
            const double ddb = (db0 * db0 + db1 * db1) + db2 * db2;
            const double wa0 = exp_neg(-dda * inv2s2), wb0 = exp_neg(-ddb * inv2s2);
            const double wa = dda <= r2 ? wa0 : 0.0;
            const double wb = (has2 && ddb <= r2) ? wb0 : 0.0;
            terms += (dda <= r2) + (has2 && ddb <= r2);
            const double na0 = list[3 * cap + j], na1 = list[4 * cap + j], na2 = list[5 * cap + j];
            const double nb0 = has2 ? list[3 * cap + j2] : 0.0, nb1 = has2 ? list[4 * cap + j2] : 0.0,
                         nb2 = has2 ? list[5 * cap + j2] : 0.0;
            W += wa;
            Px += wa * a0;
            Py += wa * a1;
            Pz += wa * a2;
            Nx += wa * na0;
            Ny += wa * na1;
            Nz += wa * na2;
            W += wb;
            Px += wb * b0;
            Py += wb * b1;
            Pz += wb * b2;
            Nx += wb * nb0;
            Ny += wb * nb1;
            Nz += wb * nb2;
        }
    } else {
        // direct scan: the home cells of the box x +- 4 sigma, one contiguous record range per
        // (y, z) row of cells; an FP32 distance test with a margin >> its rounding skips the
        // records that are certainly outside 4 sigma before the FP64 arithmetic
        const int32_t label = D.label[k];
        const double* ns = D.nseed[k];
        const Box B = home_box(P, x, 4.0 * P.sigma);
        const float xf0 = (float)x[0], xf1 = (float)x[1], xf2 = (float)x[2];
        const float rf = (float)(4.0 * P.sigma) + 1e-4f + 1e-6f * (fabsf(xf0) + fabsf(xf1) + fabsf(xf2));
        const float r2f = rf * rf;
        if (B.i0 <= B.i1)  // (a box outside the grid is empty)
        for (int ck = B.k0; ck <= B.k1; ++ck)
            for (int cj = B.j0; cj <= B.j1; ++cj) {
                const unsigned row = (unsigned)P.hx * ((unsigned)cj + (unsigned)P.hy * (unsigned)ck);
                const unsigned r0 = __ldg(&P.hoff[row + B.i0]), r1 = __ldg(&P.hoff[row + B.i1 + 1]);
                for (unsigned q = r0 + lane; q < r1; q += 32) {
                    const float4 A = __ldg(&P.hrec[2 * q]);
                    const float e0 = A.x - xf0, e1 = A.y - xf1, e2 = A.z - xf2;
                    if ((e0 * e0 + e1 * e1) + e2 * e2 > r2f) continue;
                    const double p0 = A.x, p1 = A.y, p2 = A.z;
                    const double d0 = p0 - x[0], d1 = p1 - x[1], d2 = p2 - x[2];
                    const double dd = (d0 * d0 + d1 * d1) + d2 * d2;
                    if (dd > r2) continue;
                    const float4 nv = __ldg(&P.hrec[2 * q + 1]);
                    if (__float_as_int(nv.w) != label) continue;
                    const double n0 = nv.x, n1 = nv.y, n2 = nv.z;
                    const double sg = ((n0 * ns[0] + n1 * ns[1]) + n2 * ns[2]) < 0.0 ? -1.0 : 1.0;
                    const double w = exp_neg(-dd * inv2s2);
                    ++terms;
                    W += w;
                    Px += w * p0;
                    Py += w * p1;
                    Pz += w * p2;
                    Nx += w * (sg * n0);
                    Ny += w * (sg * n1);
                    Nz += w * (sg * n2);
                }
            }
    }
    if (P.mls_cnt) {
        unsigned t = terms;
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) atomicAdd(&P.mls_cnt[0], (unsigned long long)t);
    }
    W = wsum(W);
    Px = wsum(Px);
    Py = wsum(Py);
    Pz = wsum(Pz);
    Nx = wsum(Nx);
    Ny = wsum(Ny);
    Nz = wsum(Nz);
    if (P.cycles && lane == 0) atomicAdd(&g_dbg[use_list ? 4 : 5], (unsigned long long)(clock64() - t_mls0));
    if (!(W > 0.0)) return false;
    const double iw = 1.0 / W;
    pb[0] = Px * iw;
    pb[1] = Py * iw;
    pb[2] = Pz * iw;
    // n = normalize(N / W) = N / |N| (the 1/W scale cancels; one reciprocal square root)
    const double l2 = (Nx * Nx + Ny * Ny) + Nz * Nz;
    if (!(l2 > 0.0)) return false;
    const double il = rsqrt(l2);
    nb[0] = Nx * il;
    nb[1] = Ny * il;
    nb[2] = Nz * il;
    return true;
}


// MLS with the derivatives of pbar(x) and nbar(x), one warp (the analytic Jacobian, reading R37;
// the oracle's mls_d):  w_i = exp(-|d_i|^2 / 2 s^2), d_i = p_i - x, dw_i/dx = w_i d_i / s^2;
//   dpbar/dx = (sum w d d^T / s^2 - (pbar - x) dW^T) / W,  dW = sum w d / s^2,  pbar - x = sum w d / W;
//   dnbar/dx = (I - nbar nbar^T)(sum w sn d^T / s^2) / |N|,  N = sum w sn  (sn: oriented normal).
// 22 sums in one pass over the same neighbourhood as mls_w (list or direct rows).
__device__ __noinline__ bool mls_w_d(const RP& P, const Path& D, int k, const double x[3], const lst_t* list,
                                     const Vtx& V, double dP[3][3], double dN[3][3], int lane) {
    const double s2 = P.sigma * P.sigma;
    const double inv2s2 = 1.0 / (2.0 * s2);
    const double r2 = (4.0 * P.sigma) * (4.0 * P.sigma);
    double W = 0, D0 = 0, D1 = 0, D2 = 0, S00 = 0, S01 = 0, S02 = 0, S11 = 0, S12 = 0, S22 = 0;
    double N0 = 0, N1 = 0, N2 = 0, T[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    unsigned terms = 0;
    auto acc = [&](double d0, double d1, double d2, double dd, double n0, double n1, double n2) {
        ++terms;
        const double w = exp_neg(-dd * inv2s2);
        const double w0 = w * d0, w1 = w * d1, w2 = w * d2;
        W += w;
        D0 += w0;
        D1 += w1;
        D2 += w2;
        S00 += w0 * d0;
        S01 += w0 * d1;
        S02 += w0 * d2;
        S11 += w1 * d1;
        S12 += w1 * d2;
        S22 += w2 * d2;
        const double m0 = w * n0, m1 = w * n1, m2 = w * n2;
        N0 += m0;
        N1 += m1;
        N2 += m2;
        T[0][0] += m0 * d0;
        T[0][1] += m0 * d1;
        T[0][2] += m0 * d2;
        T[1][0] += m1 * d0;
        T[1][1] += m1 * d1;
        T[1][2] += m1 * d2;
        T[2][0] += m2 * d0;
        T[2][1] += m2 * d1;
        T[2][2] += m2 * d2;
    };
    const double dxc = x[0] - V.c[0], dyc = x[1] - V.c[1], dzc = x[2] - V.c[2];
    const bool use_list = !V.direct && sqrt(dxc * dxc + dyc * dyc + dzc * dzc) <= P.mw;
    if (use_list) {
        const int n = V.n, cap = P.capw;
        for (int j = lane; j < n; j += 32) {
            const double d0 = list[j] - x[0], d1 = list[cap + j] - x[1], d2 = list[2 * cap + j] - x[2];
            const double dd = (d0 * d0 + d1 * d1) + d2 * d2;
            if (dd > r2) continue;
            acc(d0, d1, d2, dd, list[3 * cap + j], list[4 * cap + j], list[5 * cap + j]);
        }
    } else {
        const int32_t label = D.label[k];
        const double* ns = D.nseed[k];
        const Box B = home_box(P, x, 4.0 * P.sigma);
        const float xf0 = (float)x[0], xf1 = (float)x[1], xf2 = (float)x[2];
        const float rf = (float)(4.0 * P.sigma) + 1e-4f + 1e-6f * (fabsf(xf0) + fabsf(xf1) + fabsf(xf2));
        const float r2f = rf * rf;
        if (B.i0 <= B.i1)
            for (int ck = B.k0; ck <= B.k1; ++ck)
                for (int cj = B.j0; cj <= B.j1; ++cj) {
                    const unsigned row = (unsigned)P.hx * ((unsigned)cj + (unsigned)P.hy * (unsigned)ck);
                    const unsigned r0 = __ldg(&P.hoff[row + B.i0]), r1 = __ldg(&P.hoff[row + B.i1 + 1]);
                    for (unsigned q = r0 + lane; q < r1; q += 32) {
                        const float4 A = __ldg(&P.hrec[2 * q]);
                        const float e0 = A.x - xf0, e1 = A.y - xf1, e2 = A.z - xf2;
                        if ((e0 * e0 + e1 * e1) + e2 * e2 > r2f) continue;
                        const double d0 = (double)A.x - x[0], d1 = (double)A.y - x[1], d2 = (double)A.z - x[2];
                        const double dd = (d0 * d0 + d1 * d1) + d2 * d2;
                        if (dd > r2) continue;
                        const float4 nv = __ldg(&P.hrec[2 * q + 1]);
                        if (__float_as_int(nv.w) != label) continue;
                        const double n0 = nv.x, n1 = nv.y, n2 = nv.z;
                        const double sg = ((n0 * ns[0] + n1 * ns[1]) + n2 * ns[2]) < 0.0 ? -1.0 : 1.0;
                        acc(d0, d1, d2, dd, sg * n0, sg * n1, sg * n2);
                    }
                }
    }
    if (P.mls_cnt) {
        unsigned t = terms;
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) atomicAdd(&P.mls_cnt[1], (unsigned long long)t);
    }
    W = wsum(W);
    D0 = wsum(D0);
    D1 = wsum(D1);
    D2 = wsum(D2);
    S00 = wsum(S00);
    S01 = wsum(S01);
    S02 = wsum(S02);
    S11 = wsum(S11);
    S12 = wsum(S12);
    S22 = wsum(S22);
    N0 = wsum(N0);
    N1 = wsum(N1);
    N2 = wsum(N2);
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) T[a][b] = wsum(T[a][b]);
    if (!(W > 0.0)) return false;
    const double ln2 = (N0 * N0 + N1 * N1) + N2 * N2;
    if (!(ln2 > 0.0)) return false;
    const double iln = rsqrt(ln2), iW = 1.0 / W, is2 = 1.0 / s2;
    const double q[3] = {D0 * iW, D1 * iW, D2 * iW};          // pbar - x
    const double dW[3] = {D0 * is2, D1 * is2, D2 * is2};
    const double nb[3] = {N0 * iln, N1 * iln, N2 * iln};
    const double S[3][3] = {{S00, S01, S02}, {S01, S11, S12}, {S02, S12, S22}};
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) dP[a][b] = (S[a][b] * is2 - q[a] * dW[b]) * iW;
#pragma unroll
    for (int b = 0; b < 3; ++b) {
        const double nm = (nb[0] * T[0][b] + nb[1] * T[1][b]) + nb[2] * T[2][b];
#pragma unroll
        for (int a = 0; a < 3; ++a) dN[a][b] = (T[a][b] - nb[a] * nm) * is2 * iln;
    }
    return true;
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

__device__ __forceinline__ void basis_w(const double n[3], double u[3], double v[3]) {
    const double m0 = fabs(n[0]), m1 = fabs(n[1]), m2 = fabs(n[2]);
    int k = 0;
    if (m1 < m0) k = 1;
    if (m2 < (k == 0 ? m0 : m1)) k = 2;
    const double ax[3] = {k == 0 ? 1.0 : 0.0, k == 1 ? 1.0 : 0.0, k == 2 ? 1.0 : 0.0};
    u[0] = n[1] * ax[2] - n[2] * ax[1];
    u[1] = n[2] * ax[0] - n[0] * ax[2];
    u[2] = n[0] * ax[1] - n[1] * ax[0];
    const double il = rsqrt(ddot(u, u));
    u[0] *= il;
    u[1] *= il;
    u[2] *= il;
    v[0] = n[1] * u[2] - n[2] * u[1];
    v[1] = n[2] * u[0] - n[0] * u[2];
    v[2] = n[0] * u[1] - n[1] * u[0];
}

// vertex_residual() with reciprocal square roots instead of sqrt + divisions (rounding-level
// differences only; the refined results are compared with a tolerance); rk = the vertex's rows
__device__ bool vres_w(const RP& P, const Path& D, const double* z, int k, const double* pb,
                       const double* nb, double* rk) {
    double x[3], a[3], c[3];
    vpoint(P, D, z, k, x);
    vpoint(P, D, z, k - 1, a);
    vpoint(P, D, z, k + 1, c);
    const double va[3] = {x[0] - a[0], x[1] - a[1], x[2] - a[2]};
    const double vb[3] = {x[0] - c[0], x[1] - c[1], x[2] - c[2]};
    const double qa = ddot(va, va), qb = ddot(vb, vb);
    if (!(qa > 0.0 && qb > 0.0)) return false;
    const double ia = rsqrt(qa), ib = rsqrt(qb);
    const double g[3] = {va[0] * ia + vb[0] * ib, va[1] * ia + vb[1] * ib, va[2] * ia + vb[2] * ib};
    if (D.kind[k] == 0) {
        double u[3], v[3];
        basis_w(nb, u, v);
        const double xp[3] = {x[0] - pb[0], x[1] - pb[1], x[2] - pb[2]};
        rk[0] = ddot(g, u);
        rk[1] = ddot(g, v);
        rk[2] = ddot(xp, nb);
    } else {
        rk[0] = ddot(g, D.ee[k]);
    }
    return true;
}
__device__ __forceinline__ bool vertex_residual_w(const RP& P, const Path& D, const double* z, int k,
                                                  const double* pb, const double* nb, double* r) {
    return vres_w(P, D, z, k, pb, nb, r + D.col[k]);
}

// residual_all() of the warp kernel (MLS from the FP64 lists)
__device__ __noinline__ void residual_all_w(const RP& P, const Path& D, const double* z, lst_t* cand,
                                            const Vtx* V, Trial& T, int lane) {
    bool ok = true;
    double pb[3], nb[3];
    for (int k = 0; k < D.n && ok; ++k) {
        if (D.kind[k] != 0) continue;
        double x[3];
        vpoint(P, D, z, k, x);
        ok = mls_w(P, D, k, x, wlist(cand, D.slot[k], P.capw), V[D.slot[k]], pb, nb, lane);
        if (ok && lane == 0)
            for (int a = 0; a < 3; ++a) {
                T.pb[k][a] = pb[a];
                T.nb[k][a] = nb[a];
            }
    }
    __syncwarp();
    bool okv = true;
    if (ok && lane < D.n) okv = vertex_residual_w(P, D, z, lane, T.pb[lane], T.nb[lane], T.r);
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

// Analytic Jacobian rows of vertex k (reading R37; the oracle's jacobian()), one lane: chain rule
// through g_k = (x_k - x_{k-1})/|.| + (x_k - x_{k+1})/|.|, the MLS point and normal (pb, nb of the
// residual at z, their derivatives dP, dN from mls_w_d), the basis u = normalize(nb x a) (axis a
// fixed by nb), v = nb x u, and x_j = a_j + t_j e_j for diffraction neighbours.  Rows col[k].. of
// J (stride m) are written; false where the residual is undefined.
__device__ bool jac_vertex(const RP& P, const Path& D, const double* z, int k, const double nb[3],
                           const double pb[3], const double dP[3][3], const double dN[3][3], double* J, int m) {
    double x[3], xa[3], xb[3];
    vpoint(P, D, z, k, x);
    vpoint(P, D, z, k - 1, xa);
    vpoint(P, D, z, k + 1, xb);
    const double a[3] = {x[0] - xa[0], x[1] - xa[1], x[2] - xa[2]};
    const double b[3] = {x[0] - xb[0], x[1] - xb[1], x[2] - xb[2]};
    const double qa = ddot(a, a), qb = ddot(b, b);
    if (!(qa > 0.0 && qb > 0.0)) return false;
    const double ia = rsqrt(qa), ib = rsqrt(qb);
    const double ha[3] = {a[0] * ia, a[1] * ia, a[2] * ia}, hb[3] = {b[0] * ib, b[1] * ib, b[2] * ib};
    const double g[3] = {ha[0] + hb[0], ha[1] + hb[1], ha[2] + hb[2]};
    double Ma[3][3], Mb[3][3];
    for (int p = 0; p < 3; ++p)
        for (int q = 0; q < 3; ++q) {
            Ma[p][q] = ((p == q ? 1.0 : 0.0) - ha[p] * ha[q]) * ia;
            Mb[p][q] = ((p == q ? 1.0 : 0.0) - hb[p] * hb[q]) * ib;
        }
    double R[3][3][3];  // [row][neighbour k-1, k, k+1][coordinate]
    const int nrow = D.kind[k] == 0 ? 3 : 1;
    for (int r = 0; r < 3; ++r)
        for (int s = 0; s < 3; ++s)
            for (int q = 0; q < 3; ++q) R[r][s][q] = 0.0;
    if (D.kind[k] == 0) {
        double u[3], v[3];
        basis_w(nb, u, v);
        const double m0 = fabs(nb[0]), m1 = fabs(nb[1]), m2 = fabs(nb[2]);
        int ax = 0;
        if (m1 < m0) ax = 1;
        if (m2 < (ax == 0 ? m0 : m1)) ax = 2;
        const double av[3] = {ax == 0 ? 1.0 : 0.0, ax == 1 ? 1.0 : 0.0, ax == 2 ? 1.0 : 0.0};
        const double c[3] = {nb[1] * av[2] - nb[2] * av[1], nb[2] * av[0] - nb[0] * av[2],
                             nb[0] * av[1] - nb[1] * av[0]};
        const double ilc = rsqrt(ddot(c, c));
        // Ax v = av x v; dU = (I - u u^T)(-Ax) / |c|; dV = -[u]x + [nb]x dU
        const double Ax[3][3] = {{0, -av[2], av[1]}, {av[2], 0, -av[0]}, {-av[1], av[0], 0}};
        const double Ux[3][3] = {{0, -u[2], u[1]}, {u[2], 0, -u[0]}, {-u[1], u[0], 0}};
        const double Nx[3][3] = {{0, -nb[2], nb[1]}, {nb[2], 0, -nb[0]}, {-nb[1], nb[0], 0}};
        double dU[3][3], dV[3][3];
        for (int p = 0; p < 3; ++p)
            for (int q = 0; q < 3; ++q) {
                double t = 0;
                for (int r = 0; r < 3; ++r) t += ((p == r ? 1.0 : 0.0) - u[p] * u[r]) * (-Ax[r][q]);
                dU[p][q] = t * ilc;
            }
        for (int p = 0; p < 3; ++p)
            for (int q = 0; q < 3; ++q) {
                double t = -Ux[p][q];
                for (int r = 0; r < 3; ++r) t += Nx[p][r] * dU[r][q];
                dV[p][q] = t;
            }
        const double xp[3] = {x[0] - pb[0], x[1] - pb[1], x[2] - pb[2]};
        for (int q = 0; q < 3; ++q) {
            double gu = 0, gv = 0, uM = 0, vM = 0, up = 0, vp = 0, un = 0, vn = 0, fx = 0;
            for (int p = 0; p < 3; ++p) {
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
                fx += nb[p] * ((p == q ? 1.0 : 0.0) - dP[p][q]) + xp[p] * dN[p][q];
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
        const double* e = D.ee[k];
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
    for (int s = 0; s < 3; ++s) {
        const int j = k - 1 + s;
        if (j < 0 || j >= D.n) continue;
        for (int row = 0; row < nrow; ++row) {
            double* Jr = J + (D.col[k] + row) * m;
            if (D.kind[j] == 0) {
                for (int q = 0; q < 3; ++q) Jr[D.col[j] + q] += R[row][s][q];
            } else {
                double t = 0;
                for (int q = 0; q < 3; ++q) t += R[row][s][q] * D.ee[j][q];
                Jr[D.col[j]] += t;
            }
        }
    }
    return true;
}

// the whole Jacobian at z by one warp: the derivative MLS of every reflection vertex (22 sums,
// warp-wide), then lane k assembles the rows of vertex k.  dPN: scratch [NRT_MAX_INT][18].
__device__ __noinline__ bool jacobian_w(const RP& P, const Path& D, const double* z, lst_t* cand, const Vtx* V,
                                       const double (*pb)[3], const double (*nb)[3], double (*dPN)[18],
                                       double* J, int m, int lane) {
    for (int k = 0; k < D.n; ++k) {
        if (D.kind[k] != 0) continue;
        double x[3], dP[3][3], dN[3][3];
        vpoint(P, D, z, k, x);
        if (!mls_w_d(P, D, k, x, wlist(cand, D.slot[k], P.capw), V[D.slot[k]], dP, dN, lane)) return false;
        if (lane == 0)
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) {
                    dPN[k][3 * a + b] = dP[a][b];
                    dPN[k][9 + 3 * a + b] = dN[a][b];
                }
    }
    for (int e = lane; e < m * m; e += 32) J[e] = 0.0;
    __syncwarp();
    bool okv = true;
    if (lane < D.n) {
        double dP[3][3], dN[3][3];
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) {
                dP[a][b] = dPN[lane][3 * a + b];
                dN[a][b] = dPN[lane][9 + 3 * a + b];
            }
        okv = jac_vertex(P, D, z, lane, nb[lane], pb[lane], dP, dN, J, m);
    }
    const bool ok = __all_sync(0xffffffffu, okv);
    __syncwarp();
    return ok;
}

// One backtracking trial at z (the Armijo test f(z) <= bound) with the fewest MLS evaluations:
// vertices in `order` (diffractions, then reflections by decreasing step), stopping at the first
// undefined vertex residual (the trial is rejected either way) or once the partial sum of
// squared residuals exceeds the bound (every term is non-negative, so the full sum would too; the
// 1e-12 relative guard is far above the rounding of <= 24 terms).  A trial evaluated to the end
// gets T.r, T.pb/nb and f summed in index order, exactly as residual_all_w.
__device__ __noinline__ bool trial_w(const RP& P, const Path& D, const double* z, lst_t* cand,
                                     const Vtx* V, Trial& T, const int* order, double bound, int lane) {
    double part = 0.0;
    for (int q = 0; q < D.n; ++q) {
        const int k = order[q];
        double pb[3] = {0, 0, 0}, nb[3] = {0, 0, 0}, rk[3] = {0, 0, 0};
        if (D.kind[k] == 0) {
            double x[3];
            vpoint(P, D, z, k, x);
            if (!mls_w(P, D, k, x, wlist(cand, D.slot[k], P.capw), V[D.slot[k]], pb, nb, lane)) return false;
        }
        if (!vres_w(P, D, z, k, pb, nb, rk)) return false;
        const int nr = D.kind[k] == 0 ? 3 : 1;
        if (lane == 0) {
            for (int a = 0; a < nr; ++a) T.r[D.col[k] + a] = rk[a];
            for (int a = 0; a < 3; ++a) {
                T.pb[k][a] = pb[a];
                T.nb[k][a] = nb[a];
            }
        }
        for (int a = 0; a < nr; ++a) part += rk[a] * rk[a];
        if (part > bound * (1.0 + 1e-12)) {
            __syncwarp();
            return false;
        }
    }
    __syncwarp();
    double f = 0;
    for (int i = 0; i < D.dim; ++i) f += T.r[i] * T.r[i];
    if (lane == 0) {
        T.f = f;
        T.ok = 1;
    }
    __syncwarp();
    return f <= bound;
}

// FP64 occlusion of segment x0 -> x1 (R25 d), one warp.  The segment's t-range [0, len + pad]
// is cut into 32 equal pieces and lane j walks the grid cells of piece j by 3D-DDA (so the
// dependent header loads form 32 short chains instead of one long one); each round, every lane
// stops at its next non-empty cell and the warp tests the union of those cells' records
// together (flattened over the lanes, consecutive lanes on consecutive records).  The pieces'
// cells cover the cells the whole-segment walk visits (a piece starts in the cell holding its
// first point; boundary rounding is covered by the registration pad), and each
// record test is the exact per-record predicate, so the any-hit answer is the same.
__device__ __noinline__ bool occluded(const RP& P, const double x0[3], const double x1[3], const double* lam0,
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
__device__ __noinline__ bool supported(const RP& P, int32_t label, const double x[3], int lane) {
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

// ---- shared by both kernels: the GN step solve, the geometric validity checks, the shadow
// rays with their sheet exclusions, and the output record

// Gauss-Jordan on the SPD normal equations A d = b (m <= 24, lane i owns row i, one warp): no
// pivoting is needed (the pivots are the squared Cholesky diagonals, so a pivot <= 0 is exactly
// the Cholesky failure -> DEGENERATE).  A gets lam = 1e-12 tr(A)/m on its diagonal first.
// b <- d; returns |d|_inf, or -1 on a non-positive pivot.
__device__ double gj_solve(double* A, double* b, int m, int lane) {
    double tr = 0;
    for (int i = 0; i < m; ++i) tr += A[i * m + i];
    const double lam = 1e-12 * tr / m;
    __syncwarp();
    if (lane < m) A[lane * m + lane] += lam;
    __syncwarp();
    int solved = 1;
    double* Ai = A + lane * m;
    for (int k = 0; k < m; ++k) {
        const double pk = A[k * m + k];
        if (!(pk > 0.0)) {
            solved = 0;
            break;
        }
        const double* Ak = A + k * m;
        const double bk = b[k];
        double fi = 0.0;
        if (lane < m && lane != k) fi = Ai[k] / pk;
        __syncwarp();
        if (lane < m && lane != k) {
            for (int j = k + 1; j < m; ++j) Ai[j] -= fi * Ak[j];
            Ai[k] = 0.0;
            b[lane] -= fi * bk;
        }
        __syncwarp();
    }
    double dmax = 0;
    if (solved) {
        double di = 0.0;
        if (lane < m) {
            di = b[lane] / Ai[lane];
            b[lane] = di;
        }
        dmax = fabs(di);
        for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    }
    __syncwarp();
    return solved ? dmax : -1.0;
}

// R25 (a) on-edge and (b) same side, in order; I = the path points, nbf = final MLS normals
__device__ int path_shape_checks(const Path& D, const double* z, const double (*I)[3], const double (*nbf)[3],
                                 int status) {
    if (status == NRT_REF_OK)
        for (int k = 0; k < D.n; ++k)
            if (D.kind[k] == 1) {
                const double t = z[D.col[k]];
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
    return status;
}

// R25 (d) shadow ray of segment j (I[j] -> I[j+1]) with the departure / arrival sheet normals
__device__ bool segment_occluded(const RP& P, const Path& D, const double (*I)[3], const double (*nbf)[3], int j,
                                 int lane) {
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
    return occluded(P, I[j], I[j + 1], l0, n0, l1, n1, lane);
}

// the refined record (R26 delay, R27 angles), written by one thread
__device__ void write_refined(const RP& P, const Path& D, const nrt_coarse_rec& c, const double (*I)[3],
                              const double (*nbf)[3], int status, int it, double rmax, double gsq, int64_t jq,
                              long long t_start, long long t_valid) {
    if (!(P.keep_invalid || status == NRT_REF_OK)) return;
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
    o.resid = rmax;
    o.gradsq = gsq;
    if (P.cycles) {
        P.cycles[jq] = clock64() - t_start;
        atomicAdd(&g_dbg[7], (unsigned long long)(clock64() - t_valid));
    }
    const unsigned long long at = P.keep_invalid ? (unsigned long long)jq : atomicAdd(P.n_out, 1ull);
    P.out[at] = o;
}

// =======================================================================================
// Throughput regime (many paths, e.g. C4/C5): ONE WARP PER PATH.  Each warp of a block refines
// its own path with no block barrier: derivative MLS passes, backtracking trials in sequence and
// the validity checks all on that warp; the candidate lists live in a per-warp global scratch
// (L2-resident), the path state in shared memory.
// =======================================================================================
#ifndef NRT_WPB
#define NRT_WPB 4
#endif
constexpr int kWPB = NRT_WPB;  // independent warps (paths) per block
#ifndef NRT_WMINB
#define NRT_WMINB 5  // resident blocks per SM the register budget is sized for (5 x 4 = 20 warps;
                     // 96 registers with a few spills: C5 refine 705 -> 677 ms vs 4 / 128, 6 / 80 worse)
#endif

struct WS {  // one warp's path state in shared memory (J and A follow all WS, sized by m_max)
    Path D;
    Trial T;
    double z[kMaxDim], r[kMaxDim], b[kMaxDim], zt[kMaxDim];
    double pb[NRT_MAX_INT][3], nb[NRT_MAX_INT][3];
    double I[NRT_MAX_INT + 2][3];
    double dPN[NRT_MAX_INT][18];
    Vtx V[NRT_MAX_INT];
    int order[NRT_MAX_INT];  // backtracking: vertex evaluation order (cheap / far first)
};

__global__ void __launch_bounds__(32 * kWPB, NRT_WMINB) k_refine_w(RP P, lst_t* scratch, int mmax) {
    extern __shared__ __align__(16) unsigned char dyn[];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WS& S = reinterpret_cast<WS*>(dyn)[wid];
    double* J = reinterpret_cast<double*>(dyn + kWPB * sizeof(WS)) + (size_t)wid * 2 * mmax * mmax;
    double* A = J + (size_t)mmax * mmax;
    lst_t* cand = scratch + (size_t)(blockIdx.x * kWPB + wid) * P.nv_max * P.capw * 6;
    init_exp2();
    __syncthreads();
    const int64_t n_mine = P.n_in > P.rank ? (P.n_in - P.rank + P.world - 1) / P.world : 0;
    for (;;) {
        const long long t_start = clock64();
        unsigned long long q = 0;
        if (lane == 0) q = atomicAdd(P.work, 1ull);
        q = __shfl_sync(0xffffffffu, q, 0);
        if ((int64_t)q >= n_mine) break;
        const int64_t jq = n_mine - 1 - (int64_t)q;  // most interactions first (key order end)
        const int64_t pi = P.rank + jq * P.world;
        const nrt_coarse_rec& c = P.in[pi];
        Path& D = S.D;
        if (lane == 0) {
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
            for (int k = 0; k < D.n; ++k) {
                if (D.kind[k] == 0) {
                    for (int a = 0; a < 3; ++a) S.z[D.col[k] + a] = c.v[k][a];
                } else {
                    const double w[3] = {c.v[k][0] - D.ea[k][0], c.v[k][1] - D.ea[k][1], c.v[k][2] - D.ea[k][2]};
                    S.z[D.col[k]] = ddot(w, D.ee[k]);
                }
            }
        }
        for (int e = lane; e < 3 * NRT_MAX_INT; e += 32) {
            (&S.pb[0][0])[e] = 0.0;
            (&S.nb[0][0])[e] = 0.0;
            S.r[e] = 0.0;
        }
        __syncwarp();
        const int m = D.dim;
        for (int k = 0; k < D.n; ++k) {
            if (D.kind[k] != 0) continue;
            const double x[3] = {S.z[D.col[k]], S.z[D.col[k] + 1], S.z[D.col[k] + 2]};
            if (D.slot[k] < P.nv_max) {
                gather_w(P, D.label[k], D.nseed[k], x, wlist(cand, D.slot[k], P.capw), S.V[D.slot[k]], lane);
            } else if (lane == 0) {
                S.V[D.slot[k]].direct = 1;
                S.V[D.slot[k]].n = 0;
            }
        }
        __syncwarp();
        int status = NRT_REF_NO_CONVERGE, it = 0;
        if (m == 0) {
            status = NRT_REF_OK;
        } else {
            residual_all_w(P, D, S.z, cand, S.V, S.T, lane);
            if (!S.T.ok) {
                status = NRT_REF_NO_SUPPORT;
            } else {
                if (lane < m) S.r[lane] = S.T.r[lane];
                if (lane < 3 * D.n) {
                    (&S.pb[0][0])[lane] = (&S.T.pb[0][0])[lane];
                    (&S.nb[0][0])[lane] = (&S.T.nb[0][0])[lane];
                }
                __syncwarp();
                if (P.cycles && lane == 0) atomicAdd(&g_dbg[6], (unsigned long long)(clock64() - t_start));
                for (it = 1; it <= P.max_iter; ++it) {
                    long long tph = clock64();
                    auto phase = [&](int slot) {
                        if (P.cycles && lane == 0) {
                            const long long t = clock64();
                            atomicAdd(&g_dbg[slot], (unsigned long long)(t - tph));
                            tph = t;
                        }
                    };
                    if (P.cycles && lane == 0) atomicAdd(&g_dbg[15], 1ull);
                    // keep every vertex in the safe ball of its candidate list
                    for (int k = 0; k < D.n; ++k) {
                        if (D.kind[k] != 0 || D.slot[k] >= P.nv_max) continue;
                        const Vtx& V = S.V[D.slot[k]];
                        const double* x = S.z + D.col[k];
                        const double dx = x[0] - V.c[0], dy = x[1] - V.c[1], dz = x[2] - V.c[2];
                        if (sqrt(dx * dx + dy * dy + dz * dz) > 0.5 * P.mw) {
                            const double xc[3] = {x[0], x[1], x[2]};
                            __syncwarp();
                            gather_w(P, D.label[k], D.nseed[k], xc, wlist(cand, D.slot[k], P.capw),
                                     S.V[D.slot[k]], lane);
                        }
                    }
                    phase(8);
                    // ---- analytic Jacobian (R37): derivative MLS per reflection vertex + chain rule
                    if (!jacobian_w(P, D, S.z, cand, S.V, S.pb, S.nb, S.dPN, J, m, lane)) {
                        status = NRT_REF_NO_SUPPORT;
                        break;
                    }
                    phase(9);
                    // ---- normal equations + Gauss-Jordan solve
                    for (int e = lane; e < m * m + m; e += 32) {
                        if (e < m * m) {
                            const int i = e / m, j = e % m;
                            double s = 0;
                            for (int q2 = 0; q2 < m; ++q2) s += J[q2 * m + i] * J[q2 * m + j];
                            A[i * m + j] = s;
                        } else {
                            const int i = e - m * m;
                            double s = 0;
                            for (int q2 = 0; q2 < m; ++q2) s += J[q2 * m + i] * S.r[q2];
                            S.b[i] = -s;
                        }
                    }
                    __syncwarp();
                    const double dmax = gj_solve(A, S.b, m, lane);
                    if (dmax < 0.0) {
                        status = NRT_REF_DEGENERATE;
                        break;
                    }
                    if (dmax < P.tol) {  // converged: take the (tiny) full step
                        if (lane < m) S.zt[lane] = S.z[lane] + S.b[lane];
                        __syncwarp();
                        residual_all_w(P, D, S.zt, cand, S.V, S.T, lane);
                        if (S.T.ok && lane < m) S.z[lane] = S.zt[lane];
                        status = NRT_REF_OK;
                        __syncwarp();
                        break;
                    }
                    phase(10);
                    // ---- backtracking, trials in sequence: gamma = beta^e (e = 0, 1, ...)
                    double f0 = 0;
                    for (int i = 0; i < m; ++i) f0 += S.r[i] * S.r[i];
                    if (lane == 0) {  // evaluation order: diffractions, then reflections by |step|
                        double key[NRT_MAX_INT];
                        for (int k = 0; k < D.n; ++k) {
                            const double* bk = S.b + D.col[k];
                            key[k] = D.kind[k] ? 1e300 : (bk[0] * bk[0] + bk[1] * bk[1]) + bk[2] * bk[2];
                            int q = k;
                            while (q > 0 && key[S.order[q - 1]] < key[k]) {
                                S.order[q] = S.order[q - 1];
                                --q;
                            }
                            S.order[q] = k;
                        }
                    }
                    __syncwarp();
                    double gam = 1.0;
                    bool accepted = false;
                    for (int e = 0;; ++e) {
                        if (e > 0) {
                            gam *= P.beta;
                            if (!(gam > 1e-12)) break;  // exhausted
                            if (P.cycles && lane == 0 && (e - 1) % NW == 0) atomicAdd(&g_dbg[2], 1ull);
                        }
                        if (lane < m) S.zt[lane] = S.z[lane] + gam * S.b[lane];
                        __syncwarp();
                        if (P.cycles && lane == 0) atomicAdd(&g_dbg[14], 1ull);
                        if (trial_w(P, D, S.zt, cand, S.V, S.T, S.order, (1.0 - 2.0 * P.alpha * gam) * f0, lane)) {
                            if (lane < m) {
                                S.z[lane] = S.zt[lane];
                                S.r[lane] = S.T.r[lane];
                            }
                            if (lane < 3 * D.n) {
                                (&S.pb[0][0])[lane] = (&S.T.pb[0][0])[lane];
                                (&S.nb[0][0])[lane] = (&S.T.nb[0][0])[lane];
                            }
                            __syncwarp();
                            accepted = true;
                            break;
                        }
                        __syncwarp();
                    }
                    phase(11);
                    if (!accepted) {
                        status = NRT_REF_NO_CONVERGE;
                        break;
                    }
                    if (gam * dmax < P.tol) {  // R23b: stalled at a non-root
                        status = NRT_REF_NO_CONVERGE;
                        break;
                    }
                }
                if (it > P.max_iter) it = P.max_iter;
            }
        }
        __syncwarp();
        const long long t_valid = clock64();
        // ---- final residual, gradient norm, validity (R25 order), as the block kernel
        double (*I)[3] = S.I;
        if (lane <= D.n + 1) vpoint(P, D, S.z, lane - 1, I[lane]);
        __syncwarp();
        double gsq = 0, rmax = 0;
        Trial& T = S.T;
        if (status == NRT_REF_OK && m > 0) {
            residual_all_w(P, D, S.z, cand, S.V, T, lane);
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
        status = path_shape_checks(D, S.z, I, nbf, status);
        if (status == NRT_REF_OK)  // support of every reflection vertex (R25 c)
            for (int k = 0; k < D.n && status == NRT_REF_OK; ++k)
                if (D.kind[k] == 0 && !supported(P, D.label[k], I[k + 1], lane)) status = NRT_REF_NO_SUPPORT;
        if (status == NRT_REF_OK)  // every segment unoccluded (R25 d)
            for (int j = 0; j <= D.n && status == NRT_REF_OK; ++j)
                if (segment_occluded(P, D, I, nbf, j, lane)) status = NRT_REF_OCCLUDED;
        if (lane == 0) write_refined(P, D, c, I, nbf, status, it, m ? rmax : 0.0, gsq, jq, t_start, t_valid);
        __syncwarp();
    }
}
// =======================================================================================
// Latency regime (few paths, e.g. C2's 1.5e3: the kernel time is the longest GN runs): ONE
// BLOCK OF NW WARPS PER PATH.  The independent pieces of an iteration are spread over the warps:
// the derivative MLS of the reflection vertices (vertex k on warp k mod NW), the MLS of the
// gamma = 1 trial (same split), and the backtracking trials (warp w evaluates gamma =
// beta^(1 + round NW + w); the block takes the first passing one in sequence order, the step the
// sequential search takes).  Same arithmetic as k_refine_w (mls_w, mls_w_d, jac_vertex, trial_w).
// =======================================================================================
struct Smem {
    Path D;
    double J[kMaxDim * kMaxDim];
    double A[kMaxDim * kMaxDim];
    Trial tr[NW];
    double z[kMaxDim], r[kMaxDim], b[kMaxDim];
    double pb[NRT_MAX_INT][3], nb[NRT_MAX_INT][3];
    double zw[NW][kMaxDim];
    double I[NRT_MAX_INT + 2][3];
    double dPN[NRT_MAX_INT][18];
    Vtx V[NRT_MAX_INT];
    int flag[NW];
    int okv[NRT_MAX_INT];
    int order[NRT_MAX_INT];
    int vstat;
    int vflag[2 * NRT_MAX_INT + 1];  // validity: support failures [0, n), occlusions [n, 2n+1)
    double nbv[NRT_MAX_INT][3];      // final MLS normals (validity)
    double gsq, rmax;
    double dval;
    unsigned long long q;
};

// the residual at z by the whole block: MLS of reflection vertex k on warp k mod NW, vertex
// residuals on warp 0 (the values residual_all_w gives).  Ends synced.
__device__ void residual_coop_w(const RP& P, const Path& D, const double* z, lst_t* cand, const Vtx* V,
                                Trial& T, int* okv_s, int wid, int lane) {
    for (int k = wid; k < D.n; k += NW) {
        int ok = 1;
        if (D.kind[k] == 0) {
            double x[3], pb[3], nb[3];
            vpoint(P, D, z, k, x);
            ok = mls_w(P, D, k, x, wlist(cand, D.slot[k], P.capw), V[D.slot[k]], pb, nb, lane);
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
        if (ok && lane < D.n) okv = vertex_residual_w(P, D, z, lane, T.pb[lane], T.nb[lane], T.r);
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

__global__ void __launch_bounds__(32 * NW, 1) k_refine_b(RP P, lst_t* scratch) {
    extern __shared__ __align__(16) unsigned char dyn[];
    Smem& S = *reinterpret_cast<Smem*>(dyn);
    const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
    lst_t* cand = scratch + (size_t)blockIdx.x * P.nv_max * P.capw * 6;
    init_exp2();
    __syncthreads();
    const int64_t n_mine = P.n_in > P.rank ? (P.n_in - P.rank + P.world - 1) / P.world : 0;
    for (;;) {
        const long long t_start = clock64();
        if (tid == 0) S.q = atomicAdd(P.work, 1ull);
        __syncthreads();
        const unsigned long long q = S.q;
        __syncthreads();
        if ((int64_t)q >= n_mine) break;
        const int64_t jq = n_mine - 1 - (int64_t)q;
        const int64_t pi = P.rank + jq * P.world;
        const nrt_coarse_rec& c = P.in[pi];
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
            for (int k = 0; k < D.n; ++k) {
                if (D.kind[k] == 0) {
                    for (int a = 0; a < 3; ++a) S.z[D.col[k] + a] = c.v[k][a];
                } else {
                    const double w[3] = {c.v[k][0] - D.ea[k][0], c.v[k][1] - D.ea[k][1], c.v[k][2] - D.ea[k][2]};
                    S.z[D.col[k]] = ddot(w, D.ee[k]);
                }
            }
        }
        for (int e = tid; e < 3 * NRT_MAX_INT; e += blockDim.x) {
            (&S.pb[0][0])[e] = 0.0;
            (&S.nb[0][0])[e] = 0.0;
            S.r[e] = 0.0;
        }
        __syncthreads();
        const int m = D.dim;
        for (int k = wid; k < D.n; k += NW) {  // candidate lists, vertices over the warps
            if (D.kind[k] != 0) continue;
            const double x[3] = {S.z[D.col[k]], S.z[D.col[k] + 1], S.z[D.col[k] + 2]};
            gather_w(P, D.label[k], D.nseed[k], x, wlist(cand, D.slot[k], P.capw), S.V[D.slot[k]], lane);
        }
        __syncthreads();
        int status = NRT_REF_NO_CONVERGE, it = 0;
        if (m == 0) {
            status = NRT_REF_OK;
        } else {
            residual_coop_w(P, D, S.z, cand, S.V, S.tr[0], S.okv, wid, lane);
            if (!S.tr[0].ok) {
                status = NRT_REF_NO_SUPPORT;
            } else {
                if (tid < m) S.r[tid] = S.tr[0].r[tid];
                if (tid >= 32 && tid < 32 + 3 * D.n) {
                    (&S.pb[0][0])[tid - 32] = (&S.tr[0].pb[0][0])[tid - 32];
                    (&S.nb[0][0])[tid - 32] = (&S.tr[0].nb[0][0])[tid - 32];
                }
                __syncthreads();
                for (it = 1; it <= P.max_iter; ++it) {
                    for (int k = wid; k < D.n; k += NW) {  // re-centre drifted candidate lists
                        if (D.kind[k] != 0) continue;
                        const Vtx& V = S.V[D.slot[k]];
                        const double* x = S.z + D.col[k];
                        const double dx = x[0] - V.c[0], dy = x[1] - V.c[1], dz = x[2] - V.c[2];
                        if (sqrt(dx * dx + dy * dy + dz * dz) > 0.5 * P.mw) {
                            const double xc[3] = {x[0], x[1], x[2]};
                            gather_w(P, D.label[k], D.nseed[k], xc, wlist(cand, D.slot[k], P.capw), S.V[D.slot[k]], lane);
                        }
                    }
                    __syncthreads();
                    // ---- analytic Jacobian: derivative MLS of vertex k on warp k mod NW
                    for (int k = wid; k < D.n; k += NW) {
                        int ok = 1;
                        if (D.kind[k] == 0) {
                            double x[3], dP[3][3], dN[3][3];
                            vpoint(P, D, S.z, k, x);
                            ok = mls_w_d(P, D, k, x, wlist(cand, D.slot[k], P.capw), S.V[D.slot[k]], dP, dN, lane);
                            if (ok && lane == 0)
                                for (int a = 0; a < 3; ++a)
                                    for (int b = 0; b < 3; ++b) {
                                        S.dPN[k][3 * a + b] = dP[a][b];
                                        S.dPN[k][9 + 3 * a + b] = dN[a][b];
                                    }
                        }
                        if (lane == 0) S.okv[k] = ok;
                    }
                    for (int e = tid; e < m * m; e += blockDim.x) S.J[e] = 0.0;
                    __syncthreads();
                    if (wid == 0) {
                        bool ok = true;
                        for (int k = 0; k < D.n; ++k) ok = ok && S.okv[k];
                        bool okv = true;
                        if (ok && lane < D.n) {
                            double dP[3][3], dN[3][3];
                            for (int a = 0; a < 3; ++a)
                                for (int b = 0; b < 3; ++b) {
                                    dP[a][b] = S.dPN[lane][3 * a + b];
                                    dN[a][b] = S.dPN[lane][9 + 3 * a + b];
                                }
                            okv = jac_vertex(P, D, S.z, lane, S.nb[lane], S.pb[lane], dP, dN, S.J, m);
                        }
                        ok = ok && __all_sync(0xffffffffu, okv);
                        if (lane == 0) S.flag[0] = ok;
                    }
                    __syncthreads();
                    if (!S.flag[0]) {
                        status = NRT_REF_NO_SUPPORT;
                        break;
                    }
                    // ---- normal equations (whole block) + Gauss-Jordan solve (warp 0)
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
                    if (wid == 0) S.dval = gj_solve(S.A, S.b, m, lane);
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
                            residual_all_w(P, D, zt, cand, S.V, S.tr[0], lane);
                            if (S.tr[0].ok && lane < m) S.z[lane] = zt[lane];
                        }
                        status = NRT_REF_OK;
                        __syncthreads();
                        break;
                    }
                    // ---- backtracking: gamma = 1 by the block, then rounds of NW trials
                    double f0 = 0;
                    for (int i = 0; i < m; ++i) f0 += S.r[i] * S.r[i];
                    if (tid == 0) {
                        double key[NRT_MAX_INT];
                        for (int k = 0; k < D.n; ++k) {
                            const double* bk = S.b + D.col[k];
                            key[k] = D.kind[k] ? 1e300 : (bk[0] * bk[0] + bk[1] * bk[1]) + bk[2] * bk[2];
                            int q2 = k;
                            while (q2 > 0 && key[S.order[q2 - 1]] < key[k]) {
                                S.order[q2] = S.order[q2 - 1];
                                --q2;
                            }
                            S.order[q2] = k;
                        }
                    }
                    if (wid == 0 && lane < m) S.zw[0][lane] = S.z[lane] + 1.0 * S.b[lane];
                    __syncthreads();
                    residual_coop_w(P, D, S.zw[0], cand, S.V, S.tr[0], S.okv, wid, lane);
                    int accepted = -1;
                    double gacc = 0.0;
                    if (S.tr[0].ok && S.tr[0].f <= (1.0 - 2.0 * P.alpha * 1.0) * f0) {
                        if (tid < m) {
                            S.z[tid] = S.zw[0][tid];
                            S.r[tid] = S.tr[0].r[tid];
                        } else if (tid >= 32 && tid < 32 + 3 * D.n) {
                            (&S.pb[0][0])[tid - 32] = (&S.tr[0].pb[0][0])[tid - 32];
                            (&S.nb[0][0])[tid - 32] = (&S.tr[0].nb[0][0])[tid - 32];
                        }
                        accepted = 0;
                        gacc = 1.0;
                    }
                    __syncthreads();
                    for (int round = 0; accepted < 0; ++round) {
                        double gam = 1.0;
                        for (int e = 0; e < 1 + round * NW + wid; ++e) gam *= P.beta;
                        if (gam > 1e-12) {
                            double* zt = S.zw[wid];
                            if (lane < m) zt[lane] = S.z[lane] + gam * S.b[lane];
                            __syncwarp();
                            const bool pass = trial_w(P, D, zt, cand, S.V, S.tr[wid], S.order,
                                                      (1.0 - 2.0 * P.alpha * gam) * f0, lane);
                            if (lane == 0) S.flag[wid] = pass ? 1 : 0;
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
                            double gm = 1.0;
                            for (int e = 0; e < 1 + round * NW + first; ++e) gm *= P.beta;
                            gacc = gm;
                            if (tid < m) {
                                S.z[tid] = S.zw[first][tid];
                                S.r[tid] = S.tr[first].r[tid];
                            } else if (tid >= 32 && tid < 32 + 3 * D.n) {
                                (&S.pb[0][0])[tid - 32] = (&S.tr[first].pb[0][0])[tid - 32];
                                (&S.nb[0][0])[tid - 32] = (&S.tr[first].nb[0][0])[tid - 32];
                            }
                            accepted = first;
                        } else if (exhausted) {
                            accepted = NW;
                        }
                        __syncthreads();
                    }
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
        // ---- final residual, validity in R25 order (support tests and shadow rays on the warps)
        if (wid == 0) {
            double (*I)[3] = S.I;
            if (lane <= D.n + 1) vpoint(P, D, S.z, lane - 1, I[lane]);
            __syncwarp();
            double gsq = 0, rmax = 0;
            Trial& T = S.tr[0];
            if (status == NRT_REF_OK && m > 0) {
                residual_all_w(P, D, S.z, cand, S.V, T, lane);
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
            status = path_shape_checks(D, S.z, I, nbf, status);
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
            for (int t = wid; t < 2 * D.n + 1; t += NW) {
                if (t < D.n) {
                    const bool ok = D.kind[t] != 0 || supported(P, D.label[t], S.I[t + 1], lane);
                    if (lane == 0) S.vflag[t] = ok ? 0 : 1;
                } else {
                    const bool occ = segment_occluded(P, D, S.I, S.nbv, t - D.n, lane);
                    if (lane == 0) S.vflag[t] = occ ? 1 : 0;
                }
            }
        }
        __syncthreads();
        if (wid == 0) {
            if (status == NRT_REF_OK) {
                for (int k = 0; k < D.n; ++k)
                    if (S.vflag[k]) status = NRT_REF_NO_SUPPORT;
                if (status == NRT_REF_OK)
                    for (int j = 0; j <= D.n; ++j)
                        if (S.vflag[D.n + j]) status = NRT_REF_OCCLUDED;
            }
            if (lane == 0)
                write_refined(P, D, c, S.I, S.nbv, status, it, m ? S.rmax : 0.0, S.gsq, jq, t_start, t_valid);
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
    if (keep) {
        atomicMax(nrefl_max, (int)in[i].n_int - (int)in[i].n_diff);
        atomicMax(nrefl_max + 1, 3 * ((int)in[i].n_int - (int)in[i].n_diff) + (int)in[i].n_diff);  // unknowns
    }
}

// FP64 FMA throughput probe: 8 independent chains per thread, no memory traffic
__global__ void k_fp64_probe(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-9 + j;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, b);
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j];
    if (s == 12345.678) out[0] = s;  // keeps the chains alive
}

}  // namespace

double probe_fp64_tflops(int device) {
    if (cudaSetDevice(device) != cudaSuccess) return -1.0;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    double* out = nullptr;
    if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) return -1.0;
    const int iters = 4096, threads = 256, blocks = sms * 8;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_fp64_probe<<<blocks, threads>>>(out, 64, 0.999999, 1e-7);  // warm-up
    cudaEventRecord(e0);
    k_fp64_probe<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    if (cudaGetLastError() != cudaSuccess || !(ms > 0)) return -1.0;
    return 2.0 * 8.0 * iters * (double)threads * blocks / (ms * 1e-3) / 1e12;
}

nrt_status refine(nrt_scene s, nrt_paths coarse, const nrt_refine_desc* d, nrt_paths out, cudaStream_t st) {
    int64_t n = coarse->n;
    out->n = 0;
    const nrt_coarse_rec* in = (const nrt_coarse_rec*)coarse->d_rec;
    nrt_coarse_rec* sel_buf = nullptr;
    // reflection vertices per path bound the shared candidate slots; a launch handle knows its
    // max_refl, an imported or filtered set is scanned
    int nrefl = coarse->max_refl > 0 ? coarse->max_refl : -1;
    int dim_max = coarse->max_refl > 0 ? 3 * coarse->max_refl + coarse->max_diff : -1;
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
        NRT_CUDA(cudaMallocAsync(&d_ns, sizeof(int64_t) + 2 * sizeof(int), st));
        d_nr = (int*)(d_ns + 1);
        NRT_CUDA(cudaMemsetAsync(d_ns, 0, sizeof(int64_t) + 2 * sizeof(int), st));
        k_select_flags<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(in, n, d->select, flags, d_nr);
        ::nrt::count_launch();
        if (d->select != 0) cub::DeviceSelect::Flagged(tmp, tb, in, flags, sel_buf, d_ns, n, st);
        struct {
            int64_t ns;
            int nr, dm;
        } h{0, 0, 0};
        NRT_CUDA(cudaMemcpyAsync(&h, d_ns, sizeof(int64_t) + 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
        NRT_CUDA(cudaStreamSynchronize(st));
        cudaFreeAsync(flags, st);
        cudaFreeAsync(d_ns, st);
        cudaFreeAsync(tmp, st);
        if (d->select != 0) {
            in = sel_buf;
            n = h.ns;
        }
        nrefl = h.nr;
        dim_max = h.dm;
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
    P.hoff = s->hoff;
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
    P.rq = fmax(4.0 * P.sigma, (double)s->r_max + d->tau);  // support-test radius (R25 c)
    // candidate lists: radius 4 sigma + mw, used while the vertex stays within mw of the gather
    // centre, re-gathered once it drifted mw/2 (NRT_REFINE_MW / NRT_REFINE_CAPW override)
    P.mw = getenv("NRT_REFINE_MW") ? atof(getenv("NRT_REFINE_MW")) : fmax(0.004, 0.5 * P.sigma);
    P.capw = getenv("NRT_REFINE_CAPW") ? atoi(getenv("NRT_REFINE_CAPW")) : 1024;
    P.tol = d->tol_m;
    P.alpha = d->alpha;
    P.beta = d->beta;
    P.max_iter = d->max_iter;
    P.keep_invalid = d->keep_invalid;
    const int nv = nrefl < 1 ? 1 : nrefl > NRT_MAX_INT ? NRT_MAX_INT : nrefl;
    P.nv_max = nv;
    const int mmax = dim_max < 1 ? 1 : dim_max > kMaxDim ? kMaxDim : dim_max;
    const int64_t n_mine = n > d->rank ? (n - d->rank + d->world - 1) / d->world : 0;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s->device);
    // latency regime (fewer paths than ~8 rounds of the warp kernel's grid): block per path;
    // NRT_REFINE_IMPL=block|warp forces one
    const char* impl = getenv("NRT_REFINE_IMPL");
    const bool warp_impl = impl ? strcmp(impl, "warp") == 0 : n_mine >= (int64_t)sms * 16 * 4;
    const size_t smem_w = kWPB * sizeof(WS) + (size_t)kWPB * 2 * mmax * mmax * sizeof(double);
    const size_t smem_b = sizeof(Smem);
    int per_sm = 0;
    if (warp_impl) {
        NRT_CUDA(cudaFuncSetAttribute(k_refine_w, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_w));
        if (const char* cv = getenv("NRT_REFINE_CARVEOUT"))  // A/B: shared-memory share of L1 (%)
            cudaFuncSetAttribute(k_refine_w, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(cv));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_refine_w, 32 * kWPB, smem_w);
        if (getenv("NRT_REFINE_CARVEOUT"))
            fprintf(stderr, "nrt: k_refine_w smem %zu B per block, %d blocks/SM\n", smem_w, per_sm);
    } else {
        NRT_CUDA(cudaFuncSetAttribute(k_refine_b, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_b));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_refine_b, 32 * NW, smem_b);
    }
    if (per_sm < 1) per_sm = 1;
    if (d->blocks_per_sm > 0 && d->blocks_per_sm < per_sm) per_sm = d->blocks_per_sm;
    int64_t blocks = (int64_t)sms * per_sm;
    const int64_t per_block = warp_impl ? kWPB : 1;  // paths in flight per block
    if (blocks > (n_mine + per_block - 1) / per_block) blocks = (n_mine + per_block - 1) / per_block;
    if (blocks < 1) blocks = 1;
    lst_t* scratch = nullptr;  // candidate lists: per warp (warp kernel) or per block
    NRT_CUDA(cudaMallocAsync(&scratch, (size_t)blocks * per_block * nv * P.capw * 6 * sizeof(lst_t), st));
    float* d_rx = nullptr;
    const size_t nrx = coarse->rx.size();
    NRT_CUDA(cudaMallocAsync(&d_rx, (nrx ? nrx : 3) * sizeof(float), st));
    if (nrx) NRT_CUDA(cudaMemcpyAsync(d_rx, coarse->rx.data(), nrx * sizeof(float), cudaMemcpyHostToDevice, st));
    P.rx = d_rx;
    nrt_refined_rec* o = nullptr;
    NRT_CUDA(cudaMallocAsync(&o, (size_t)(n_mine > 0 ? n_mine : 1) * sizeof(nrt_refined_rec), st));
    unsigned long long* ctr = nullptr;
    NRT_CUDA(cudaMallocAsync(&ctr, 4 * sizeof(unsigned long long), st));
    NRT_CUDA(cudaMemsetAsync(ctr, 0, 4 * sizeof(unsigned long long), st));
    P.out = o;
    P.n_out = ctr;
    P.work = ctr + 1;
    P.mls_cnt = d->counters ? ctr + 2 : nullptr;
    const bool timing = getenv("NRT_REFINE_TIMING") != nullptr && d->keep_invalid;
    if (timing) {
        NRT_CUDA(cudaMallocAsync(&P.cycles, (size_t)(n_mine > 0 ? n_mine : 1) * 8, st));
        NRT_CUDA(cudaMemsetAsync(P.cycles, 0, (size_t)(n_mine > 0 ? n_mine : 1) * 8, st));
        const unsigned long long zero[16] = {};
        NRT_CUDA(cudaMemcpyToSymbolAsync(g_dbg, zero, sizeof(zero), 0, cudaMemcpyHostToDevice, st));
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
    if (n_mine > 0) {
        if (warp_impl) k_refine_w<<<(unsigned)blocks, 32 * kWPB, smem_w, st>>>(P, scratch, mmax);
        else k_refine_b<<<(unsigned)blocks, 32 * NW, smem_b, st>>>(P, scratch);
        ::nrt::count_launch();
    }
    cudaEventRecord(e1, st);
    NRT_CUDA(cudaGetLastError());
    cudaFreeAsync(scratch, st);
    unsigned long long hctr[4] = {0, 0, 0, 0};
    NRT_CUDA(cudaMemcpyAsync(hctr, ctr, sizeof(hctr), cudaMemcpyDeviceToHost, st));
    NRT_CUDA(cudaStreamSynchronize(st));
    const unsigned long long n_ok = hctr[0];
    out->info.mls_value = hctr[2];
    out->info.mls_deriv = hctr[3];
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
        fprintf(stderr, "[nrt] refine (%s kernel): %lld paths, sum %.3g cycles, blocks %lld\n",
                warp_impl ? "warp" : "block", (long long)n_mine, (double)tot, (long long)blocks);
        unsigned long long dbg[16];
        cudaMemcpyFromSymbol(dbg, g_dbg, sizeof(dbg));
        fprintf(stderr, "[nrt]   warp cycles: prologue %.3g regather %.3g jacobian %.3g solve %.3g linesearch %.3g validity %.3g\n",
                (double)dbg[6], (double)dbg[8], (double)dbg[9], (double)dbg[10], (double)dbg[11], (double)dbg[7]);
        fprintf(stderr, "[nrt]   mls list %llu direct %llu, gathers %llu, GN iterations %llu, trials %llu\n",
                dbg[0], dbg[1], dbg[3], dbg[15], dbg[14]);
        fprintf(stderr, "[nrt]   avg cycles: mls list %.0f direct %.0f\n", (double)dbg[4] / (dbg[0] + 1),
                (double)dbg[5] / (dbg[1] + 1));
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
