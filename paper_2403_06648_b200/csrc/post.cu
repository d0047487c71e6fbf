// post.cu — post-processing of refined paths (PAPER §II-E, P:234-242;
// DESIGN.md readings R33-R36):
//   1. exact label of every reflection vertex = label of the nearest surfel within 2 r_s
//      (lowest id on ties; none -> the coarse label stays)       — k_relabel, one warp/vertex;
//   2. shortest path per (rx, interaction chain, labels)         — dedupe_refined (R28);
//   3. propagation-delay order (stable radix sort on the delay bits: ties keep key order);
//   4. greedy first-Fresnel-zone dedupe (Eq. 13): in delay order a path is dropped when it lies
//      inside the first Fresnel zones of an earlier kept path with the same rx and chain and
//      every pair of k-th rays is closer than the angle threshold.  Duplicates only arise
//      within a (rx, n_int, kinds) group, so the groups run in parallel (one warp each, members
//      in delay order, lanes over the group's earlier kept paths) — the same decisions as the
//      sequential walk over the whole delay-ordered list.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <cmath>

#include "internal.cuh"

namespace nrt {

namespace {

struct PostP {
    const uint2* hcell;
    const float4* hrec;
    const unsigned* hid;
    float ox, oy, oz, inv_hv;
    int hx, hy, hz;
    float box_r;     // 2 r_s + slack, for the cell range only
    double lim2;     // (2 r_s)^2
    double lambda, cos_max;
    double tx[3];
    const float* rx;
};

__device__ __forceinline__ double dot3d(const double a[3], const double b[3]) {
    return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
}

// step 1: warp w handles vertex slot (path w / 8, vertex w % 8)
__global__ void k_relabel(PostP P, nrt_refined_rec* r, int64_t n) {
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= n * NRT_MAX_INT) return;
    const int64_t i = w / NRT_MAX_INT;
    const int k = (int)(w % NRT_MAX_INT);
    if (k >= r[i].n_int || ((r[i].kinds >> k) & 1u)) return;
    const double x[3] = {r[i].v[k][0], r[i].v[k][1], r[i].v[k][2]};
    const int i0 = max(0, (int)floorf(((float)x[0] - P.box_r - P.ox) * P.inv_hv));
    const int i1 = min(P.hx - 1, (int)floorf(((float)x[0] + P.box_r - P.ox) * P.inv_hv));
    const int j0 = max(0, (int)floorf(((float)x[1] - P.box_r - P.oy) * P.inv_hv));
    const int j1 = min(P.hy - 1, (int)floorf(((float)x[1] + P.box_r - P.oy) * P.inv_hv));
    const int k0 = max(0, (int)floorf(((float)x[2] - P.box_r - P.oz) * P.inv_hv));
    const int k1 = min(P.hz - 1, (int)floorf(((float)x[2] + P.box_r - P.oz) * P.inv_hv));
    double bd = INFINITY;
    unsigned bid = 0xffffffffu;
    int blab = 0;
    for (int c = k0; c <= k1; ++c)
        for (int b = j0; b <= j1; ++b)
            for (int a = i0; a <= i1; ++a) {
                const uint2 rg = __ldg(&P.hcell[a + P.hx * (b + P.hy * c)]);
                for (unsigned q = rg.x + lane; q < rg.y; q += 32) {
                    const float4 A = __ldg(&P.hrec[2 * q]);
                    const double d[3] = {(double)A.x - x[0], (double)A.y - x[1], (double)A.z - x[2]};
                    const double d2 = dot3d(d, d);
                    if (!(d2 <= P.lim2)) continue;
                    const unsigned id = __ldg(&P.hid[q]);
                    if (d2 < bd || (d2 == bd && id < bid)) {
                        bd = d2;
                        bid = id;
                        blab = __float_as_int(__ldg(&P.hrec[2 * q + 1]).w);
                    }
                }
            }
    for (int o = 16; o > 0; o >>= 1) {  // lexicographic (d2, id) minimum over the warp
        const double od = __shfl_xor_sync(0xffffffffu, bd, o);
        const unsigned oid = __shfl_xor_sync(0xffffffffu, bid, o);
        const int ol = __shfl_xor_sync(0xffffffffu, blab, o);
        if (od < bd || (od == bd && oid < bid)) {
            bd = od;
            bid = oid;
            blab = ol;
        }
    }
    if (lane == 0 && bid != 0xffffffffu) r[i].label[k] = blab;
}

__global__ void k_delay_keys(const nrt_refined_rec* r, int64_t n, unsigned long long* key, unsigned* idx) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    key[i] = (unsigned long long)__double_as_longlong(r[i].delay);  // delay > 0: bit order = order
    idx[i] = (unsigned)i;
}

// group key of the t-th path in delay order
__global__ void k_group_keys(const nrt_refined_rec* r, const unsigned* perm_d, int64_t n, unsigned* g,
                             unsigned* t_out) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const nrt_refined_rec& c = r[perm_d[t]];
    g[t] = (c.rx << 16) | ((unsigned)c.n_int << 8) | (c.kinds & 0xffu);
    t_out[t] = (unsigned)t;
}

__global__ void k_group_heads(const unsigned* gs, int64_t n, unsigned char* head) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s < n) head[s] = (s == 0 || gs[s] != gs[s - 1]) ? 1 : 0;
}

__device__ void path_points(const PostP& P, const nrt_refined_rec& c, double I[NRT_MAX_INT + 2][3]) {
    for (int a = 0; a < 3; ++a) {
        I[0][a] = P.tx[a];
        I[c.n_int + 1][a] = (double)P.rx[3 * (size_t)c.rx + a];
    }
    for (int k = 0; k < c.n_int; ++k)
        for (int a = 0; a < 3; ++a) I[k + 1][a] = c.v[k][a];
}

// R36: is b a duplicate of the kept path a (same rx and chain)
__device__ bool fresnel_dup(const PostP& P, const nrt_refined_rec& a, const nrt_refined_rec& b) {
    double A[NRT_MAX_INT + 2][3], B[NRT_MAX_INT + 2][3];
    path_points(P, a, A);
    path_points(P, b, B);
    const int n = a.n_int;
    for (int k = 1; k <= n; ++k) {
        const double u1[3] = {A[k - 1][0] - A[k][0], A[k - 1][1] - A[k][1], A[k - 1][2] - A[k][2]};
        const double u2[3] = {A[k + 1][0] - A[k][0], A[k + 1][1] - A[k][1], A[k + 1][2] - A[k][2]};
        const double s1 = sqrt(dot3d(u1, u1)), s2 = sqrt(dot3d(u2, u2));
        const double psi2 = P.lambda * s1 * s2 / (s1 + s2);
        const double d[3] = {B[k][0] - A[k][0], B[k][1] - A[k][1], B[k][2] - A[k][2]};
        if (!(dot3d(d, d) <= psi2)) return false;
    }
    for (int k = 0; k <= n; ++k) {
        const double u[3] = {A[k + 1][0] - A[k][0], A[k + 1][1] - A[k][1], A[k + 1][2] - A[k][2]};
        const double w[3] = {B[k + 1][0] - B[k][0], B[k + 1][1] - B[k][1], B[k + 1][2] - B[k][2]};
        const double c = dot3d(u, w) / (sqrt(dot3d(u, u)) * sqrt(dot3d(w, w)));
        if (!(c > P.cos_max)) return false;
    }
    return true;
}

// step 4: warp per group; members s in [start, end) of the group-major order are in delay order
__global__ void k_fresnel(PostP P, const nrt_refined_rec* r, const unsigned* perm_d, const unsigned* tg,
                          const unsigned* gstart, int64_t ngroups, int64_t n, volatile unsigned char* keep_t) {
    const int64_t gi = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (gi >= ngroups) return;
    const int64_t s0 = gstart[gi], s1 = gi + 1 < ngroups ? (int64_t)gstart[gi + 1] : n;
    for (int64_t s = s0; s < s1; ++s) {
        const nrt_refined_rec& b = r[perm_d[tg[s]]];
        bool dup = false;
        for (int64_t q = s0 + lane; q < s; q += 32)
            if (keep_t[tg[q]] && fresnel_dup(P, r[perm_d[tg[q]]], b)) dup = true;
        dup = __any_sync(0xffffffffu, dup);
        if (lane == 0) keep_t[tg[s]] = dup ? 0 : 1;
        __syncwarp();
    }
}

__global__ void k_take_perm(const nrt_refined_rec* in, const unsigned* perm_d, const unsigned* sel_t,
                            int64_t m, nrt_refined_rec* out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) out[i] = in[perm_d[sel_t[i]]];
}

__global__ void k_ok_flags(const nrt_refined_rec* r, int64_t n, unsigned char* f) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) f[i] = r[i].status == NRT_REF_OK;
}

inline unsigned nb(int64_t n, int per = 256) { return (unsigned)((n + per - 1) / per); }

struct Bufs {  // stream-ordered frees on every exit path
    cudaStream_t st;
    std::vector<void*> p;
    template <class T>
    nrt_status get(T** out, size_t count) {
        void* q = nullptr;
        if (cudaMallocAsync(&q, (count ? count : 1) * sizeof(T), st) != cudaSuccess)
            return set_error(NRT_E_NOMEM, "post-processing buffer");
        p.push_back(q);
        *out = (T*)q;
        return NRT_OK;
    }
    ~Bufs() {
        for (void* q : p) cudaFreeAsync(q, st);
    }
};

}  // namespace

nrt_status postprocess(nrt_scene s, nrt_paths in, const nrt_post_desc* d, nrt_paths out, cudaStream_t st) {
    out->n = 0;
    out->d_rec = nullptr;
    const int64_t n0 = in->n;
    Bufs B{st, {}};
    // valid paths only
    nrt_refined_rec* work = nullptr;
    int64_t n = 0;
    {
        unsigned char* f = nullptr;
        int64_t* dn = nullptr;
        NRT_TRY(B.get(&work, n0));
        NRT_TRY(B.get(&f, n0));
        NRT_TRY(B.get(&dn, 1));
        if (n0 > 0) {
            k_ok_flags<<<nb(n0), 256, 0, st>>>((const nrt_refined_rec*)in->d_rec, n0, f);
            ::nrt::count_launch();
            size_t tb = 0;
            void* tmp = nullptr;
            cub::DeviceSelect::Flagged(nullptr, tb, (const nrt_refined_rec*)in->d_rec, f, work, dn, n0, st);
            NRT_TRY(B.get((char**)&tmp, tb));
            cub::DeviceSelect::Flagged(tmp, tb, (const nrt_refined_rec*)in->d_rec, f, work, dn, n0, st);
            NRT_CUDA(cudaMemcpyAsync(&n, dn, sizeof(n), cudaMemcpyDeviceToHost, st));
            NRT_CUDA(cudaStreamSynchronize(st));
        }
    }
    PostP P{};
    P.hcell = s->hcell;
    P.hrec = s->hrec;
    P.hid = s->hid;
    P.ox = s->org[0];
    P.oy = s->org[1];
    P.oz = s->org[2];
    P.inv_hv = s->inv_hv;
    P.hx = s->hdims[0];
    P.hy = s->hdims[1];
    P.hz = s->hdims[2];
    P.box_r = (float)(2.0 * d->r_s) + 1e-4f;
    P.lim2 = (2.0 * d->r_s) * (2.0 * d->r_s);
    P.lambda = d->lambda_m;
    {
        double sn_, cs;
        nrt_sincos(d->angle_deg * (kPi / 180.0), &sn_, &cs);
        P.cos_max = cs;
    }
    for (int a = 0; a < 3; ++a) P.tx[a] = in->tx[a];
    float* d_rx = nullptr;
    NRT_TRY(B.get(&d_rx, in->rx.size()));
    if (!in->rx.empty())
        NRT_CUDA(cudaMemcpyAsync(d_rx, in->rx.data(), in->rx.size() * sizeof(float), cudaMemcpyHostToDevice, st));
    P.rx = d_rx;
    if (n == 0) return NRT_OK;
    // 1. exact labels
    k_relabel<<<nb(n * NRT_MAX_INT * 32, 128), 128, 0, st>>>(P, work, n);
    ::nrt::count_launch();
    // 2. shortest per key (R28 with the exact labels)
    nrt_refined_rec* u = nullptr;
    NRT_TRY(B.get(&u, n));
    int64_t m = 0;
    NRT_TRY(dedupe_refined(work, n, u, &m, st));
    // 3. delay order
    unsigned long long *dk0 = nullptr, *dk1 = nullptr;
    unsigned *pi0 = nullptr, *perm_d = nullptr, *g0 = nullptr, *g1 = nullptr, *t0 = nullptr, *tg = nullptr;
    NRT_TRY(B.get(&dk0, m));
    NRT_TRY(B.get(&dk1, m));
    NRT_TRY(B.get(&pi0, m));
    NRT_TRY(B.get(&perm_d, m));
    NRT_TRY(B.get(&g0, m));
    NRT_TRY(B.get(&g1, m));
    NRT_TRY(B.get(&t0, m));
    NRT_TRY(B.get(&tg, m));
    k_delay_keys<<<nb(m), 256, 0, st>>>(u, m, dk0, pi0);
    ::nrt::count_launch();
    {
        size_t tb = 0, tb2 = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, dk0, dk1, pi0, perm_d, (int)m, 0, 64, st);
        cub::DeviceRadixSort::SortPairs(nullptr, tb2, g0, g1, t0, tg, (int)m, 0, 32, st);
        char* tmp = nullptr;
        NRT_TRY(B.get(&tmp, tb > tb2 ? tb : tb2));
        size_t t1 = tb;
        cub::DeviceRadixSort::SortPairs(tmp, t1, dk0, dk1, pi0, perm_d, (int)m, 0, 64, st);
        // groups (rx, n_int, kinds), members kept in delay order (stable sort)
        k_group_keys<<<nb(m), 256, 0, st>>>(u, perm_d, m, g0, t0);
        ::nrt::count_launch();
        size_t t2 = tb2;
        cub::DeviceRadixSort::SortPairs(tmp, t2, g0, g1, t0, tg, (int)m, 0, 32, st);
    }
    // group starts
    unsigned char* head = nullptr;
    unsigned *gstart = nullptr, *iota = nullptr;
    int64_t* d_ng = nullptr;
    NRT_TRY(B.get(&head, m));
    NRT_TRY(B.get(&gstart, m));
    NRT_TRY(B.get(&iota, m));
    NRT_TRY(B.get(&d_ng, 1));
    k_group_heads<<<nb(m), 256, 0, st>>>(g1, m, head);
    ::nrt::count_launch();
    int64_t ng = 0;
    {
        thrust::counting_iterator<unsigned> cnt(0);
        size_t tb = 0;
        cub::DeviceSelect::Flagged(nullptr, tb, cnt, head, gstart, d_ng, m, st);
        char* tmp = nullptr;
        NRT_TRY(B.get(&tmp, tb));
        cub::DeviceSelect::Flagged(tmp, tb, cnt, head, gstart, d_ng, m, st);
        NRT_CUDA(cudaMemcpyAsync(&ng, d_ng, sizeof(ng), cudaMemcpyDeviceToHost, st));
        NRT_CUDA(cudaStreamSynchronize(st));
    }
    // 4. greedy Fresnel dedupe per group
    unsigned char* keep_t = nullptr;
    NRT_TRY(B.get(&keep_t, m));
    NRT_CUDA(cudaMemsetAsync(keep_t, 0, m, st));
    k_fresnel<<<nb(ng * 32, 128), 128, 0, st>>>(P, u, perm_d, tg, gstart, ng, m, keep_t);
    ::nrt::count_launch();
    // compact in delay order
    unsigned* sel = nullptr;
    int64_t* d_nk = nullptr;
    NRT_TRY(B.get(&sel, m));
    NRT_TRY(B.get(&d_nk, 1));
    int64_t nk = 0;
    {
        thrust::counting_iterator<unsigned> cnt(0);
        size_t tb = 0;
        cub::DeviceSelect::Flagged(nullptr, tb, cnt, keep_t, sel, d_nk, m, st);
        char* tmp = nullptr;
        NRT_TRY(B.get(&tmp, tb));
        cub::DeviceSelect::Flagged(tmp, tb, cnt, keep_t, sel, d_nk, m, st);
        NRT_CUDA(cudaMemcpyAsync(&nk, d_nk, sizeof(nk), cudaMemcpyDeviceToHost, st));
        NRT_CUDA(cudaStreamSynchronize(st));
    }
    nrt_refined_rec* o = nullptr;
    NRT_CUDA(cudaMallocAsync(&o, (size_t)(nk > 0 ? nk : 1) * sizeof(nrt_refined_rec), st));
    if (nk > 0) {
        k_take_perm<<<nb(nk), 256, 0, st>>>(u, perm_d, sel, nk, o);
        ::nrt::count_launch();
    }
    NRT_CUDA(cudaGetLastError());
    NRT_CUDA(cudaStreamSynchronize(st));
    out->d_rec = o;
    out->n = nk;
    return NRT_OK;
}

}  // namespace nrt
