// dedupe.cu — A8 (coarse dedupe, R17, "only kappa shortest paths with a given label and
// interaction type combination are saved"), R14 (event dedupe) and R28 (refined dedupe).
//
// Exact keys (no hashing): the coarse key (rx, n_int, kinds, label[0..7]) packs into 124 bits
// (16 + 4 + 8 + 8x12), ordered most-significant first so that integer order = tuple order.
// Records are ordered by (key, L, ray id) with LSD passes of CUB's stable radix sort over an
// index permutation, then the first kappa of every key run are compacted in that order.
#include <cub/cub.cuh>

#include "internal.cuh"

namespace nrt {

namespace {

__global__ void k_coarse_keys(const nrt_coarse_rec* r, int64_t n, uint64_t* hi, uint64_t* lo,
                              uint64_t* lk, uint64_t* rid) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const nrt_coarse_rec& c = r[i];
    uint64_t L[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) L[k] = (uint64_t)(uint32_t)c.label[k] & 0xfffull;
    hi[i] = ((uint64_t)c.rx << 48) | ((uint64_t)c.n_int << 44) | ((uint64_t)(c.kinds & 0xff) << 36) |
            (L[0] << 24) | (L[1] << 12) | L[2];
    lo[i] = (L[3] << 52) | (L[4] << 40) | (L[5] << 28) | (L[6] << 16) | (L[7] << 4);
    lk[i] = (uint64_t)__float_as_uint(c.L);
    rid[i] = c.ray_id;
}

__global__ void k_event_keys(const nrt_event_rec* r, int64_t n, uint64_t* hi, uint64_t* lo,
                             uint64_t* dk, uint64_t* rid) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const nrt_event_rec& e = r[i];
    uint64_t L[7];
#pragma unroll
    for (int k = 0; k < 7; ++k) L[k] = (uint64_t)(uint32_t)e.label[k] & 0xfffull;
    hi[i] = ((uint64_t)e.n_hist << 60) | (L[0] << 48) | (L[1] << 36) | (L[2] << 24) |
            (L[3] << 12) | L[4];
    lo[i] = (L[5] << 52) | (L[6] << 40) | ((uint64_t)(e.edge & 0xfff) << 28) |
            ((uint64_t)(uint32_t)e.sbin & 0xfffffffull);
    dk[i] = (uint64_t)__float_as_uint(e.dist2);
    rid[i] = e.ray_id;
}

__global__ void k_refined_keys(const nrt_refined_rec* r, int64_t n, uint64_t* hi, uint64_t* lo,
                               uint64_t* lk, uint64_t* rid) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const nrt_refined_rec& c = r[i];
    uint64_t L[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) L[k] = (uint64_t)(uint32_t)c.label[k] & 0xfffull;
    hi[i] = ((uint64_t)c.rx << 48) | ((uint64_t)c.n_int << 44) | ((uint64_t)(c.kinds & 0xff) << 36) |
            (L[0] << 24) | (L[1] << 12) | L[2];
    lo[i] = (L[3] << 52) | (L[4] << 40) | (L[5] << 28) | (L[6] << 16) | (L[7] << 4);
    lk[i] = (uint64_t)__double_as_longlong(c.L);
    rid[i] = c.ray_id;
}

__global__ void k_iota(unsigned int* p, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = (unsigned)i;
}
__global__ void k_gather(const uint64_t* src, const unsigned int* perm, uint64_t* dst, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[perm[i]];
}
// head index of the key run containing sorted position i (0 if not a head)
__global__ void k_heads(const uint64_t* hi, const uint64_t* lo, const unsigned int* perm, int64_t n,
                        unsigned int* head) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    bool h = (i == 0) || hi[perm[i]] != hi[perm[i - 1]] || lo[perm[i]] != lo[perm[i - 1]];
    head[i] = h ? (unsigned)i : 0u;
}
__global__ void k_keep(const unsigned int* runhead, int64_t n, int32_t kappa, unsigned char* keep) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) keep[i] = ((int64_t)i - (int64_t)runhead[i]) < (int64_t)kappa ? 1 : 0;
}
template <class R>
__global__ void k_take(const R* in, const unsigned int* sel, int64_t m, R* out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) out[i] = in[sel[i]];
}

inline unsigned nblk(int64_t n) { return (unsigned)((n + 255) / 256); }

// order by keys[0] (most significant) .. keys[nk-1]; keep first kappa per (keys[0], keys[1])
template <class R>
nrt_status sort_unique(const R* in, int64_t n, uint64_t* keys[4], int32_t kappa, R* out,
                       int64_t* n_out, cudaStream_t st) {
    unsigned int *perm = nullptr, *perm2 = nullptr, *run = nullptr, *sel = nullptr;
    uint64_t *k1 = nullptr, *k2 = nullptr;
    unsigned char* keep = nullptr;
    int* nsel = nullptr;
    NRT_CUDA(cudaMallocAsync(&perm, n * 4, st));
    NRT_CUDA(cudaMallocAsync(&perm2, n * 4, st));
    NRT_CUDA(cudaMallocAsync(&run, n * 4, st));
    NRT_CUDA(cudaMallocAsync(&sel, n * 4, st));
    NRT_CUDA(cudaMallocAsync(&k1, n * 8, st));
    NRT_CUDA(cudaMallocAsync(&k2, n * 8, st));
    NRT_CUDA(cudaMallocAsync(&keep, n, st));
    NRT_CUDA(cudaMallocAsync(&nsel, sizeof(int), st));
    k_iota<<<nblk(n), 256, 0, st>>>(perm, n); ::nrt::count_launch();
    size_t tb = 0, tb2 = 0;
    void* tmp = nullptr;
    {
        cub::DoubleBuffer<uint64_t> kb(k1, k2);
        cub::DoubleBuffer<unsigned int> vb(perm, perm2);
        cub::DeviceRadixSort::SortPairs(nullptr, tb, kb, vb, (int)n, 0, 64, st);
        cub::DeviceScan::InclusiveScan(nullptr, tb2, run, run, cub::Max(), (int)n, st);
        if (tb2 > tb) tb = tb2;
        cub::DeviceSelect::Flagged(nullptr, tb2, perm, keep, sel, nsel, (int)n, st);
        if (tb2 > tb) tb = tb2;
    }
    NRT_CUDA(cudaMallocAsync(&tmp, tb, st));
    unsigned int* cur = perm;
    unsigned int* alt = perm2;
    for (int pass = 3; pass >= 0; --pass) {  // LSD: least significant key first
        k_gather<<<nblk(n), 256, 0, st>>>(keys[pass], cur, k1, n); ::nrt::count_launch();
        cub::DoubleBuffer<uint64_t> kb(k1, k2);
        cub::DoubleBuffer<unsigned int> vb(cur, alt);
        size_t t = tb;
        cub::DeviceRadixSort::SortPairs(tmp, t, kb, vb, (int)n, 0, 64, st);
        cur = vb.Current();
        alt = vb.Alternate();
        if (kb.Current() != k1) {  // keep k1 as the scratch for the next gather
            uint64_t* x = k1;
            k1 = k2;
            k2 = x;
        }
    }
    k_heads<<<nblk(n), 256, 0, st>>>(keys[0], keys[1], cur, n, run); ::nrt::count_launch();
    {
        size_t t = tb;
        cub::DeviceScan::InclusiveScan(tmp, t, run, run, cub::Max(), (int)n, st);
    }
    k_keep<<<nblk(n), 256, 0, st>>>(run, n, kappa, keep); ::nrt::count_launch();
    {
        size_t t = tb;
        cub::DeviceSelect::Flagged(tmp, t, cur, keep, sel, nsel, (int)n, st);
    }
    int m = 0;
    NRT_CUDA(cudaMemcpyAsync(&m, nsel, sizeof(int), cudaMemcpyDeviceToHost, st));
    NRT_CUDA(cudaStreamSynchronize(st));
    if (m > 0) {
        k_take<R><<<nblk(m), 256, 0, st>>>(in, sel, m, out);
        ::nrt::count_launch();
    }
    NRT_CUDA(cudaGetLastError());
    *n_out = m;
    cudaFreeAsync(perm, st);
    cudaFreeAsync(perm2, st);
    cudaFreeAsync(run, st);
    cudaFreeAsync(sel, st);
    cudaFreeAsync(k1, st);
    cudaFreeAsync(k2, st);
    cudaFreeAsync(keep, st);
    cudaFreeAsync(nsel, st);
    cudaFreeAsync(tmp, st);
    return NRT_OK;
}

}  // namespace

nrt_status dedupe_coarse(const nrt_coarse_rec* in, int64_t n, int32_t kappa, nrt_coarse_rec* out,
                         int64_t* n_out, cudaStream_t st) {
    *n_out = 0;
    if (n <= 0) return NRT_OK;
    uint64_t* k[4];
    for (int j = 0; j < 4; ++j) NRT_CUDA(cudaMallocAsync(&k[j], n * 8, st));
    k_coarse_keys<<<nblk(n), 256, 0, st>>>(in, n, k[0], k[1], k[2], k[3]); ::nrt::count_launch();
    NRT_CUDA(cudaGetLastError());
    nrt_status rc = sort_unique(in, n, k, kappa, out, n_out, st);
    for (int j = 0; j < 4; ++j) cudaFreeAsync(k[j], st);
    return rc;
}

nrt_status dedupe_events(const nrt_event_rec* in, int64_t n, nrt_event_rec* out, int64_t* n_out,
                         cudaStream_t st) {
    *n_out = 0;
    if (n <= 0) return NRT_OK;
    uint64_t* k[4];
    for (int j = 0; j < 4; ++j) NRT_CUDA(cudaMallocAsync(&k[j], n * 8, st));
    k_event_keys<<<nblk(n), 256, 0, st>>>(in, n, k[0], k[1], k[2], k[3]); ::nrt::count_launch();
    NRT_CUDA(cudaGetLastError());
    nrt_status rc = sort_unique(in, n, k, 1, out, n_out, st);
    for (int j = 0; j < 4; ++j) cudaFreeAsync(k[j], st);
    return rc;
}

nrt_status dedupe_refined(const nrt_refined_rec* in, int64_t n, nrt_refined_rec* out,
                          int64_t* n_out, cudaStream_t st) {
    *n_out = 0;
    if (n <= 0) return NRT_OK;
    uint64_t* k[4];
    for (int j = 0; j < 4; ++j) NRT_CUDA(cudaMallocAsync(&k[j], n * 8, st));
    k_refined_keys<<<nblk(n), 256, 0, st>>>(in, n, k[0], k[1], k[2], k[3]); ::nrt::count_launch();
    NRT_CUDA(cudaGetLastError());
    nrt_status rc = sort_unique(in, n, k, 1, out, n_out, st);
    for (int j = 0; j < 4; ++j) cudaFreeAsync(k[j], st);
    return rc;
}

}  // namespace nrt
