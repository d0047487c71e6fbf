// scene.cu — A1: GPU voxelisation of the oriented-surfel cloud.
//
// The paper forms a three-level voxel/subvoxel/AABB hierarchy for OptiX; B200
// has no RT cores, so the B200 build is one uniform fine grid walked by a 3D-DDA:
//   1. validate + pack surfels (p, r), (n, label); bounds by block reduction;
//   2. per surfel, the exact disk AABB half extent r*sqrt(1 - n_a^2/|n|^2) + pad gives the
//      overlapped cell box; counts -> CUB exclusive scan -> (Morton u64, id u32) pairs;
//   3. CUB radix sort by Morton code (stable: ids ascend within a cell);
//   4. records duplicated per cell, AoS 32 B {p, r^2 | n, id} in Morton order, plus a
//      dense (start, end) table indexed by the linear cell index (8 B per cell).
// Registering a surfel in every cell its padded AABB overlaps is what makes the DDA's
// nearest hit equal the brute-force global argmin.
#include <cub/cub.cuh>

#include <cmath>
#include <cstring>

#include "internal.cuh"

namespace nrt {

namespace {

__device__ __forceinline__ unsigned int f2ord(float f) {
    unsigned int u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__host__ __device__ inline float ord2f(unsigned int u) {
    unsigned int b = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
    float f;
    memcpy(&f, &b, 4);
    return f;
}

struct BuildIn {
    const float* p;
    const float* n;
    const float* r;
    float radius;
    const int32_t* label;
    int64_t count;
};

// validate + pack; bounds (ordered-int atomics); first bad index (atomicMin)
__global__ void k_pack(BuildIn in, float4* sp, float4* sn, unsigned int* bounds,
                       unsigned long long* bad, int* bad_kind, unsigned int* rmax) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
    float rm = 0.0f;
    if (i < in.count) {
        float px = in.p[3 * i], py = in.p[3 * i + 1], pz = in.p[3 * i + 2];
        float nx = in.n[3 * i], ny = in.n[3 * i + 1], nz = in.n[3 * i + 2];
        float r = in.r ? in.r[i] : in.radius;
        int32_t lab = in.label ? in.label[i] : 0;
        int kind = 0;
        if (!(isfinite(px) && isfinite(py) && isfinite(pz))) kind = 1;
        float nn = sqrtf((nx * nx + ny * ny) + nz * nz);
        if (!kind && !(fabsf(nn - 1.0f) <= 1e-3f)) kind = 2;
        if (!kind && !(r > 0.0f && isfinite(r))) kind = 3;
        if (!kind && (lab < 0 || lab >= 4096)) kind = 4;
        if (kind) {
            unsigned long long old = atomicMin(bad, (unsigned long long)i);
            if ((unsigned long long)i < old) atomicExch(bad_kind, kind);
        }
        sp[i] = make_float4(px, py, pz, r);
        sn[i] = make_float4(nx, ny, nz, __int_as_float(lab));
        mn[0] = mx[0] = px;
        mn[1] = mx[1] = py;
        mn[2] = mx[2] = pz;
        rm = r;
    }
    typedef cub::BlockReduce<float, 256> BR;
    __shared__ typename BR::TempStorage tmp;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        float v = BR(tmp).Reduce(mn[a], cub::Min());
        if (threadIdx.x == 0) atomicMin(&bounds[a], f2ord(v));
        __syncthreads();
        v = BR(tmp).Reduce(mx[a], cub::Max());
        if (threadIdx.x == 0) atomicMax(&bounds[3 + a], f2ord(v));
        __syncthreads();
    }
    float v = BR(tmp).Reduce(rm, cub::Max());
    if (threadIdx.x == 0) atomicMax(rmax, __float_as_uint(v));
}

// R6: pseudo-label = linear index of the 0.5 m cell of p relative to the bounds minimum
__global__ void k_pseudo_label(float4* sn, const float4* sp, int64_t n, float bx, float by,
                               float bz, int lx, int ly, unsigned long long* bad) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float4 p = sp[i];
    int ix = (int)floorf((p.x - bx) / 0.5f), iy = (int)floorf((p.y - by) / 0.5f),
        iz = (int)floorf((p.z - bz) / 0.5f);
    long long lab = (long long)ix + (long long)lx * ((long long)iy + (long long)ly * iz);
    if (lab < 0 || lab >= 4096) atomicMin(bad, (unsigned long long)i);
    sn[i].w = __int_as_float((int)lab);
}

struct Grid {
    float ox, oy, oz, v, inv_v, pad;
    int nx, ny, nz;
};

__device__ __forceinline__ void cell_box(const Grid& g, float4 p, float4 n, int lo[3], int hi[3]) {
    float nn = (n.x * n.x + n.y * n.y) + n.z * n.z;
    float c[3] = {p.x, p.y, p.z};
    float o[3] = {g.ox, g.oy, g.oz};
    float na[3] = {n.x, n.y, n.z};
    int dim[3] = {g.nx, g.ny, g.nz};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        float h = p.w * sqrtf(fmaxf(0.0f, 1.0f - (na[a] * na[a]) / nn)) * 1.0001f + g.pad;
        int l = (int)floorf((c[a] - h - o[a]) * g.inv_v);
        int u = (int)floorf((c[a] + h - o[a]) * g.inv_v);
        lo[a] = max(0, min(dim[a] - 1, l));
        hi[a] = max(0, min(dim[a] - 1, u));
    }
}

__global__ void k_count(Grid g, const float4* sp, const float4* sn, int64_t n, unsigned int* cnt) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int lo[3], hi[3];
    cell_box(g, sp[i], sn[i], lo, hi);
    cnt[i] = (unsigned)((hi[0] - lo[0] + 1) * (hi[1] - lo[1] + 1) * (hi[2] - lo[2] + 1));
}

__device__ __forceinline__ uint64_t spread3(uint64_t x) {
    x &= 0x1fffff;
    x = (x | x << 32) & 0x1f00000000ffffull;
    x = (x | x << 16) & 0x1f0000ff0000ffull;
    x = (x | x << 8) & 0x100f00f00f00f00full;
    x = (x | x << 4) & 0x10c30c30c30c30c3ull;
    x = (x | x << 2) & 0x1249249249249249ull;
    return x;
}
__device__ __forceinline__ uint64_t morton3(int x, int y, int z) {
    return spread3(x) | (spread3(y) << 1) | (spread3(z) << 2);
}
__device__ __forceinline__ int compact3(uint64_t x) {
    x &= 0x1249249249249249ull;
    x = (x ^ (x >> 2)) & 0x10c30c30c30c30c3ull;
    x = (x ^ (x >> 4)) & 0x100f00f00f00f00full;
    x = (x ^ (x >> 8)) & 0x1f0000ff0000ffull;
    x = (x ^ (x >> 16)) & 0x1f00000000ffffull;
    x = (x ^ (x >> 32)) & 0x1fffffull;
    return (int)x;
}

template <class K>  // Morton keys: 32 bits when 3 x bits-per-axis <= 32, else 64
__global__ void k_emit(Grid g, const float4* sp, const float4* sn, int64_t n,
                       const unsigned int* off, K* keys, unsigned int* vals) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int lo[3], hi[3];
    cell_box(g, sp[i], sn[i], lo, hi);
    unsigned int k = off[i];
    for (int z = lo[2]; z <= hi[2]; ++z)
        for (int y = lo[1]; y <= hi[1]; ++y)
            for (int x = lo[0]; x <= hi[0]; ++x) {
                keys[k] = (K)morton3(x, y, z);
                vals[k] = (unsigned)i;
                ++k;
            }
}

template <class K>
__global__ void k_records(Grid g, const K* keys, const unsigned int* ids, int64_t nref,
                          const float4* sp, const float4* sn, float4* rec, uint2* cell) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nref) return;
    unsigned id = ids[k];
    float4 p = sp[id], nv = sn[id];
    rec[2 * k] = make_float4(p.x, p.y, p.z, p.w);  // record carries r; the test squares it as the definition does
    rec[2 * k + 1] = make_float4(nv.x, nv.y, nv.z, __uint_as_float(id));
    const uint64_t key = (uint64_t)keys[k];
    bool first = (k == 0) || keys[k - 1] != key;
    bool last = (k == nref - 1) || keys[k + 1] != key;
    if (first || last) {
        int x = compact3(key), y = compact3(key >> 1), z = compact3(key >> 2);
        int64_t lin = (int64_t)x + (int64_t)g.nx * ((int64_t)y + (int64_t)g.ny * z);
        if (first) cell[lin].x = (unsigned)k;
        if (last) cell[lin].y = (unsigned)(k + 1);
    }
}

// Chebyshev distance field.  f = 0 on non-empty cells, kSkipCap elsewhere; one pass per axis:
// g(x) = min_{|s| <= cap} max(|s|, f(x + s e_axis)) — exact for the L-infinity metric because
// max distributes over min.
constexpr int kSkipCap = 24;
__global__ void k_occ(const uint2* cell, int64_t ncell, unsigned char* f) {
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncell) return;
    const uint2 r = cell[c];
    f[c] = r.y > r.x ? 0 : kSkipCap;
}
__global__ void k_cheb_pass(const unsigned char* f, unsigned char* g, int nx, int ny, int nz,
                            int axis) {
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t ncell = (int64_t)nx * ny * nz;
    if (c >= ncell) return;
    const int x = (int)(c % nx), y = (int)((c / nx) % ny), z = (int)(c / ((int64_t)nx * ny));
    const int pos = axis == 0 ? x : (axis == 1 ? y : z);
    const int len = axis == 0 ? nx : (axis == 1 ? ny : nz);
    const int64_t stride = axis == 0 ? 1 : (axis == 1 ? nx : (int64_t)nx * ny);
    int best = f[c];
    for (int s = 1; s < best && s <= kSkipCap; ++s) {
        int m = kSkipCap;
        if (pos - s >= 0) m = min(m, (int)f[c - s * stride]);
        if (pos + s < len) m = min(m, (int)f[c + s * stride]);
        best = min(best, max(s, m));
    }
    g[c] = (unsigned char)best;
}
__global__ void k_pack_skip(uint2* cell, int64_t ncell, const unsigned char* f) {
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncell) return;
    const uint2 r = cell[c];
    if (r.y > r.x) return;
    const unsigned D = f[c] < 1 ? 1u : (unsigned)f[c];
    cell[c] = make_uint2(D, D);  // empty: x == y == Chebyshev distance to non-empty (>= 1)
}

// home grid: key = linear index of the hv-cell containing p (each surfel exactly once)
__global__ void k_home_keys(const float4* sp, int64_t n, float ox, float oy, float oz, float inv_hv,
                            int hx, int hy, int hz, unsigned* keys, unsigned* vals) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float4 p = sp[i];
    const int x = min(hx - 1, max(0, (int)floorf((p.x - ox) * inv_hv)));
    const int y = min(hy - 1, max(0, (int)floorf((p.y - oy) * inv_hv)));
    const int z = min(hz - 1, max(0, (int)floorf((p.z - oz) * inv_hv)));
    keys[i] = (unsigned)(x + hx * (y + hy * z));
    vals[i] = (unsigned)i;
}
__global__ void k_home_records(const unsigned* keys, const unsigned* ids, int64_t n, const float4* sp,
                               const float4* sn, float4* hrec, uint2* hcell) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const unsigned id = ids[k];
    hrec[2 * k] = sp[id];
    hrec[2 * k + 1] = sn[id];
    const unsigned key = keys[k];
    if (k == 0 || keys[k - 1] != key) hcell[key].x = (unsigned)k;
    if (k == n - 1 || keys[k + 1] != key) hcell[key].y = (unsigned)(k + 1);
}

__global__ void k_home_counts(const uint2* hcell, int64_t nh, unsigned* cnt) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c > nh) return;
    cnt[c] = c < nh ? hcell[c].y - hcell[c].x : 0u;
}


// ---- NEXT-1 AABB primitives (DESIGN R40) ------------------------------------
// key of point i: the linear index of the a-cell holding it (division as the definition does)
__global__ void k_sdf_keys(const float4* sp, int64_t n, float ox, float oy, float oz, float a, int dx,
                           int dy, int dz, unsigned* keys, unsigned* vals) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float4 p = sp[i];
    const int cx = min(dx - 1, max(0, (int)floorf((p.x - ox) / a)));
    const int cy = min(dy - 1, max(0, (int)floorf((p.y - oy) / a)));
    const int cz = min(dz - 1, max(0, (int)floorf((p.z - oz) / a)));
    keys[i] = (unsigned)((int64_t)cx + (int64_t)dx * ((int64_t)cy + (int64_t)dy * cz));
    vals[i] = (unsigned)i;
}
// points in (cell, id) order: (p, 0), (n, id bits)
__global__ void k_sdf_pts(const unsigned* ids, int64_t n, const float4* sp, const float4* sn, float4* pts) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const unsigned id = ids[k];
    const float4 p = sp[id], q = sn[id];
    pts[2 * k] = make_float4(p.x, p.y, p.z, 0.0f);
    pts[2 * k + 1] = make_float4(q.x, q.y, q.z, __uint_as_float(id));
}
// R40: AABB j = its points' extent per axis, or the cell's full extent where that exceeds a/2
__global__ void k_sdf_boxes(const unsigned* cells, const unsigned* off, int64_t na, const float4* pts,
                            float ox, float oy, float oz, float a, int dx, int dy, float4* box) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= na) return;
    const unsigned c = cells[j], k0 = off[j], k1 = off[j + 1];
    const int ci[3] = {(int)(c % (unsigned)dx), (int)((c / (unsigned)dx) % (unsigned)dy),
                       (int)(c / ((unsigned)dx * (unsigned)dy))};
    const float org[3] = {ox, oy, oz};
    float lo[3], hi[3];
    for (int k = 0; k < 3; ++k) {
        float l = INFINITY, h = -INFINITY;
        for (unsigned t = k0; t < k1; ++t) {
            const float4 p = pts[2 * t];
            const float v = k == 0 ? p.x : (k == 1 ? p.y : p.z);
            if (v < l) l = v;
            if (v > h) h = v;
        }
        if (h - l > 0.5f * a) {
            l = org[k] + (float)ci[k] * a;
            h = org[k] + (float)(ci[k] + 1) * a;
        }
        lo[k] = l;
        hi[k] = h;
    }
    box[2 * j] = make_float4(lo[0], lo[1], lo[2], __uint_as_float(k0));
    box[2 * j + 1] = make_float4(hi[0], hi[1], hi[2], __uint_as_float(k1));
}
// cell -> point range of its AABB (NEXT-4 neighbourhood normals)
__global__ void k_sdf_crange(const unsigned* cells, const float4* box, int64_t na, uint2* crange) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= na) return;
    crange[cells[j]] = make_uint2(__float_as_uint(box[2 * j].w), __float_as_uint(box[2 * j + 1].w));
}
// traversal grid: the cells the padded AABB overlaps
struct SdfGrid {
    float ox, oy, oz, inv_a, pad;
    int nx, ny, nz;
};
__device__ __forceinline__ void sdf_cell_box(const SdfGrid& g, const float4* box, int64_t j, int lo[3],
                                             int hi[3]) {
    const float4 L = box[2 * j], H = box[2 * j + 1];
    const float l[3] = {L.x, L.y, L.z}, h[3] = {H.x, H.y, H.z}, o[3] = {g.ox, g.oy, g.oz};
    const int dim[3] = {g.nx, g.ny, g.nz};
    for (int k = 0; k < 3; ++k) {
        lo[k] = max(0, min(dim[k] - 1, (int)floorf((l[k] - g.pad - o[k]) * g.inv_a)));
        hi[k] = max(0, min(dim[k] - 1, (int)floorf((h[k] + g.pad - o[k]) * g.inv_a)));
    }
}
__global__ void k_sdf_reg_count(SdfGrid g, const float4* box, int64_t na, unsigned* cnt) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= na) return;
    int lo[3], hi[3];
    sdf_cell_box(g, box, j, lo, hi);
    cnt[j] = (unsigned)((hi[0] - lo[0] + 1) * (hi[1] - lo[1] + 1) * (hi[2] - lo[2] + 1));
}
__global__ void k_sdf_reg_emit(SdfGrid g, const float4* box, int64_t na, const unsigned* off, unsigned* keys,
                               unsigned* vals) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= na) return;
    int lo[3], hi[3];
    sdf_cell_box(g, box, j, lo, hi);
    unsigned k = off[j];
    for (int z = lo[2]; z <= hi[2]; ++z)
        for (int y = lo[1]; y <= hi[1]; ++y)
            for (int x = lo[0]; x <= hi[0]; ++x) {
                keys[k] = (unsigned)(x + g.nx * (y + g.ny * z));
                vals[k] = (unsigned)j;
                ++k;
            }
}
__global__ void k_sdf_reg_ranges(const unsigned* keys, int64_t nr, uint2* gcell) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nr) return;
    const unsigned key = keys[k];
    if (k == 0 || keys[k - 1] != key) gcell[key].x = (unsigned)k;
    if (k == nr - 1 || keys[k + 1] != key) gcell[key].y = (unsigned)(k + 1);
}

template <class T>
nrt_status dmalloc(T** p, size_t count, cudaStream_t st) {
    if (count == 0) count = 1;
    NRT_CUDA(cudaMallocAsync((void**)p, count * sizeof(T), st));
    return NRT_OK;
}

}  // namespace

// (cell key, surfel id) pairs -> radix sort -> records + cell table.  Keys are 32-bit when the
// Morton code fits (3 x bits <= 32: grids up to 1024 cells per axis), halving the key traffic
// of the sort; the order (and hence every record) is the same either way.
template <class K>
static nrt_status sort_records(const Grid& g, nrt_scene S, int64_t n, const unsigned* off, int64_t nref,
                               int64_t ncell, int bits, cudaStream_t st) {
    const unsigned nb = (unsigned)((n + 255) / 256);
    K *k0 = nullptr, *k1 = nullptr;
    unsigned int *v0 = nullptr, *v1 = nullptr;
    NRT_TRY(dmalloc(&k0, nref, st));
    NRT_TRY(dmalloc(&k1, nref, st));
    NRT_TRY(dmalloc(&v0, nref, st));
    NRT_TRY(dmalloc(&v1, nref, st));
    k_emit<K><<<nb, 256, 0, st>>>(g, S->sp, S->sn, n, off, k0, v0); ::nrt::count_launch();
    NRT_CUDA(cudaGetLastError());
    cub::DoubleBuffer<K> kb(k0, k1);
    cub::DoubleBuffer<unsigned int> vb(v0, v1);
    size_t tb = 0;
    void* tmp = nullptr;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, kb, vb, (int)nref, 0, 3 * bits, st);
    NRT_CUDA(cudaMallocAsync(&tmp, tb, st));
    cub::DeviceRadixSort::SortPairs(tmp, tb, kb, vb, (int)nref, 0, 3 * bits, st);
    cudaFreeAsync(tmp, st);
    NRT_TRY(dmalloc(&S->rec, 2 * nref, st));
    NRT_TRY(dmalloc(&S->cell, ncell, st));
    NRT_CUDA(cudaMemsetAsync(S->cell, 0, ncell * sizeof(uint2), st));
    k_records<K><<<(unsigned)((nref + 255) / 256), 256, 0, st>>>(g, kb.Current(), vb.Current(), nref,
                                                                S->sp, S->sn, S->rec, S->cell);
    ::nrt::count_launch();
    NRT_CUDA(cudaGetLastError());
    cudaFreeAsync(k0, st);
    cudaFreeAsync(k1, st);
    cudaFreeAsync(v0, st);
    cudaFreeAsync(v1, st);
    return NRT_OK;
}


static int bits_for(int64_t n) {
    int b = 1;
    while (((int64_t)1 << b) < n) ++b;
    return b;
}

// NEXT-1: AABB primitives (R40) + their traversal grid.  org = the points'
// minimum, dims = floor((max - org) / a) + 1, cell of p = floor((p - org) / a) clamped, as
// the definition (oracle/sdf.c) states them.
static nrt_status sdf_build(nrt_scene S, float a, const float bmin[3], const float bmax[3], cudaStream_t st) {
    const int64_t n = S->n;
    const unsigned nb = (unsigned)((n + 255) / 256);
    int dims[3];
    int64_t ncell = 1;
    for (int k = 0; k < 3; ++k) {
        const float q = floorf((bmax[k] - bmin[k]) / a);
        if (!(q < (float)(1 << 20))) return set_error(NRT_E_INVALID, "sdf_cell too small for the scene");
        dims[k] = (int)q + 1;
        ncell *= dims[k] + 2;
    }
    if (ncell >= ((int64_t)1 << 31)) return set_error(NRT_E_INVALID, "sdf grid has >= 2^31 cells");
    S->sdf_a = a;
    for (int k = 0; k < 3; ++k) {
        S->sdf_org[k] = bmin[k];
        S->sdf_bmax[k] = bmax[k];
        S->sdf_dims[k] = dims[k];
        S->sdf_gorg[k] = bmin[k] - a;
        S->sdf_gdims[k] = dims[k] + 2;
    }
    float ext = 0.0f;
    for (int k = 0; k < 3; ++k) ext = fmaxf(ext, fmaxf(fabsf(bmin[k]), fabsf(bmax[k])));
    S->sdf_pad = fmaxf(fmaxf(1e-3f * a, 2e-5f), 4e-6f * ext);
    // (cell, id) pairs, stable radix sort: ids ascend within a cell
    unsigned *k0 = nullptr, *k1 = nullptr, *v0 = nullptr, *v1 = nullptr;
    NRT_TRY(dmalloc(&k0, n, st));
    NRT_TRY(dmalloc(&k1, n, st));
    NRT_TRY(dmalloc(&v0, n, st));
    NRT_TRY(dmalloc(&v1, n, st));
    k_sdf_keys<<<nb, 256, 0, st>>>(S->sp, n, bmin[0], bmin[1], bmin[2], a, dims[0], dims[1], dims[2], k0, v0);
    ::nrt::count_launch();
    const int cbits = bits_for((int64_t)dims[0] * dims[1] * dims[2]);
    cub::DoubleBuffer<unsigned> kb(k0, k1), vb(v0, v1);
    size_t tb = 0;
    void* tmp = nullptr;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, kb, vb, (int)n, 0, cbits, st);
    NRT_CUDA(cudaMallocAsync(&tmp, tb, st));
    cub::DeviceRadixSort::SortPairs(tmp, tb, kb, vb, (int)n, 0, cbits, st);
    cudaFreeAsync(tmp, st);
    NRT_TRY(dmalloc(&S->sdf_pts, 2 * n, st));
    k_sdf_pts<<<nb, 256, 0, st>>>(vb.Current(), n, S->sp, S->sn, S->sdf_pts);
    ::nrt::count_launch();
    // runs of equal cells -> AABBs (cell, first point, count)
    unsigned *cells = nullptr, *cnt = nullptr, *off = nullptr;
    int64_t* nruns = nullptr;
    NRT_TRY(dmalloc(&cells, n, st));
    NRT_TRY(dmalloc(&cnt, n + 1, st));
    NRT_TRY(dmalloc(&off, n + 1, st));
    NRT_TRY(dmalloc(&nruns, 1, st));
    tb = 0;
    cub::DeviceRunLengthEncode::Encode(nullptr, tb, kb.Current(), cells, cnt, nruns, (int64_t)n, st);
    NRT_CUDA(cudaMallocAsync(&tmp, tb, st));
    cub::DeviceRunLengthEncode::Encode(tmp, tb, kb.Current(), cells, cnt, nruns, (int64_t)n, st);
    cudaFreeAsync(tmp, st);
    int64_t na = 0;
    NRT_CUDA(cudaMemcpyAsync(&na, nruns, 8, cudaMemcpyDeviceToHost, st));
    NRT_CUDA(cudaStreamSynchronize(st));
    S->n_aabb = na;
    NRT_CUDA(cudaMemsetAsync(cnt + na, 0, 4, st));
    tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, off, (int)(na + 1), st);
    NRT_CUDA(cudaMallocAsync(&tmp, tb, st));
    cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, off, (int)(na + 1), st);
    cudaFreeAsync(tmp, st);
    NRT_TRY(dmalloc(&S->sdf_box, 2 * na, st));
    const unsigned ab = (unsigned)((na + 255) / 256);
    k_sdf_boxes<<<ab, 256, 0, st>>>(cells, off, na, S->sdf_pts, bmin[0], bmin[1], bmin[2], a, dims[0], dims[1],
                                    S->sdf_box);
    ::nrt::count_launch();
    NRT_CUDA(cudaGetLastError());
    S->sdf_acell = cells;  // [na] cell of each AABB (the tail past na is unused)
    {
        const int64_t nc = (int64_t)dims[0] * dims[1] * dims[2];
        NRT_TRY(dmalloc(&S->sdf_crange, nc, st));
        NRT_CUDA(cudaMemsetAsync(S->sdf_crange, 0, nc * sizeof(uint2), st));
        k_sdf_crange<<<ab, 256, 0, st>>>(cells, S->sdf_box, na, S->sdf_crange);
        ::nrt::count_launch();
    }
    cudaFreeAsync(k0, st);
    cudaFreeAsync(k1, st);
    cudaFreeAsync(v0, st);
    cudaFreeAsync(v1, st);
    // traversal grid: every AABB in all cells its padded box overlaps
    SdfGrid g;
    g.ox = S->sdf_gorg[0];
    g.oy = S->sdf_gorg[1];
    g.oz = S->sdf_gorg[2];
    g.inv_a = 1.0f / a;
    g.pad = S->sdf_pad;
    g.nx = S->sdf_gdims[0];
    g.ny = S->sdf_gdims[1];
    g.nz = S->sdf_gdims[2];
    k_sdf_reg_count<<<ab, 256, 0, st>>>(g, S->sdf_box, na, cnt);
    ::nrt::count_launch();
    NRT_CUDA(cudaMemsetAsync(cnt + na, 0, 4, st));
    tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, off, (int)(na + 1), st);
    NRT_CUDA(cudaMallocAsync(&tmp, tb, st));
    cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, off, (int)(na + 1), st);
    cudaFreeAsync(tmp, st);
    unsigned nr32 = 0;
    NRT_CUDA(cudaMemcpyAsync(&nr32, off + na, 4, cudaMemcpyDeviceToHost, st));
    NRT_CUDA(cudaStreamSynchronize(st));
    const int64_t nr = nr32;
    S->n_aref = nr;
    NRT_TRY(dmalloc(&k0, nr, st));
    NRT_TRY(dmalloc(&k1, nr, st));
    NRT_TRY(dmalloc(&v0, nr, st));
    NRT_TRY(dmalloc(&v1, nr, st));
    k_sdf_reg_emit<<<ab, 256, 0, st>>>(g, S->sdf_box, na, off, k0, v0);
    ::nrt::count_launch();
    cub::DoubleBuffer<unsigned> rkb(k0, k1), rvb(v0, v1);
    const int gbits = bits_for(ncell);
    tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, rkb, rvb, (int)nr, 0, gbits, st);
    NRT_CUDA(cudaMallocAsync(&tmp, tb, st));
    cub::DeviceRadixSort::SortPairs(tmp, tb, rkb, rvb, (int)nr, 0, gbits, st);
    cudaFreeAsync(tmp, st);
    NRT_TRY(dmalloc(&S->sdf_gcell, ncell, st));
    NRT_CUDA(cudaMemsetAsync(S->sdf_gcell, 0, ncell * sizeof(uint2), st));
    k_sdf_reg_ranges<<<(unsigned)((nr + 255) / 256), 256, 0, st>>>(rkb.Current(), nr, S->sdf_gcell);
    ::nrt::count_launch();
    S->sdf_aref = rvb.Current();
    cudaFreeAsync(rvb.Current() == v0 ? v1 : v0, st);
    cudaFreeAsync(k0, st);
    cudaFreeAsync(k1, st);
    cudaFreeAsync(cnt, st);
    cudaFreeAsync(off, st);
    cudaFreeAsync(nruns, st);
    // empty-space skip (Chebyshev distance), as for the surfel grid
    {
        unsigned char *f0 = nullptr, *f1 = nullptr;
        NRT_TRY(dmalloc(&f0, ncell, st));
        NRT_TRY(dmalloc(&f1, ncell, st));
        const unsigned cb = (unsigned)((ncell + 255) / 256);
        k_occ<<<cb, 256, 0, st>>>(S->sdf_gcell, ncell, f0); ::nrt::count_launch();
        k_cheb_pass<<<cb, 256, 0, st>>>(f0, f1, g.nx, g.ny, g.nz, 2); ::nrt::count_launch();
        k_cheb_pass<<<cb, 256, 0, st>>>(f1, f0, g.nx, g.ny, g.nz, 1); ::nrt::count_launch();
        k_cheb_pass<<<cb, 256, 0, st>>>(f0, f1, g.nx, g.ny, g.nz, 0); ::nrt::count_launch();
        k_pack_skip<<<cb, 256, 0, st>>>(S->sdf_gcell, ncell, f1); ::nrt::count_launch();
        NRT_CUDA(cudaGetLastError());
        cudaFreeAsync(f0, st);
        cudaFreeAsync(f1, st);
    }
    return NRT_OK;
}

static nrt_status build_impl(const nrt_scene_desc* D, nrt_scene S, cudaStream_t st) {
    const int64_t n = D->n;
    const unsigned nb = (unsigned)((n + 255) / 256);
    // ---- stage inputs on the device
    const float *dp = D->points, *dn = D->normals, *dr = D->radii;
    const int32_t* dl = D->labels;
    float *tp = nullptr, *tn = nullptr, *tr = nullptr;
    int32_t* tl = nullptr;
    if (D->mem == NRT_MEM_HOST) {
        NRT_TRY(dmalloc(&tp, 3 * n, st));
        NRT_TRY(dmalloc(&tn, 3 * n, st));
        NRT_CUDA(cudaMemcpyAsync(tp, D->points, 12 * n, cudaMemcpyHostToDevice, st));
        NRT_CUDA(cudaMemcpyAsync(tn, D->normals, 12 * n, cudaMemcpyHostToDevice, st));
        dp = tp;
        dn = tn;
        if (D->radii) {
            NRT_TRY(dmalloc(&tr, n, st));
            NRT_CUDA(cudaMemcpyAsync(tr, D->radii, 4 * n, cudaMemcpyHostToDevice, st));
            dr = tr;
        }
        if (D->labels) {
            NRT_TRY(dmalloc(&tl, n, st));
            NRT_CUDA(cudaMemcpyAsync(tl, D->labels, 4 * n, cudaMemcpyHostToDevice, st));
            dl = tl;
        }
    }
    NRT_TRY(dmalloc(&S->sp, n, st));
    NRT_TRY(dmalloc(&S->sn, n, st));
    NRT_TRY(dmalloc(&S->label, n, st));
    // scratch: bounds[6], rmax, bad, bad_kind
    struct Scratch {
        unsigned int bounds[6];
        unsigned int rmax;
        int bad_kind;
        unsigned long long bad;
    };
    Scratch h{}, *ds = nullptr;
    for (int a = 0; a < 3; ++a) {
        h.bounds[a] = 0xffffffffu;
        h.bounds[3 + a] = 0u;
    }
    h.rmax = 0;
    h.bad_kind = 0;
    h.bad = ~0ull;
    NRT_TRY(dmalloc(&ds, 1, st));
    NRT_CUDA(cudaMemcpyAsync(ds, &h, sizeof(h), cudaMemcpyHostToDevice, st));
    BuildIn in{dp, dn, dr, D->radius, dl, n};
    k_pack<<<nb, 256, 0, st>>>(in, S->sp, S->sn, ds->bounds, &ds->bad, &ds->bad_kind, &ds->rmax); ::nrt::count_launch();
    NRT_CUDA(cudaGetLastError());
    NRT_CUDA(cudaMemcpyAsync(&h, ds, sizeof(h), cudaMemcpyDeviceToHost, st));
    NRT_CUDA(cudaStreamSynchronize(st));
    cudaFreeAsync(tp, st);
    cudaFreeAsync(tn, st);
    cudaFreeAsync(tr, st);
    cudaFreeAsync(tl, st);
    if (h.bad != ~0ull) {
        static const char* what[] = {"", "non-finite position", "normal not unit (|n|-1 > 1e-3)",
                                     "radius <= 0 or non-finite", "label outside [0,4096)"};
        cudaFreeAsync(ds, st);
        return set_error(NRT_E_INVALID, "surfel %llu: %s", h.bad, what[h.bad_kind & 7]);
    }
    float bmin[3], bmax[3];
    for (int a = 0; a < 3; ++a) {
        bmin[a] = ord2f(h.bounds[a]);
        bmax[a] = ord2f(h.bounds[3 + a]);
    }
    memcpy(&S->r_max, &h.rmax, 4);
    {
        // FP32 error of |q| (either form) is a few ulp of the coordinates; 25x margin
        float ext = 0.0f;
        for (int a = 0; a < 3; ++a) ext = fmaxf(ext, fmaxf(fabsf(bmin[a]), fabsf(bmax[a])));
        S->slack = fmaxf(1e-4f, 4e-6f * ext);
    }
    if (!dl) {  // R6 pseudo-labels
        int lx = (int)floorf((bmax[0] - bmin[0]) / 0.5f) + 1;
        int ly = (int)floorf((bmax[1] - bmin[1]) / 0.5f) + 1;
        h.bad = ~0ull;
        NRT_CUDA(cudaMemcpyAsync(&ds->bad, &h.bad, 8, cudaMemcpyHostToDevice, st));
        k_pseudo_label<<<nb, 256, 0, st>>>(S->sn, S->sp, n, bmin[0], bmin[1], bmin[2], lx, ly,
                                           &ds->bad); ::nrt::count_launch();
        NRT_CUDA(cudaMemcpyAsync(&h.bad, &ds->bad, 8, cudaMemcpyDeviceToHost, st));
        NRT_CUDA(cudaStreamSynchronize(st));
        if (h.bad != ~0ull) {
            cudaFreeAsync(ds, st);
            return set_error(NRT_E_INVALID, "pseudo-label of surfel %llu exceeds 4095 (scene too "
                             "large for 0.5 m pseudo-labels; pass labels)", h.bad);
        }
    }
    cudaFreeAsync(ds, st);
    // ---- grid: origin = bmin - (ceil(r_max/v) + 1.5) v so every disk lies inside the grid
    // and axis-aligned walls sit mid-cell; covers bmax + the same margin.
    const float v = D->voxel_size;
    Grid g;
    g.v = v;
    g.inv_v = 1.0f / v;
    g.pad = fmaxf(1e-3f * v, 2e-5f);
    const float margin = (ceilf(S->r_max / v) + 1.5f) * v;
    g.ox = bmin[0] - margin;
    g.oy = bmin[1] - margin;
    g.oz = bmin[2] - margin;
    float o3[3] = {g.ox, g.oy, g.oz};
    int dims[3];
    for (int a = 0; a < 3; ++a) {
        double ext = ((double)bmax[a] + (double)margin - (double)o3[a]) / v;
        dims[a] = (int)ceil(ext) + 1;
        if (dims[a] < 1) dims[a] = 1;
        if (dims[a] > (1 << 20)) return set_error(NRT_E_INVALID, "grid too large: voxel too small");
    }
    g.nx = dims[0];
    g.ny = dims[1];
    g.nz = dims[2];
    const int64_t ncell = (int64_t)dims[0] * dims[1] * dims[2];
    if (ncell > (int64_t)1 << 31) return set_error(NRT_E_INVALID, "grid has > 2^31 cells");
    S->ncell = ncell;
    memcpy(S->dims, dims, sizeof(dims));
    memcpy(S->org, o3, sizeof(o3));
    S->v = v;
    S->inv_v = g.inv_v;
    S->pad = g.pad;
    // ---- counts, offsets
    unsigned int *cnt = nullptr, *off = nullptr;
    NRT_TRY(dmalloc(&cnt, n + 1, st));
    NRT_TRY(dmalloc(&off, n + 1, st));
    k_count<<<nb, 256, 0, st>>>(g, S->sp, S->sn, n, cnt); ::nrt::count_launch();
    NRT_CUDA(cudaGetLastError());
    NRT_CUDA(cudaMemsetAsync(cnt + n, 0, 4, st));
    size_t tb = 0;
    void* tmp = nullptr;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, off, n + 1, st);
    NRT_CUDA(cudaMallocAsync(&tmp, tb, st));
    cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, off, n + 1, st);
    cudaFreeAsync(tmp, st);
    unsigned int nref32 = 0;
    NRT_CUDA(cudaMemcpyAsync(&nref32, off + n, 4, cudaMemcpyDeviceToHost, st));
    NRT_CUDA(cudaStreamSynchronize(st));
    const int64_t nref = nref32;
    S->nref = nref;
    // ---- pairs, sort
    {
        int maxd = dims[0] > dims[1] ? dims[0] : dims[1];
        maxd = maxd > dims[2] ? maxd : dims[2];
        int bits = 1;
        while ((1 << bits) < maxd) ++bits;
        NRT_TRY(3 * bits <= 32 ? sort_records<uint32_t>(g, S, n, off, nref, ncell, bits, st)
                               : sort_records<uint64_t>(g, S, n, off, nref, ncell, bits, st));
    }
    cudaFreeAsync(cnt, st);
    cudaFreeAsync(off, st);
    // ---- empty-space skip field (the paper's "march distance", P:154 / P:281): Chebyshev
    // distance (in cells, capped) from every empty cell to the nearest non-empty one, computed
    // exactly by three separable min-max passes, then packed into empty entries as (D, D).
    {
        unsigned char *f0 = nullptr, *f1 = nullptr;
        NRT_TRY(dmalloc(&f0, ncell, st));
        NRT_TRY(dmalloc(&f1, ncell, st));
        const unsigned cb = (unsigned)((ncell + 255) / 256);
        k_occ<<<cb, 256, 0, st>>>(S->cell, ncell, f0); ::nrt::count_launch();
        k_cheb_pass<<<cb, 256, 0, st>>>(f0, f1, g.nx, g.ny, g.nz, 2); ::nrt::count_launch();
        k_cheb_pass<<<cb, 256, 0, st>>>(f1, f0, g.nx, g.ny, g.nz, 1); ::nrt::count_launch();
        k_cheb_pass<<<cb, 256, 0, st>>>(f0, f1, g.nx, g.ny, g.nz, 0); ::nrt::count_launch();
        k_pack_skip<<<cb, 256, 0, st>>>(S->cell, ncell, f1); ::nrt::count_launch();
        NRT_CUDA(cudaGetLastError());
        cudaFreeAsync(f0, st);
        cudaFreeAsync(f1, st);
    }
    // ---- home grid (refinement neighbourhoods): cell 2v, one record per surfel
    {
        S->hv = 2.0f * v;
        S->inv_hv = 1.0f / S->hv;
        for (int a = 0; a < 3; ++a) S->hdims[a] = (dims[a] + 1) / 2;
        const int64_t nh = (int64_t)S->hdims[0] * S->hdims[1] * S->hdims[2];
        unsigned *hk0 = nullptr, *hk1 = nullptr, *hv0 = nullptr, *hv1 = nullptr;
        NRT_TRY(dmalloc(&hk0, n, st));
        NRT_TRY(dmalloc(&hk1, n, st));
        NRT_TRY(dmalloc(&hv0, n, st));
        NRT_TRY(dmalloc(&hv1, n, st));
        k_home_keys<<<nb, 256, 0, st>>>(S->sp, n, g.ox, g.oy, g.oz, S->inv_hv, S->hdims[0], S->hdims[1],
                                        S->hdims[2], hk0, hv0);
        ::nrt::count_launch();
        int hbits = 1;
        while (((int64_t)1 << hbits) < nh) ++hbits;
        cub::DoubleBuffer<unsigned> hkb(hk0, hk1), hvb(hv0, hv1);
        tb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, hkb, hvb, (int)n, 0, hbits, st);
        NRT_CUDA(cudaMallocAsync(&tmp, tb, st));
        cub::DeviceRadixSort::SortPairs(tmp, tb, hkb, hvb, (int)n, 0, hbits, st);
        cudaFreeAsync(tmp, st);
        NRT_TRY(dmalloc(&S->hrec, 2 * n, st));
        NRT_TRY(dmalloc(&S->hcell, nh, st));
        NRT_CUDA(cudaMemsetAsync(S->hcell, 0, nh * sizeof(uint2), st));
        k_home_records<<<nb, 256, 0, st>>>(hkb.Current(), hvb.Current(), n, S->sp, S->sn, S->hrec,
                                           S->hcell);
        ::nrt::count_launch();
        NRT_CUDA(cudaGetLastError());
        // offsets of every home cell (empty ones included): runs of consecutive cells are
        // contiguous record ranges (refinement's direct neighbourhood scans walk cell rows)
        {
            unsigned* cnt = nullptr;
            NRT_TRY(dmalloc(&cnt, nh + 1, st));
            NRT_TRY(dmalloc(&S->hoff, nh + 1, st));
            k_home_counts<<<(unsigned)((nh + 256) / 256), 256, 0, st>>>(S->hcell, nh, cnt);
            ::nrt::count_launch();
            size_t tbs = 0;
            cub::DeviceScan::ExclusiveSum(nullptr, tbs, cnt, S->hoff, (int)(nh + 1), st);
            NRT_CUDA(cudaMallocAsync(&tmp, tbs, st));
            cub::DeviceScan::ExclusiveSum(tmp, tbs, cnt, S->hoff, (int)(nh + 1), st);
            cudaFreeAsync(tmp, st);
            cudaFreeAsync(cnt, st);
        }
        cudaFreeAsync(hk0, st);
        cudaFreeAsync(hk1, st);
        S->hid = hvb.Current();  // kept: surfel ids of the home records (post-processing)
        cudaFreeAsync(hvb.Current() == hv0 ? hv1 : hv0, st);
    }
    if (D->sdf_cell > 0.0f) NRT_TRY(sdf_build(S, D->sdf_cell, bmin, bmax, st));
    // labels array (int) for the history
    {
        // sn.w holds the label bits; extract with a tiny kernel-free trick: copy strided
        NRT_CUDA(cudaMemcpy2DAsync(S->label, 4, (const char*)S->sn + 12, 16, 4, n,
                                   cudaMemcpyDeviceToDevice, st));
    }
    NRT_CUDA(cudaStreamSynchronize(st));
    return NRT_OK;
}

nrt_status scene_build(const nrt_scene_desc* D, nrt_scene* out) {
    if (!D || !out) return set_error(NRT_E_INVALID, "null argument");
    *out = nullptr;
    if (D->n <= 0) return set_error(NRT_E_EMPTY, "scene has no points");
    if (D->n >= ((int64_t)1 << 31)) return set_error(NRT_E_INVALID, "n >= 2^31");
    if (!D->points || !D->normals) return set_error(NRT_E_INVALID, "points/normals are NULL");
    if (!(D->voxel_size > 0.0f) || !std::isfinite(D->voxel_size))
        return set_error(NRT_E_INVALID, "voxel_size must be > 0");
    if (!D->radii && !(D->radius > 0.0f)) return set_error(NRT_E_INVALID, "radius must be > 0");
    if (!(D->sdf_cell >= 0.0f) || !std::isfinite(D->sdf_cell))
        return set_error(NRT_E_INVALID, "sdf_cell must be finite and >= 0");
    if (D->n_edges < 0 || (D->n_edges > 0 && !D->edges))
        return set_error(NRT_E_INVALID, "bad edge array");
    NRT_CUDA(cudaSetDevice(D->device));
    ensure_pool(D->device);
    cudaStream_t st = (cudaStream_t)D->stream;
    nrt_scene S = new nrt_scene_s();
    S->device = D->device;
    S->n = D->n;
    // edges (host): validate, precompute e and len with the definition's FP32 formula
    for (int j = 0; j < D->n_edges; ++j) {
        const nrt_edge& E = D->edges[j];
        DevEdge g{};
        if (!(E.n_exp > 1.0f && E.n_exp < 2.0f)) {
            delete S;
            return set_error(NRT_E_INVALID, "edge %d: exterior angle n_exp=%g outside (1,2) "
                             "(only exterior edges are supported, P:73)", j, (double)E.n_exp);
        }
        if (E.label < 0 || E.label >= 4096) {
            delete S;
            return set_error(NRT_E_INVALID, "edge %d: label outside [0,4096)", j);
        }
        float ev[3] = {E.b[0] - E.a[0], E.b[1] - E.a[1], E.b[2] - E.a[2]};
        float len = sqrtf((ev[0] * ev[0] + ev[1] * ev[1]) + ev[2] * ev[2]);
        if (!(len > 0.0f) || !std::isfinite(len)) {
            delete S;
            return set_error(NRT_E_INVALID, "edge %d: zero or non-finite length", j);
        }
        for (int k = 0; k < 3; ++k) {
            g.a[k] = E.a[k];
            g.e[k] = ev[k] / len;
            g.t0[k] = E.t0[k];
            g.n0[k] = E.n0[k];
            g.n1[k] = E.n1[k];
        }
        g.len = len;
        g.n_exp = E.n_exp;
        g.label = E.label;
        for (int k = 0; k < 3; ++k) g.c[k] = 0.5f * (E.a[k] + E.b[k]);
        for (int k = 0; k < 3; ++k) g.b_[k] = E.b[k];
        g.hl = 0.5f * len * 1.001f + 1e-4f;
        S->h_edges.push_back(g);
    }
    S->n_edges = D->n_edges;
    nrt_status rc = build_impl(D, S, st);
    if (rc == NRT_OK && S->n_edges > 0) {
        cudaError_t e = cudaMallocAsync((void**)&S->edges, sizeof(DevEdge) * S->n_edges, st);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(S->edges, S->h_edges.data(), sizeof(DevEdge) * S->n_edges,
                                cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) rc = set_error(NRT_E_CUDA, "edge upload: %s", cudaGetErrorString(e));
    }
    if (rc != NRT_OK) {
        nrt_scene_free(S);
        return rc;
    }
    *out = S;
    return NRT_OK;
}

}  // namespace nrt
