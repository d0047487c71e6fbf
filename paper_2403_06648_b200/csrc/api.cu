// api.cu — the extern "C" boundary of libnrt (include/nrt.h).  Argument validation, handle
// lifetime, phase orchestration (primary -> events -> fans -> dedupe) and path-set plumbing.
#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <cstdlib>
#include <mutex>
#include <vector>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "internal.cuh"

namespace nrt {
static thread_local char g_err[1024] = "";

nrt_status set_error(nrt_status st, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return st;
}
void clear_error() { g_err[0] = 0; }

static std::atomic<unsigned long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// Stream-ordered allocations come from the device's default pool; keep freed blocks cached
// (release threshold = max) so that repeated launches do not return memory to the driver.
void ensure_pool(int dev) {
    static std::atomic<unsigned long long> done{0};
    if (dev < 0 || dev >= 64) return;
    const unsigned long long bit = 1ull << dev;
    if (done.load() & bit) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        // pre-reserve: one large allocation returned to the pool keeps its physical backing
        // mapped, so later launches sub-allocate without growing the pool (NRT_POOL_GB, def. 4)
        const char* e = getenv("NRT_POOL_GB");
        const double gb = e ? atof(e) : 4.0;
        if (gb > 0) {
            void* p = nullptr;
            if (cudaMallocAsync(&p, (size_t)(gb * (1ull << 30)), nullptr) == cudaSuccess) {
                cudaFreeAsync(p, nullptr);
                cudaStreamSynchronize(nullptr);
            } else {
                cudaGetLastError();
            }
        }
    }
    done.fetch_or(bit);
}

// Keep the stream-ordered pool's physical backing at 1.5x the high-water mark of its use: a pool
// that must grow inside a step maps new pages there (measured on C5: scene builds of 0.1-1.5 s
// instead of 6 ms in 4 of 10 steps); one reservation after the first large call removes that.
void pool_keep_headroom(int dev, cudaStream_t st) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return;
    uint64_t reserved = 0, used = 0, high = 0;
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &high);
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    uint64_t target = high + high / 2;
    if (target > total_b / 2) target = total_b / 2;  // never more than half of the device
    if (reserved >= target || target <= used) return;
    void* p = nullptr;
    if (cudaMallocAsync(&p, (size_t)(target - used), st) == cudaSuccess) {
        cudaFreeAsync(p, st);
    } else {
        cudaGetLastError();
    }
    // the reservation itself is not use: restore the high-water mark to the real one
    cudaStreamSynchronize(st);
    uint64_t zero = 0;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &zero);
}

namespace {
struct WsBlock {
    int dev;
    void* p;
    size_t bytes;
    bool busy;
};
std::mutex g_ws_mu;
std::vector<WsBlock> g_ws;
}  // namespace

void* ws_get(int dev, size_t bytes, cudaStream_t st) {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    WsBlock* best = nullptr;
    for (auto& b : g_ws)
        if (!b.busy && b.dev == dev && b.bytes >= bytes && (!best || b.bytes < best->bytes))
            best = &b;
    if (best) {
        best->busy = true;
        return best->p;
    }
    const size_t gran = 64ull << 20;
    const size_t sz = (bytes + gran - 1) / gran * gran;
    void* p = nullptr;
    if (cudaMallocAsync(&p, sz, st) != cudaSuccess) {
        cudaGetLastError();
        // idle cached blocks of this device may be what stands in the way: drop them, retry
        for (auto it = g_ws.begin(); it != g_ws.end();) {
            if (!it->busy && it->dev == dev) {
                cudaFreeAsync(it->p, st);
                it = g_ws.erase(it);
            } else {
                ++it;
            }
        }
        cudaStreamSynchronize(st);
        if (cudaMallocAsync(&p, sz, st) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
    }
    g_ws.push_back({dev, p, sz, true});
    return p;
}

void ws_put(void* p) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_ws_mu);
    for (auto& b : g_ws)
        if (b.p == p) b.busy = false;
}

struct RxGuard {  // frees a launch's receiver grid on every exit path
    RxGrid* g;
    cudaStream_t st;
    ~RxGuard() { rxgrid_free(g, st); }
};

// NRT_PHASES=1: synchronise and print host wall time per phase (diagnostics only)
struct PhaseLog {
    bool on;
    cudaStream_t st;
    std::chrono::steady_clock::time_point t;
    explicit PhaseLog(cudaStream_t s) : on(getenv("NRT_PHASES") != nullptr), st(s) {
        if (on) {
            cudaStreamSynchronize(st);
            t = std::chrono::steady_clock::now();
        }
    }
    void mark(const char* what) {
        if (!on) return;
        cudaStreamSynchronize(st);
        auto n = std::chrono::steady_clock::now();
        fprintf(stderr, "[nrt] %-16s %8.3f ms\n", what,
                std::chrono::duration<double, std::milli>(n - t).count());
        t = n;
    }
};

static bool finite3(const float* x) {
    return std::isfinite(x[0]) && std::isfinite(x[1]) && std::isfinite(x[2]);
}

static size_t rec_size(int kind) {
    switch (kind) {
        case NRT_PATHS_COARSE: return sizeof(nrt_coarse_rec);
        case NRT_PATHS_REFINED: return sizeof(nrt_refined_rec);
        default: return sizeof(nrt_event_rec);
    }
}

struct EventTimer {
    cudaEvent_t a = nullptr, b = nullptr;
    cudaStream_t st;
    explicit EventTimer(cudaStream_t s) : st(s) {
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, st);
    }
    float stop() {
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        return ms;
    }
    ~EventTimer() {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    }
};

static nrt_status check_launch(nrt_scene s, const float* tx, const float* rx, int32_t n_rx,
                               int64_t n_rays, int32_t max_refl, int32_t max_diff,
                               const nrt_launch_desc& d) {
    if (!s) return set_error(NRT_E_INVALID, "scene is NULL");
    if (!tx) return set_error(NRT_E_INVALID, "tx is NULL");
    if (n_rx < 0 || n_rx > 65535) return set_error(NRT_E_INVALID, "n_rx must be in [0, 65535]");
    if (n_rx > 0 && !rx) return set_error(NRT_E_INVALID, "rx is NULL");
    if (n_rays < 1 || n_rays >= ((int64_t)1 << 32))
        return set_error(NRT_E_INVALID, "n_rays must be in [1, 2^32)");
    if (max_refl < 0 || max_diff < 0 || max_refl + max_diff > NRT_MAX_INT)
        return set_error(NRT_E_INVALID, "need max_refl, max_diff >= 0 and max_refl + max_diff <= %d",
                         NRT_MAX_INT);
    if (d.kappa < 1) return set_error(NRT_E_INVALID, "kappa must be >= 1");
    if (!(d.tau >= 0.0f) || !(d.c_R > 0.0f) || !(d.dphi_deg > 0.0f) || !(d.edge_bin > 0.0f))
        return set_error(NRT_E_INVALID, "tau >= 0, c_R > 0, dphi_deg > 0, edge_bin > 0 required");
    if (!(d.theta_ex_deg > 0.0f && d.theta_ex_deg < 90.0f))
        return set_error(NRT_E_INVALID, "theta_ex_deg must be in (0, 90)");
    if (d.world < 1 || d.rank < 0 || d.rank >= d.world)
        return set_error(NRT_E_INVALID, "need 0 <= rank < world");
    if (d.stage < 0 || d.stage > 1) return set_error(NRT_E_INVALID, "stage must be 0 or 1");
    if (d.stage == 0 && d.world > 1 && max_diff > 0 && s->n_edges > 0)
        return set_error(NRT_E_STATE, "world > 1 with diffraction needs the two-stage protocol "
                                      "(stage 1 + event all-gather + nrt_launch_fans)");
    if (d.intersect < 0 || d.intersect > 1) return set_error(NRT_E_INVALID, "intersect must be 0 or 1");
    if (d.tracer < 0 || d.tracer > 1) return set_error(NRT_E_INVALID, "tracer must be 0 or 1");
    if (d.tracer == 1 && d.intersect != 1)
        return set_error(NRT_E_STATE, "tracer = 1 (cone tracing) validates with the SDF: needs intersect = 1");
    if (d.intersect == 1) {
        if (!s->n_aabb)
            return set_error(NRT_E_STATE, "intersect = 1 (SDF) needs a scene built with sdf_cell > 0");
        if (!(d.sdf_r_s > 0.0f) || !(d.sdf_t_sdf > 0.0f) || !(d.sdf_xi > 0.0f) ||
            !std::isfinite(d.sdf_r_s) || !std::isfinite(d.sdf_t_sdf) || !std::isfinite(d.sdf_xi))
            return set_error(NRT_E_INVALID, "sdf_r_s, sdf_t_sdf, sdf_xi must be finite and > 0");
    }
    for (int j = 0; j < s->n_edges; ++j)
        if (s->h_edges[j].len / d.edge_bin >= (float)(1 << 27))
            return set_error(NRT_E_INVALID, "edge %d too long for edge_bin", j);
    return NRT_OK;
}

}  // namespace nrt

using namespace nrt;

extern "C" {

const char* nrt_last_error(void) { return g_err; }
const char* nrt_version(void) { return "nrt 0.1 (sm_100a)"; }
uint64_t nrt_kernel_launches(void) { return g_launches.load(); }

double nrt_probe_fp64_tflops(int device) { return ::nrt::probe_fp64_tflops(device); }

uint64_t nrt_workspace_bytes(void) {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    uint64_t t = 0;
    for (auto& b : g_ws) t += b.bytes;
    return t;
}

void nrt_workspace_trim(void) {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    for (auto it = g_ws.begin(); it != g_ws.end();) {
        if (!it->busy) {
            int cur = 0;
            cudaGetDevice(&cur);
            cudaSetDevice(it->dev);
            cudaFreeAsync(it->p, nullptr);
            cudaStreamSynchronize(nullptr);
            cudaSetDevice(cur);
            it = g_ws.erase(it);
        } else {
            ++it;
        }
    }
}

nrt_status nrt_scene_build(const float* points, const float* normals, int64_t n, float voxel_size,
                           nrt_scene* out) {
    nrt_scene_desc d{};
    d.points = points;
    d.normals = normals;
    d.radius = 0.015f;
    d.n = n;
    d.voxel_size = voxel_size;
    d.mem = NRT_MEM_HOST;
    return nrt_scene_build_ex(&d, out);
}

nrt_status nrt_scene_build_ex(const nrt_scene_desc* desc, nrt_scene* out) {
    clear_error();
    return scene_build(desc, out);
}

// Every entry point synchronises its stream before returning and handle memory is private,
// so no device work can still reference it: free into the stream-ordered pool directly.
void nrt_scene_free(nrt_scene s) {
    if (!s) return;
    cudaSetDevice(s->device);
    cudaFreeAsync(s->cell, nullptr);
    cudaFreeAsync(s->rec, nullptr);
    cudaFreeAsync(s->sp, nullptr);
    cudaFreeAsync(s->sn, nullptr);
    cudaFreeAsync(s->label, nullptr);
    cudaFreeAsync(s->hcell, nullptr);
    cudaFreeAsync(s->hrec, nullptr);
    cudaFreeAsync(s->hid, nullptr);
    cudaFreeAsync(s->hoff, nullptr);
    cudaFreeAsync(s->edges, nullptr);
    cudaFreeAsync(s->sdf_pts, nullptr);
    cudaFreeAsync(s->sdf_box, nullptr);
    cudaFreeAsync(s->sdf_acell, nullptr);
    cudaFreeAsync(s->sdf_gcell, nullptr);
    cudaFreeAsync(s->sdf_aref, nullptr);
    cudaFreeAsync(s->sdf_crange, nullptr);
    delete s;
}

nrt_status nrt_scene_info_get(nrt_scene s, nrt_scene_info* info) {
    if (!s || !info) return set_error(NRT_E_INVALID, "null argument");
    info->n_surfels = s->n;
    info->n_refs = s->nref;
    info->n_cells = s->ncell;
    for (int a = 0; a < 3; ++a) {
        info->dims[a] = s->dims[a];
        info->origin[a] = s->org[a];
    }
    info->voxel = s->v;
    info->r_max = s->r_max;
    info->n_aabb = s->n_aabb;
    info->n_aabb_refs = s->n_aref;
    info->sdf_cell = s->sdf_a;
    return NRT_OK;
}

void nrt_launch_desc_default(nrt_launch_desc* d) {
    if (!d) return;
    memset(d, 0, sizeof(*d));
    d->kappa = 1;
    d->tau = 0.0015f;
    d->c_R = 1.0f;
    d->dphi_deg = 2.5f;
    d->theta_ex_deg = 25.0f;
    d->edge_bin = 0.25f;
    d->rank = 0;
    d->world = 1;
    d->stage = 0;
    d->mem = NRT_MEM_HOST;
    d->stream = nullptr;
    d->intersect = 0;
    d->tracer = 0;
    d->sdf_r_s = 0.015f;
    d->sdf_t_sdf = 0.0015f;
    d->sdf_xi = 2.0f;
}

nrt_status nrt_launch(nrt_scene s, const float tx[3], const float* rx, int32_t n_rx, int64_t n_rays,
                      int32_t max_refl, int32_t max_diff, nrt_paths* out) {
    nrt_launch_desc d;
    nrt_launch_desc_default(&d);
    return nrt_launch_ex(s, tx, rx, n_rx, n_rays, max_refl, max_diff, &d, out);
}

static nrt_status finish_coarse(nrt_paths P, nrt_coarse_rec* raw, int64_t n_raw, int32_t kappa,
                                cudaStream_t st) {
    EventTimer t(st);
    nrt_coarse_rec* out = nullptr;
    NRT_CUDA(cudaMallocAsync(&out, (n_raw > 0 ? n_raw : 1) * sizeof(nrt_coarse_rec), st));
    int64_t m = 0;
    NRT_TRY(dedupe_coarse(raw, n_raw, kappa, out, &m, st));
    P->d_rec = out;
    P->n = m;
    P->info.n = m;
    P->info.ms_dedupe += t.stop();
    return NRT_OK;
}

nrt_status nrt_launch_ex(nrt_scene s, const float tx[3], const float* rx, int32_t n_rx,
                         int64_t n_rays, int32_t max_refl, int32_t max_diff,
                         const nrt_launch_desc* desc, nrt_paths* out) {
    clear_error();
    if (!out) return set_error(NRT_E_INVALID, "out is NULL");
    *out = nullptr;
    nrt_launch_desc d;
    if (desc) d = *desc;
    else nrt_launch_desc_default(&d);
    NRT_TRY(check_launch(s, tx, rx, n_rx, n_rays, max_refl, max_diff, d));
    NRT_CUDA(cudaSetDevice(s->device));
    ensure_pool(s->device);
    cudaStream_t st = (cudaStream_t)d.stream;
    LaunchArgs a{};
    float htx[3];
    std::vector<float> hrx(3 * (size_t)n_rx);
    if (d.mem == NRT_MEM_DEVICE) {
        NRT_CUDA(cudaMemcpyAsync(htx, tx, 12, cudaMemcpyDeviceToHost, st));
        if (n_rx) NRT_CUDA(cudaMemcpyAsync(hrx.data(), rx, 12 * n_rx, cudaMemcpyDeviceToHost, st));
        NRT_CUDA(cudaStreamSynchronize(st));
    } else {
        memcpy(htx, tx, 12);
        if (n_rx) memcpy(hrx.data(), rx, 12 * (size_t)n_rx);
    }
    if (!finite3(htx)) return set_error(NRT_E_INVALID, "tx not finite");
    for (int j = 0; j < n_rx; ++j)
        if (!finite3(&hrx[3 * j])) return set_error(NRT_E_INVALID, "rx %d not finite", j);
    float* d_rx = nullptr;
    NRT_CUDA(cudaMallocAsync(&d_rx, 12 * (size_t)(n_rx > 0 ? n_rx : 1), st));
    if (n_rx)
        NRT_CUDA(cudaMemcpyAsync(d_rx, hrx.data(), 12 * (size_t)n_rx, cudaMemcpyHostToDevice, st));
    memcpy(a.tx, htx, 12);
    a.d_rx = d_rx;
    a.n_rx = n_rx;
    a.n_rays = n_rays;
    a.max_refl = max_refl;
    a.max_diff = max_diff;
    a.desc = d;
    a.h_rx = hrx.data();
    float r_prim = 0, r_fan = 0;
    capture_radius_bounds(s, a, &r_prim, &r_fan);
    NRT_TRY(rxgrid_build(s, hrx.data(), n_rx, r_prim, &a.rxg, st));
    RxGuard rx_guard{&a.rxg, st};
    LaunchArgs af = a;  // fans: capture radii up to r_fan (R16)
    af.rxg = RxGrid{};
    if (max_diff > 0 && s->n_edges > 0) NRT_TRY(rxgrid_build(s, hrx.data(), n_rx, r_fan, &af.rxg, st));
    RxGuard rx_guard_f{&af.rxg, st};

    nrt_paths P = new nrt_paths_s();
    P->kind = NRT_PATHS_COARSE;
    P->device = s->device;
    memcpy(P->tx, htx, 12);
    P->rx = hrx;
    P->n_rays = n_rays;
    P->max_refl = max_refl;
    P->max_diff = max_diff;
    P->info.kind = NRT_PATHS_COARSE;

    EventTimer total(st);
    PhaseLog ph(st);
    if (d.tracer == 1) {  // NEXT-2: environment-driven launch + voxel cone tracing
        nrt_coarse_rec* raw = nullptr;
        int64_t n_raw = 0;
        uint64_t rays = 0;
        float ms = 0.0f;
        uint64_t terms = 0;
        nrt_status rc = launch_env(s, a, &raw, &n_raw, &rays, &ms, &terms, st);
        cudaFreeAsync(d_rx, st);
        P->info.bounces = rays;
        P->info.surfel_tests = terms;  // Gaussian terms of the validation traces (counters = 1)
        P->info.ms_trace = ms;
        P->info.n_raw = n_raw;
        if (rc == NRT_OK) rc = finish_coarse(P, raw, n_raw, d.kappa, st);
        cudaFreeAsync(raw, st);
        if (rc != NRT_OK) {
            nrt_paths_free(P);
            return rc;
        }
        P->info.ms_total = total.stop();
        pool_keep_headroom(s->device, st);
        *out = P;
        return NRT_OK;
    }
    nrt_coarse_rec* raw = nullptr;
    nrt_event_rec* ev = nullptr;
    int64_t n_raw = 0, n_ev = 0;
    uint64_t b1 = 0;
    nrt_status rc;
    {
        KernelStats ks;
        rc = launch_primary(s, a, &raw, &n_raw, &ev, &n_ev, &b1, &ks, st);
        ph.mark("primary");
        P->info.ms_trace = ks.ms_kernel;
        P->info.surfel_tests = ks.tests;
        P->info.cells_visited = ks.cells;
        P->info.cells_nonempty = ks.nonempty;
    }
    if (rc != NRT_OK) {
        cudaFreeAsync(d_rx, st);
        delete P;
        return rc;
    }
    P->info.bounces = b1;
    // local event dedupe (global when world == 1)
    nrt_event_rec* evu = nullptr;
    int64_t n_evu = 0;
    if (n_ev > 0) {
        EventTimer t(st);
        rc = cudaMallocAsync(&evu, n_ev * sizeof(nrt_event_rec), st) == cudaSuccess
                 ? dedupe_events(ev, n_ev, evu, &n_evu, st)
                 : set_error(NRT_E_NOMEM, "event buffer");
        P->info.ms_dedupe += t.stop();
        ph.mark("event dedupe");
    }
    cudaFreeAsync(ev, st);
    if (rc != NRT_OK) {
        cudaFreeAsync(d_rx, st);
        cudaFreeAsync(raw, st);
        delete P;
        return rc;
    }
    P->n_ev = n_evu;
    P->info.n_events = n_evu;
    if (d.stage == 0 && n_evu > 0) {
        nrt_coarse_rec* fraw = nullptr;
        int64_t nf = 0, nfr = 0;
        uint64_t b2 = 0;
        {
            KernelStats ks;
            rc = launch_fans(s, af, evu, n_evu, &fraw, &nf, &nfr, &b2, &ks, st);
            P->info.ms_fans = ks.ms_kernel;
            P->info.surfel_tests += ks.tests;
            P->info.cells_visited += ks.cells;
            P->info.cells_nonempty += ks.nonempty;
            ph.mark("fans");
        }
        if (rc == NRT_OK && nf > 0) {
            nrt_coarse_rec* both = nullptr;
            if (cudaMallocAsync(&both, (n_raw + nf) * sizeof(nrt_coarse_rec), st) != cudaSuccess) {
                rc = set_error(NRT_E_NOMEM, "record buffer");
            } else {
                cudaMemcpyAsync(both, raw, n_raw * sizeof(nrt_coarse_rec), cudaMemcpyDeviceToDevice, st);
                cudaMemcpyAsync(both + n_raw, fraw, nf * sizeof(nrt_coarse_rec),
                                cudaMemcpyDeviceToDevice, st);
                cudaFreeAsync(raw, st);
                raw = both;
                n_raw += nf;
            }
        }
        cudaFreeAsync(fraw, st);
        P->info.bounces += b2;
        P->info.n_fan_rays = nfr;
        cudaFreeAsync(evu, st);
        evu = nullptr;
    }
    P->d_ev = evu;
    cudaFreeAsync(d_rx, st);
    P->info.n_raw = n_raw;
    ph.mark("append");
    if (rc == NRT_OK) rc = finish_coarse(P, raw, n_raw, d.kappa, st);
    ph.mark("record dedupe");
    cudaFreeAsync(raw, st);
    if (rc != NRT_OK) {
        nrt_paths_free(P);
        return rc;
    }
    P->info.ms_total = total.stop();
    pool_keep_headroom(s->device, st);
    *out = P;
    return NRT_OK;
}

nrt_status nrt_launch_fans(nrt_scene s, nrt_paths coarse, const void* events, int64_t n_events,
                           nrt_mem mem, const nrt_launch_desc* desc) {
    clear_error();
    if (!s || !coarse || !desc) return set_error(NRT_E_INVALID, "null argument");
    if (coarse->kind != NRT_PATHS_COARSE) return set_error(NRT_E_STATE, "not a coarse set");
    if (n_events < 0 || (n_events > 0 && !events)) return set_error(NRT_E_INVALID, "bad events");
    NRT_CUDA(cudaSetDevice(s->device));
    ensure_pool(s->device);
    cudaStream_t st = (cudaStream_t)desc->stream;
    nrt_launch_desc d = *desc;
    LaunchArgs a{};
    memcpy(a.tx, coarse->tx, 12);
    a.n_rx = (int32_t)(coarse->rx.size() / 3);
    a.n_rays = coarse->n_rays;
    a.max_refl = coarse->max_refl;
    a.max_diff = coarse->max_diff;
    a.desc = d;
    NRT_TRY(check_launch(s, coarse->tx, coarse->rx.data(), a.n_rx, a.n_rays, a.max_refl, a.max_diff,
                         [&] { nrt_launch_desc x = d; x.stage = 1; return x; }()));
    float r_prim = 0, r_fan = 0;
    capture_radius_bounds(s, a, &r_prim, &r_fan);
    NRT_TRY(rxgrid_build(s, coarse->rx.data(), a.n_rx, r_fan, &a.rxg, st));
    RxGuard rx_guard{&a.rxg, st};
    float* d_rx = nullptr;
    NRT_CUDA(cudaMallocAsync(&d_rx, 12 * (size_t)(a.n_rx > 0 ? a.n_rx : 1), st));
    if (a.n_rx)
        NRT_CUDA(cudaMemcpyAsync(d_rx, coarse->rx.data(), 12 * (size_t)a.n_rx, cudaMemcpyHostToDevice, st));
    a.d_rx = d_rx;
    nrt_event_rec *ev = nullptr, *evu = nullptr;
    const size_t evb = (size_t)(n_events > 0 ? n_events : 1) * sizeof(nrt_event_rec);
    NRT_CUDA(cudaMallocAsync(&ev, evb, st));
    NRT_CUDA(cudaMallocAsync(&evu, evb, st));
    if (n_events)
        NRT_CUDA(cudaMemcpyAsync(ev, events, n_events * sizeof(nrt_event_rec),
                                 mem == NRT_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st));
    int64_t n_evu = 0;
    NRT_TRY(dedupe_events(ev, n_events, evu, &n_evu, st));
    nrt_coarse_rec* fraw = nullptr;
    int64_t nf = 0, nfr = 0;
    uint64_t b2 = 0;
    {
        KernelStats ks;
        NRT_TRY(launch_fans(s, a, evu, n_evu, &fraw, &nf, &nfr, &b2, &ks, st));
        coarse->info.ms_fans = ks.ms_kernel;
        coarse->info.surfel_tests += ks.tests;
        coarse->info.cells_visited += ks.cells;
        coarse->info.cells_nonempty += ks.nonempty;
    }
    cudaFreeAsync(ev, st);
    cudaFreeAsync(evu, st);
    cudaFreeAsync(d_rx, st);
    // append to the current (deduped) set and dedupe again
    const int64_t n0 = coarse->n;
    nrt_coarse_rec* both = nullptr;
    NRT_CUDA(cudaMallocAsync(&both, (size_t)(n0 + nf > 0 ? n0 + nf : 1) * sizeof(nrt_coarse_rec), st));
    if (n0) NRT_CUDA(cudaMemcpyAsync(both, coarse->d_rec, n0 * sizeof(nrt_coarse_rec), cudaMemcpyDeviceToDevice, st));
    if (nf) NRT_CUDA(cudaMemcpyAsync(both + n0, fraw, nf * sizeof(nrt_coarse_rec), cudaMemcpyDeviceToDevice, st));
    cudaFreeAsync(fraw, st);
    cudaFreeAsync(coarse->d_rec, st);
    coarse->d_rec = nullptr;
    coarse->info.bounces += b2;
    coarse->info.n_fan_rays = nfr;
    coarse->info.n_raw += nf;
    nrt_status rc = finish_coarse(coarse, both, n0 + nf, d.kappa, st);
    cudaFreeAsync(both, st);
    NRT_CUDA(cudaStreamSynchronize(st));
    return rc;
}

void nrt_refine_desc_default(nrt_refine_desc* d) {
    if (!d) return;
    memset(d, 0, sizeof(*d));
    d->xi = 2.0;
    d->r_s = 0.003;
    d->tol_m = 1e-10;
    d->max_iter = 100;
    d->alpha = 0.4;
    d->beta = 0.4;
    d->delta = 1e-4;
    d->tau = 0.0015;
    d->theta_ex_deg = 25.0;
    d->rank = 0;
    d->world = 1;
    d->keep_invalid = 0;
    d->select = 0;
    d->blocks_per_sm = 0;
    d->stream = nullptr;
    d->method = 0;
    d->gd_rho = 2000;
    d->gd_t_sdf = 0.001;
    d->gd_t_d = 0.02;
    d->gd_t_a_deg = 1.0;
}

nrt_status nrt_refine(nrt_scene s, nrt_paths coarse, nrt_paths* out) {
    nrt_refine_desc d;
    nrt_refine_desc_default(&d);
    return nrt_refine_ex(s, coarse, &d, out);
}

void nrt_post_desc_default(nrt_post_desc* d) {
    if (!d) return;
    d->lambda_m = 299792458.0 / 60e9;
    d->angle_deg = 10.0;
    d->r_s = 0.003;
    d->stream = nullptr;
}

nrt_status nrt_postprocess(nrt_scene s, nrt_paths refined, const nrt_post_desc* desc, nrt_paths* out) {
    clear_error();
    if (!s || !refined || !out) return set_error(NRT_E_INVALID, "null argument");
    *out = nullptr;
    if (refined->kind != NRT_PATHS_REFINED) return set_error(NRT_E_STATE, "post-processing needs a refined set");
    nrt_post_desc d;
    if (desc) d = *desc;
    else nrt_post_desc_default(&d);
    if (!(d.lambda_m > 0 && d.angle_deg > 0 && d.angle_deg < 180 && d.r_s >= 0))
        return set_error(NRT_E_INVALID, "bad post-processing parameters");
    NRT_CUDA(cudaSetDevice(s->device));
    ensure_pool(s->device);
    nrt_paths P = new nrt_paths_s();
    P->kind = NRT_PATHS_REFINED;
    P->device = s->device;
    memcpy(P->tx, refined->tx, 12);
    P->rx = refined->rx;
    P->info.kind = NRT_PATHS_REFINED;
    nrt_status rc = postprocess(s, refined, &d, P, (cudaStream_t)d.stream);
    if (rc != NRT_OK) {
        nrt_paths_free(P);
        return rc;
    }
    P->info.n = P->n;
    P->info.n_raw = refined->n;
    *out = P;
    return NRT_OK;
}

nrt_status nrt_refine_ex(nrt_scene s, nrt_paths coarse, const nrt_refine_desc* desc,
                         nrt_paths* out) {
    clear_error();
    if (!s || !coarse || !out) return set_error(NRT_E_INVALID, "null argument");
    *out = nullptr;
    if (coarse->kind != NRT_PATHS_COARSE) return set_error(NRT_E_STATE, "refine needs a coarse set");
    nrt_refine_desc d;
    if (desc) d = *desc;
    else nrt_refine_desc_default(&d);
    if (!(d.xi > 0 && d.r_s > 0 && d.tol_m > 0 && d.max_iter >= 1 && d.alpha > 0 && d.alpha < 0.5 &&
          d.beta > 0 && d.beta < 1 && d.tau >= 0 && d.theta_ex_deg > 0 && d.theta_ex_deg < 90))
        return set_error(NRT_E_INVALID, "bad refine parameters");
    if (d.world < 1 || d.rank < 0 || d.rank >= d.world)
        return set_error(NRT_E_INVALID, "need 0 <= rank < world");
    if (d.select < 0 || d.select > 2) return set_error(NRT_E_INVALID, "select must be 0, 1 or 2");
    if (d.blocks_per_sm < 0) return set_error(NRT_E_INVALID, "blocks_per_sm must be >= 0");
    if (d.method < 0 || d.method > 1) return set_error(NRT_E_INVALID, "method must be 0 or 1");
    if (d.method == 1) {
        if (!s->n_aabb)
            return set_error(NRT_E_STATE, "method = 1 (paper GD) needs a scene built with sdf_cell > 0");
        if (d.select != 0) return set_error(NRT_E_INVALID, "method = 1 supports select = 0 only");
        if (!(d.gd_rho >= 0 && d.gd_t_sdf > 0 && d.gd_t_d >= 0 && d.gd_t_a_deg >= 0 && d.gd_t_a_deg <= 180 &&
              d.delta > 0))
            return set_error(NRT_E_INVALID, "bad gradient-descent parameters");
    }
    NRT_CUDA(cudaSetDevice(s->device));
    ensure_pool(s->device);
    nrt_paths P = new nrt_paths_s();
    P->kind = NRT_PATHS_REFINED;
    P->device = s->device;
    memcpy(P->tx, coarse->tx, 12);
    P->rx = coarse->rx;
    P->info.kind = NRT_PATHS_REFINED;
    nrt_status rc = d.method == 1 ? refine_gd(s, coarse, &d, P, (cudaStream_t)d.stream)
                                  : refine(s, coarse, &d, P, (cudaStream_t)d.stream);
    if (rc == NRT_OK) pool_keep_headroom(s->device, (cudaStream_t)d.stream);
    if (rc != NRT_OK) {
        nrt_paths_free(P);
        return rc;
    }
    *out = P;
    return NRT_OK;
}

nrt_status nrt_paths_count(nrt_paths p, int64_t* n) {
    if (!p || !n) return set_error(NRT_E_INVALID, "null argument");
    *n = p->n;
    return NRT_OK;
}

nrt_status nrt_paths_record_size(nrt_paths p, int64_t* bytes) {
    if (!p || !bytes) return set_error(NRT_E_INVALID, "null argument");
    *bytes = (int64_t)rec_size(p->kind);
    return NRT_OK;
}

nrt_status nrt_paths_info_get(nrt_paths p, nrt_paths_info* info) {
    if (!p || !info) return set_error(NRT_E_INVALID, "null argument");
    *info = p->info;
    info->kind = p->kind;
    info->n = p->n;
    return NRT_OK;
}

nrt_status nrt_paths_export(nrt_paths p, void* dst, int64_t cap, nrt_mem mem) {
    clear_error();
    if (!p) return set_error(NRT_E_INVALID, "null paths");
    const int64_t need = p->n * (int64_t)rec_size(p->kind);
    if (cap < need) return set_error(NRT_E_OVERFLOW, "need %lld bytes", (long long)need);
    if (need == 0) return NRT_OK;
    if (!dst) return set_error(NRT_E_INVALID, "dst is NULL");
    NRT_CUDA(cudaSetDevice(p->device));
    NRT_CUDA(cudaMemcpy(dst, p->d_rec, need,
                        mem == NRT_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice));
    return NRT_OK;
}

nrt_status nrt_paths_export_events(nrt_paths p, void* dst, int64_t cap, int64_t* n_events,
                                   nrt_mem mem) {
    clear_error();
    if (!p || !n_events) return set_error(NRT_E_INVALID, "null argument");
    *n_events = p->d_ev ? p->n_ev : 0;
    const int64_t need = *n_events * (int64_t)sizeof(nrt_event_rec);
    if (cap < need) return set_error(NRT_E_OVERFLOW, "need %lld bytes", (long long)need);
    if (need == 0) return NRT_OK;
    if (!dst) return set_error(NRT_E_INVALID, "dst is NULL");
    NRT_CUDA(cudaSetDevice(p->device));
    NRT_CUDA(cudaMemcpy(dst, p->d_ev, need,
                        mem == NRT_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice));
    return NRT_OK;
}

nrt_status nrt_paths_import(const void* src, int64_t n, int32_t kind, nrt_mem mem,
                            const float tx[3], const float* rx, int32_t n_rx, nrt_paths* out) {
    clear_error();
    if (!out) return set_error(NRT_E_INVALID, "out is NULL");
    *out = nullptr;
    if (kind != NRT_PATHS_COARSE && kind != NRT_PATHS_REFINED)
        return set_error(NRT_E_INVALID, "kind must be COARSE or REFINED");
    if (n < 0 || (n > 0 && !src) || !tx || n_rx < 0 || (n_rx > 0 && !rx))
        return set_error(NRT_E_INVALID, "bad arguments");
    int dev = 0;
    NRT_CUDA(cudaGetDevice(&dev));
    nrt_paths P = new nrt_paths_s();
    P->kind = kind;
    P->device = dev;
    P->n = n;
    memcpy(P->tx, tx, 12);
    P->rx.assign(rx, rx + 3 * (size_t)n_rx);
    P->info.kind = kind;
    P->info.n = n;
    const size_t b = (size_t)n * rec_size(kind);
    ensure_pool(dev);
    if (cudaMallocAsync(&P->d_rec, b > 0 ? b : 1, nullptr) != cudaSuccess) {
        delete P;
        return set_error(NRT_E_NOMEM, "import buffer");
    }
    if (b && cudaMemcpy(P->d_rec, src, b, mem == NRT_MEM_HOST ? cudaMemcpyHostToDevice
                                                              : cudaMemcpyDeviceToDevice) != cudaSuccess) {
        nrt_paths_free(P);
        return set_error(NRT_E_CUDA, "import copy failed");
    }
    *out = P;
    return NRT_OK;
}

nrt_status nrt_paths_merge(const nrt_paths* parts, int32_t n_parts, int32_t kappa, nrt_paths* out) {
    clear_error();
    if (!parts || n_parts < 1 || !out || kappa < 1) return set_error(NRT_E_INVALID, "bad arguments");
    *out = nullptr;
    const int kind = parts[0]->kind;
    int64_t total = 0;
    for (int i = 0; i < n_parts; ++i) {
        if (!parts[i] || parts[i]->kind != kind) return set_error(NRT_E_STATE, "mixed kinds");
        total += parts[i]->n;
    }
    NRT_CUDA(cudaSetDevice(parts[0]->device));
    cudaStream_t st = nullptr;
    const size_t rs = rec_size(kind);
    char* all = nullptr;
    ensure_pool(parts[0]->device);
    NRT_CUDA(cudaMallocAsync(&all, (total > 0 ? total : 1) * rs, st));
    int64_t off = 0;
    for (int i = 0; i < n_parts; ++i) {
        if (parts[i]->n)
            NRT_CUDA(cudaMemcpy(all + off * rs, parts[i]->d_rec, parts[i]->n * rs, cudaMemcpyDeviceToDevice));
        off += parts[i]->n;
    }
    nrt_paths P = new nrt_paths_s();
    P->kind = kind;
    P->device = parts[0]->device;
    memcpy(P->tx, parts[0]->tx, 12);
    P->rx = parts[0]->rx;
    P->n_rays = parts[0]->n_rays;
    P->max_refl = parts[0]->max_refl;
    P->max_diff = parts[0]->max_diff;
    P->info.kind = kind;
    for (int i = 0; i < n_parts; ++i) {
        P->info.bounces += parts[i]->info.bounces;
        P->info.n_raw += parts[i]->info.n_raw;
    }
    nrt_status rc;
    void* o = nullptr;
    if (cudaMallocAsync(&o, (total > 0 ? total : 1) * rs, st) != cudaSuccess) {
        rc = set_error(NRT_E_NOMEM, "merge buffer");
    } else {
        int64_t m = 0;
        if (kind == NRT_PATHS_COARSE)
            rc = dedupe_coarse((nrt_coarse_rec*)all, total, kappa, (nrt_coarse_rec*)o, &m, st);
        else
            rc = dedupe_refined((nrt_refined_rec*)all, total, (nrt_refined_rec*)o, &m, st);
        P->d_rec = o;
        P->n = m;
        P->info.n = m;
    }
    cudaFreeAsync(all, st);
    if (rc != NRT_OK) {
        nrt_paths_free(P);
        return rc;
    }
    NRT_CUDA(cudaStreamSynchronize(st));
    *out = P;
    return NRT_OK;
}

void nrt_paths_free(nrt_paths p) {
    if (!p) return;
    cudaSetDevice(p->device);
    if (p->pool_owned) {
        cudaFreeAsync(p->d_rec, nullptr);
        cudaFreeAsync(p->d_ev, nullptr);
    } else {
        cudaFree(p->d_rec);
        cudaFree(p->d_ev);
    }
    delete p;
}

nrt_status nrt_debug_trace_rays(nrt_scene s, const float tx[3], int64_t n_rays, int32_t max_refl,
                                const nrt_launch_desc* desc, const uint64_t* ray_ids, int64_t n,
                                int64_t* hit_ids) {
    clear_error();
    nrt_launch_desc d;
    if (desc) d = *desc;
    else nrt_launch_desc_default(&d);
    float dummy[3] = {0, 0, 0};
    NRT_TRY(check_launch(s, tx, dummy, 0, n_rays, max_refl, 0, d));
    if (n < 0 || (n > 0 && (!ray_ids || !hit_ids))) return set_error(NRT_E_INVALID, "bad arrays");
    NRT_CUDA(cudaSetDevice(s->device));
    ensure_pool(s->device);
    LaunchArgs a{};
    memcpy(a.tx, tx, 12);
    a.d_rx = nullptr;
    a.n_rx = 0;
    a.n_rays = n_rays;
    a.max_refl = max_refl;
    a.max_diff = 0;
    a.desc = d;
    return debug_trace(s, a, ray_ids, n, hit_ids, (cudaStream_t)d.stream);
}

}  // extern "C"
