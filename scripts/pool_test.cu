// microbenchmark: stream-ordered pool allocation cost after a pre-reserve
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
static double now() { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main() {
    cudaFree(0);
    cudaMemPool_t pool;
    cudaDeviceGetDefaultMemPool(&pool, 0);
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    double t = now();
    void* big;
    cudaMallocAsync(&big, 4ull << 30, 0);
    cudaFreeAsync(big, 0);
    cudaStreamSynchronize(0);
    printf("reserve 4GB %.3f ms\n", now() - t);
    cudaStream_t st;
    cudaStreamCreate(&st);
    for (int rep = 0; rep < 3; ++rep) {
        for (int which = 0; which < 2; ++which) {
            cudaStream_t s = which ? st : 0;
            void* p[8];
            t = now();
            for (int i = 0; i < 8; ++i) cudaMallocAsync(&p[i], 370ull << 20, s);
            cudaStreamSynchronize(s);
            double ta = now() - t;
            t = now();
            for (int i = 0; i < 8; ++i) cudaMemsetAsync(p[i], 0, 370ull << 20, s);
            cudaStreamSynchronize(s);
            double tm = now() - t;
            for (int i = 0; i < 8; ++i) cudaFreeAsync(p[i], s);
            cudaStreamSynchronize(s);
            size_t used, res;
            cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &res);
            cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
            printf("rep %d stream %d alloc %.3f ms memset %.3f ms reserved %.2f GB used %.2f GB\n", rep, which, ta, tm, res / 1e9, used / 1e9);
        }
    }
    return 0;
}
