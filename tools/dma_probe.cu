// D2H bandwidth from cudaMalloc vs cudaMallocAsync (default pool) device
// memory into cudaHostAlloc'd memory: 2 GiB in 256 MiB chunks on one stream.
#include <cstdio>
#include <cuda_runtime.h>
#include <chrono>

static double run(void *dst, const void *src, size_t n, cudaStream_t s) {
    double best = 0;
    for (int rep = 0; rep < 4; ++rep) {
        cudaStreamSynchronize(s);
        auto t0 = std::chrono::steady_clock::now();
        for (size_t off = 0; off < n; off += (size_t(256) << 20))
            cudaMemcpyAsync((char *)dst + off, (const char *)src + off, size_t(256) << 20,
                            cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (n / dt / 1e9 > best) best = n / dt / 1e9;
    }
    return best;
}

int main() {
    const size_t n = size_t(2) << 30;
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    void *h, *d1, *d2;
    cudaHostAlloc(&h, n, cudaHostAllocPortable);
    cudaMalloc(&d1, n);
    cudaMemPool_t pool;
    cudaDeviceGetDefaultMemPool(&pool, 0);
    unsigned long long thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    cudaMallocAsync(&d2, n, s);
    cudaMemsetAsync(d1, 1, n, s);
    cudaMemsetAsync(d2, 1, n, s);
    printf("{\"cudaMalloc_GBs\": %.1f, \"cudaMallocAsync_pool_GBs\": %.1f}\n", run(h, d1, n, s),
           run(h, d2, n, s));
    return 0;
}
