// Host-side internals shared by the C ABI translation units (api.cu,
// gca_pipeline.cu): the device mesh replica and an RAII device buffer.
#pragma once
#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "gcabem_b200.h"
#include "gcabem_common.cuh"

int gcabem_internal_error(int code, const char *msg);  // api.cu

namespace gcabem {

// GCABEM_TRACE=1: stage timings of the host-side set-up paths on stderr
struct Trace {
    const char *who;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    bool on = std::getenv("GCABEM_TRACE") != nullptr;
    explicit Trace(const char *w) : who(w) {}
    void mark(const char *what) {
        if (!on) return;
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[%s] %-12s %8.2f ms\n", who, what,
                     std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

template <typename T>
struct DevBuf {
    T *p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    cudaError_t alloc(size_t count) {
        release();
        n = count;
        if (count == 0) return cudaSuccess;
        return cudaMalloc(&p, sizeof(T) * count);
    }
    // grow-only (keeps the allocation when it is large enough)
    cudaError_t reserve(size_t count) {
        if (count <= n && p) return cudaSuccess;
        return alloc(count);
    }
    cudaError_t upload(const T *host, size_t count, cudaStream_t s) {
        cudaError_t e = alloc(count);
        if (e != cudaSuccess || count == 0) return e;
        return cudaMemcpyAsync(p, host, sizeof(T) * count, cudaMemcpyHostToDevice, s);
    }
};

// Stream-ordered allocation from the device's default memory pool, whose
// release threshold is raised once per device so freed blocks stay cached:
// payloads of hundreds of MB are allocated and released per assembly call,
// and cudaMalloc/cudaFree of that size cost milliseconds each.
cudaError_t pool_init(int device);

template <typename T>
struct PoolBuf {
    T *p = nullptr;
    size_t n = 0;
    cudaStream_t s = nullptr;
    PoolBuf() = default;
    PoolBuf(const PoolBuf &) = delete;
    PoolBuf &operator=(const PoolBuf &) = delete;
    ~PoolBuf() { release(); }
    void release() {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        n = 0;
    }
    cudaError_t alloc(size_t count, cudaStream_t stream) {
        release();
        n = count;
        s = stream;
        if (count == 0) return cudaSuccess;
        return cudaMallocAsync(reinterpret_cast<void **>(&p), sizeof(T) * count, stream);
    }
};

}  // namespace gcabem

struct gcabem_mesh_s {
    int device = 0;
    int64_t nv = 0, nt = 0;
    cudaStream_t stream = nullptr;
    gcabem::DevBuf<double> V;
    gcabem::DevBuf<int32_t> T;
    gcabem::DevBuf<gcabem::Chart> charts;
};

// Dense host kernels of the GCA operator construction (aca.cpp).
namespace gcabem {
// One cluster: ACA (eps, one tighter retry), pivot-block condition check and
// V = A[:, cols] inv(A[rows, cols]) with two refinement sweeps
// (reference gca.py:182-282). A is nr x nc row-major, real or interleaved
// complex. Returns 0, 1 (zero Green matrix) or 2 (singular pivot block).
int gca_operator(bool is_complex, const double *A, int64_t nr, int64_t nc, double epsilon,
                 std::vector<int64_t> &rows, std::vector<double> &V);
}  // namespace gcabem
