// Host-side internals shared by the C ABI translation units (api.cu,
// gca_pipeline.cu): the device mesh replica and an RAII device buffer.
#pragma once
#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <atomic>
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
// free the GCA pipeline's staging ring of `device` (gca_pipeline.cu)
void gca_release_staging(int device);

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
    cudaError_t upload(const T *host, size_t count, cudaStream_t stream) {
        cudaError_t e = alloc(count, stream);
        if (e != cudaSuccess || count == 0) return e;
        return cudaMemcpyAsync(p, host, sizeof(T) * count, cudaMemcpyHostToDevice, stream);
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
    std::vector<gcabem::Chart> charts_host;
};

// Device layout of one package set: uploaded once, shared by every plan
// (operator) assembled from the same packages (e.g. SLP and DLP).
struct gcabem_layout_s {
    gcabem_mesh_t mesh = nullptr;
    int64_t payload_len = 0;
    // stream-ordered pool allocations (layouts are created per assembly call)
    gcabem::PoolBuf<gcabem::BlockDesc> blocks;
    gcabem::PoolBuf<int2> tasks;
    int64_t ntasks = 0;
    // mirrored evaluation (gcabem::BlockRole): tasks of ROLE_PRIMARY/SELF
    // blocks (mirrored kernel) and of ROLE_NORMAL blocks (plain kernel);
    // ROLE_SKIP blocks have none. Empty when no leaf has a mirror.
    gcabem::PoolBuf<int2> mtasks, rtasks;
    // the same three task lists as TaskDesc records (block descriptor + first
    // pair) for the disjoint kernels (task_desc_kernel, at layout creation)
    gcabem::PoolBuf<gcabem::TaskDesc> tdesc, mtdesc, rtdesc;
    int64_t nmtasks = 0, nrtasks = 0;
    std::vector<int64_t> block_mtask_at, block_rtask_at;
    // {evaluations by the mirrored kernel, by the plain kernel (pairs sharing
    // a vertex excluded), pairs of PRIMARY/SELF blocks, pairs of SKIP blocks}
    int64_t mirror_info[4] = {0, 0, 0, 0};
    // vertex items split for mirrored execution (the vertex rule is symmetric):
    // vm = items of PRIMARY / SELF-upper positions, each also writing its
    // transpose at vm_mout; vp = items of NORMAL leaves (alone); the items of
    // SKIP / SELF-lower positions are written by their partners. Empty unless
    // every partner was found.
    gcabem::PoolBuf<gcabem::SingItem> vm_items, vp_items;
    gcabem::PoolBuf<int64_t> vm_mout;
    std::vector<int64_t> vm_out, vp_out;
    bool vertex_mirror = false;
    // symmetric download of a mirrored single layer (gcabem_plan_set_symmetric_
    // download): the SKIP leaves of runs of at least SYM_MIN_RUN payload
    // entries are not copied; the host writes each as the transpose of its
    // PRIMARY (the mirrored kernels write one value to both entries), then its
    // singular entries (written by their own items: the edge rule is not
    // symmetric) from a device gather. Per such leaf, in payload order: its
    // start, shape and its PRIMARY's start; its singular entries are
    // patch_out[hf_item_at[s], hf_item_at[s + 1]) (payload indices).
    std::vector<int64_t> hf_lo, hf_m, hf_item_at, patch_out;
    std::vector<int32_t> hf_nr, hf_nc;
    gcabem::PoolBuf<int64_t> patch_dev;
    gcabem::PoolBuf<int32_t> panels;
    gcabem::PoolBuf<gcabem::SingItem> items;
    int64_t case_at[4] = {0, 0, 0, 0};  // items of case c at [case_at[c-1], case_at[c])
    // host copies for chunked execution
    std::vector<int64_t> block_task_at, block_leaf, block_base, block_pairs, item_out;
    std::atomic<int> refs{1};
};

// Dense host kernels of the GCA operator construction (aca.cpp).
namespace gcabem {
// One cluster: ACA (eps, one tighter retry), pivot-block condition check and
// V = A[:, cols] inv(A[rows, cols]) with two refinement sweeps
// (reference gca.py:182-282). A is nr x nc row-major, real or interleaved
// complex. Returns 0, 1 (zero Green matrix) or 2 (singular pivot block).
// ambiguous (optional): set to 1 when an ACA decision fell inside the tie
// window (aca.cpp TIE_REL/TIE_ABS/STOP_REL).
int gca_operator(bool is_complex, const double *A, int64_t nr, int64_t nc, double epsilon,
                 std::vector<int64_t> &rows, std::vector<double> &V, int *ambiguous = nullptr);
// The same operator with every entry evaluated on the host in the
// reference's numpy arithmetic (green_exact.h), on demand: the redo of a
// cluster whose ACA on the device's Green matrix was ambiguous.
struct GreenExact;
int gca_operator_exact(bool is_complex, const GreenExact &g, double epsilon,
                       std::vector<int64_t> &rows, std::vector<double> &V);
// The first attempt's ACA alone: pivots into rows/cols (capacity min(nr, nc)),
// returns the rank.
int64_t gca_aca(bool is_complex, const double *A, int64_t nr, int64_t nc, double epsilon,
                int64_t *rows, int64_t *cols);
}  // namespace gcabem
