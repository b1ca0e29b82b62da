// GCA interpolation operators of many clusters (reference
// gca.build_interpolation_operators, gca.py:285-310), as one native pipeline:
//
//   device   Green matrices of a batch of clusters (green_box_kernel: sources
//            generated on the device from the enlarged boxes), D2H into a
//            free slot of a ring of pinned staging buffers;
//   host     ACA per cluster (the pivots, aca.cpp) on a thread pool, each
//            worker copying its cluster out of the slot first, while the
//            device computes the next batches;
//   host     the pivot-block check and the refined V solve (gca_operator).
//
// Every ACA decision (argmax of a residual row/column, the stopping test) is
// made on the device's Green matrix, whose entries agree with the
// reference's numpy evaluation to a few ulps; a decision whose margin is
// inside that error (exact ties from the mesh's symmetry, mostly) is FLAGGED
// per cluster (gcabem_gca_flags) so the caller can redo that cluster on a
// bit-exact host evaluation of the reference's Green matrix (gca.py).
//
// Clusters run largest first (the longest host jobs start early: no tail with
// idle threads). North star split: the Green matrices (dense FP64 kernel
// evaluations) are device work, the pivoting (and by default the small
// solves) stays on the CPU.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <memory>
#include <cmath>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "green_exact.h"
#include "internal.h"

using namespace gcabem;

struct gcabem_gca_s {
    int is_complex = 0;
    int64_t ncl = 0;
    std::vector<std::vector<int64_t>> rows;  // local row pivots per cluster
    std::vector<std::vector<double>> V;      // |t| x rank per cluster (row-major)
    std::vector<char> ambiguous;             // an ACA decision within roundoff of a tie
    // device wait, pipeline wall, total, batches, host thread-seconds, threads
    double phase[6] = {0, 0, 0, 0, 0, 0};
};

namespace {

using clk = std::chrono::steady_clock;
double since(clk::time_point t0) {
    return std::chrono::duration<double>(clk::now() - t0).count();
}

// grow-only pinned host buffer
struct Pinned {
    void *p = nullptr;
    size_t n = 0;
    ~Pinned() {
        if (p) cudaFreeHost(p);
    }
    cudaError_t reserve(size_t bytes) {
        if (bytes <= n && p) return cudaSuccess;
        if (p) cudaFreeHost(p);
        p = nullptr;
        n = 0;
        cudaError_t e = cudaHostAlloc(&p, bytes, cudaHostAllocPortable);
        if (e == cudaSuccess) n = bytes;
        return e;
    }
};

// Staging buffers survive across calls (per device): pinned allocation of
// hundreds of MB costs more than a whole L6 GCA build.
constexpr int SLOTS = 4;  // batches in flight: device output + pinned staging each
constexpr int64_t INPLACE_ROWS = 256;  // clusters up to this size run ACA in the slot

struct Staging {
    Pinned host[SLOTS];
    DevBuf<double> out[SLOTS];
    std::vector<std::vector<double>> aown;  // per worker: its cluster's Green matrix
    std::mutex busy;  // one build per device at a time (builds on other devices run in parallel)
};
std::mutex g_staging_mutex;
std::vector<Staging *> g_staging;  // indexed by device

Staging &staging_for(int device) {
    std::lock_guard<std::mutex> lock(g_staging_mutex);
    if ((int)g_staging.size() <= device) g_staging.resize(device + 1, nullptr);
    if (!g_staging[device]) g_staging[device] = new Staging();
    return *g_staging[device];
}

}  // namespace

void gcabem::gca_release_staging(int device) {
    Staging *st = nullptr;
    {
        std::lock_guard<std::mutex> lock(g_staging_mutex);
        if (device < (int)g_staging.size()) std::swap(st, g_staging[device]);
    }
    if (st) {
        std::lock_guard<std::mutex> busy(st->busy);  // wait for a running build
    }
    delete st;
}

extern "C" {

int gcabem_gca_build(gcabem_mesh_t mesh, int equation, double kappa, int64_t ncl,
                     const int64_t *cl_ids, const int64_t *cl_first, const int64_t *cl_size,
                     const double *box_lo,
                     const double *box_hi, int64_t nperm, const int64_t *perm, double delta,
                     int m, const double *gauss_pts, const double *gauss_wts,
                     double scene_diameter, int64_t nduffy, const double *duffy, double epsilon,
                     int nthreads, int64_t batch_bytes, gcabem_gca_t *out) {
    if (!mesh || !out) return gcabem_internal_error(GCABEM_ERR_ARG, "null argument");
    *out = nullptr;
    if (!(equation == 0 || equation == 1) || (equation == 1 && kappa < 0.0))
        return gcabem_internal_error(GCABEM_ERR_ARG, "bad equation or kappa");
    if (ncl < 0 || m < 1 || nduffy < 1 || !(delta > 0.0) || !(epsilon > 0.0))
        return gcabem_internal_error(GCABEM_ERR_ARG, "bad GCA parameters");
    const int64_t nsrc = 12 * (int64_t)m * m, ng = nsrc / 2;
    const int width = equation == 0 ? 1 : 2;
    const auto t_all = clk::now();
    Trace tr("gca");
    auto *G = new gcabem_gca_s();
    G->is_complex = equation == 1;
    G->ncl = ncl;
    G->rows.resize(ncl);
    G->V.resize(ncl);
    G->ambiguous.assign(ncl, 0);
    std::vector<int32_t> perm32(nperm);
    for (int64_t k = 0; k < nperm; ++k) {
        if (perm[k] < 0 || perm[k] >= mesh->nt) {
            delete G;
            return gcabem_internal_error(GCABEM_ERR_ARG, "panel index out of range");
        }
        perm32[k] = (int32_t)perm[k];
    }
    // enlarged boxes, in the reference's operation order (gca.py:103-107)
    std::vector<GreenBox> boxes(ncl);
    for (int64_t c = 0; c < ncl; ++c) {
        const double *lo = box_lo + 3 * c, *hi = box_hi + 3 * c;
        if (cl_size[c] < 1 || cl_first[c] < 0 || cl_first[c] + cl_size[c] > nperm) {
            delete G;
            return gcabem_internal_error(GCABEM_ERR_ARG, "cluster panel range out of bounds");
        }
        double ext = hi[0] - lo[0];
        ext = std::max(ext, hi[1] - lo[1]);
        ext = std::max(ext, hi[2] - lo[2]);
        const double hmax = 0.5 * std::max(ext, 1e-8 * scene_diameter);
        if (!(hmax > 0.0)) {
            delete G;
            return gcabem_internal_error(GCABEM_ERR_ARG,
                                         "degenerate box with no scene diameter to fall back on");
        }
        for (int k = 0; k < 3; ++k) {
            boxes[c].center[k] = 0.5 * (lo[k] + hi[k]);
            const double dh = delta * hmax;
            boxes[c].half[k] = 0.5 * (hi[k] - lo[k]) + dh;
        }
    }
    tr.mark("boxes");
    // processing order: largest clusters first (their host work is the
    // longest; issued last they would leave a tail with most threads idle),
    // ties by index. Everything below is indexed by position in this order.
    std::vector<int64_t> ord(ncl);
    for (int64_t c = 0; c < ncl; ++c) ord[c] = c;
    std::stable_sort(ord.begin(), ord.end(),
                     [&](int64_t a, int64_t b) { return cl_size[a] > cl_size[b]; });
    // batches of consecutive positions by output bytes
    const int64_t row_bytes = nsrc * 8 * width;
    if (batch_bytes <= 0) batch_bytes = int64_t(32) << 20;
    std::vector<int64_t> bstart{0};
    {
        int64_t acc = 0;
        for (int64_t c = 0; c < ncl; ++c) {
            const int64_t b = cl_size[ord[c]] * row_bytes;
            if (acc > 0 && acc + b > batch_bytes) {
                bstart.push_back(c);
                acc = 0;
            }
            acc += b;
        }
        bstart.push_back(ncl);
    }
    const int64_t nb = (int64_t)bstart.size() - 1;
    int64_t max_elems = 0;
    std::vector<std::vector<int64_t>> out_at(nb);
    std::vector<std::vector<int2>> tasks(nb);
    for (int64_t b = 0; b < nb; ++b) {
        int64_t acc = 0;
        for (int64_t c = bstart[b]; c < bstart[b + 1]; ++c) {
            out_at[b].push_back(acc);
            const int64_t ne = cl_size[ord[c]] * ng;
            if (ne >= (int64_t(1) << 31)) {
                delete G;
                return gcabem_internal_error(GCABEM_ERR_ARG, "cluster too large");
            }
            for (int64_t e0 = 0; e0 < ne; e0 += GREEN_TPB)
                tasks[b].push_back(make_int2((int)(c - bstart[b]), (int)e0));
            acc += cl_size[ord[c]] * nsrc;
        }
        max_elems = std::max(max_elems, acc);
    }
    if (nthreads <= 0) nthreads = (int)std::max(1u, std::thread::hardware_concurrency());
    tr.mark("batches");

    cudaError_t e = cudaSetDevice(mesh->device);
    cudaStream_t s = mesh->stream;
    Staging &st = staging_for(mesh->device);
    std::lock_guard<std::mutex> build_lock(st.busy);
    // per-call buffers from the device pool (stream-ordered: no implicit
    // device-wide synchronisation on free)
    if (e == cudaSuccess) e = pool_init(mesh->device);
    PoolBuf<int64_t> d_first, d_at;
    PoolBuf<int32_t> d_size, d_perm;
    PoolBuf<GreenBox> d_box;
    PoolBuf<double> d_gq, d_duffy;
    PoolBuf<int2> d_task;
    std::vector<int64_t> first(ncl);
    std::vector<int32_t> size32(ncl);
    std::vector<GreenBox> box_ord(ncl);
    for (int64_t c = 0; c < ncl; ++c) {
        first[c] = cl_first[ord[c]];
        size32[c] = (int32_t)cl_size[ord[c]];
        box_ord[c] = boxes[ord[c]];
    }
    std::vector<double> gq(2 * m);
    for (int k = 0; k < m; ++k) {
        gq[k] = gauss_pts[k];
        gq[m + k] = gauss_wts[k];
    }
    if (e == cudaSuccess) e = d_first.upload(first.data(), ncl, s);
    if (e == cudaSuccess) e = d_size.upload(size32.data(), ncl, s);
    if (e == cudaSuccess) e = d_perm.upload(perm32.data(), nperm, s);
    if (e == cudaSuccess) e = d_box.upload(box_ord.data(), ncl, s);
    if (e == cudaSuccess) e = d_gq.upload(gq.data(), gq.size(), s);
    if (e == cudaSuccess) e = d_duffy.upload(duffy, 3 * nduffy, s);
    size_t max_tasks = 0, max_cl = 0;
    for (int64_t b = 0; b < nb; ++b) {
        max_tasks = std::max(max_tasks, tasks[b].size());
        max_cl = std::max(max_cl, out_at[b].size());
    }
    if (e == cudaSuccess) e = d_task.alloc(max_tasks * SLOTS, s);
    if (e == cudaSuccess) e = d_at.alloc(max_cl * SLOTS, s);
    tr.mark("uploads");
    for (int k = 0; k < SLOTS && e == cudaSuccess; ++k) {
        e = st.out[k].reserve((size_t)(max_elems * width));
        if (e == cudaSuccess) e = st.host[k].reserve((size_t)(max_elems * width) * 8);
    }
    tr.mark("staging");
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    tr.mark("sync");
    cudaEvent_t done[SLOTS] = {};
    for (int k = 0; k < SLOTS && e == cudaSuccess; ++k)
        e = cudaEventCreateWithFlags(&done[k], cudaEventDisableTiming | cudaEventBlockingSync);

    // batch b uses slot slot_of[b] (tasks, offsets, device output, staging),
    // taken from the free list when the batch is issued
    std::vector<int> slot_of(nb, -1);
    auto enqueue = [&](int64_t b, int k) -> cudaError_t {
        slot_of[b] = k;
        int2 *tk = d_task.p + k * max_tasks;
        int64_t *at = d_at.p + k * max_cl;
        cudaError_t r = cudaMemcpyAsync(tk, tasks[b].data(), sizeof(int2) * tasks[b].size(),
                                        cudaMemcpyHostToDevice, s);
        if (r == cudaSuccess)
            r = cudaMemcpyAsync(at, out_at[b].data(), sizeof(int64_t) * out_at[b].size(),
                                cudaMemcpyHostToDevice, s);
        const int64_t c0 = bstart[b];
        if (r == cudaSuccess)
            r = launch_green_box(equation, mesh->charts.p, tk, (int64_t)tasks[b].size(),
                                 d_first.p + c0, d_size.p + c0, d_perm.p, d_box.p + c0, m, d_gq.p,
                                 d_duffy.p, (int)nduffy, at, st.out[k].p, kappa, s);
        int64_t elems = 0;
        for (int64_t c = bstart[b]; c < bstart[b + 1]; ++c) elems += cl_size[ord[c]] * nsrc;
        if (r == cudaSuccess)
            r = cudaMemcpyAsync(st.host[k].p, st.out[k].p, sizeof(double) * elems * width,
                                cudaMemcpyDeviceToHost, s);
        if (r == cudaSuccess) r = cudaEventRecord(done[k], s);
        return r;
    };

    // Workers pull clusters in batch order from one queue and copy their
    // cluster's Green matrix out of the staging slot before working on it, so
    // a slot is free again as soon as all its clusters are claimed (no
    // per-batch barrier, no wait on the slowest cluster); the calling thread
    // issues batches into whichever slots are free (a slot held by the long
    // copy-out of a large cluster does not stall the others) and publishes
    // each batch when its D2H has landed.
    std::vector<int64_t> batch_of(ncl);
    for (int64_t b = 0; b < nb; ++b)
        for (int64_t c = bstart[b]; c < bstart[b + 1]; ++c) batch_of[c] = b;
    std::unique_ptr<std::atomic<int64_t>[]> remaining(new std::atomic<int64_t>[nb > 0 ? nb : 1]);
    for (int64_t b = 0; b < nb; ++b) remaining[b] = bstart[b + 1] - bstart[b];
    std::vector<char> ready(nb, 0);
    std::vector<int> free_slots;
    for (int k = SLOTS - 1; k >= 0; --k) free_slots.push_back(k);
    std::mutex mu;
    std::condition_variable cv;
    bool abort = false;
    std::atomic<int64_t> next{0};
    std::atomic<int64_t> err_cluster{INT64_MAX};
    std::atomic<int> err_code{0};
    std::vector<double> busy(nthreads, 0.0), first_at(nthreads, -1.0), last_at(nthreads, 0.0),
        starved(nthreads, 0.0);
    const auto t_start = clk::now();
    if ((int)st.aown.size() < nthreads) st.aown.resize(nthreads);
    std::atomic<int64_t> n_host{0}, n_exact{0};
    auto fail = [&](int64_t c, int rc) {
        int64_t prev = err_cluster.load();
        while (c < prev && !err_cluster.compare_exchange_weak(prev, c)) {
        }
        if (c <= err_cluster.load()) err_code = rc;
    };
    auto worker = [&](int tid) {
        std::vector<double> &Aown = st.aown[tid];  // grow-only across calls: no page faults
        for (;;) {
            const int64_t pos = next.fetch_add(1);
            if (pos >= ncl) return;
            const int64_t b = batch_of[pos], c = ord[pos];
            const auto tw = clk::now();
            {
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [&] { return ready[b] || abort; });
                if (abort) return;
            }
            const auto t0 = clk::now();
            starved[tid] += std::chrono::duration<double>(t0 - tw).count();
            if (first_at[tid] < 0.0) first_at[tid] = std::chrono::duration<double>(t0 - t_start).count();
            const double *A = static_cast<const double *>(st.host[slot_of[b]].p) +
                              out_at[b][pos - bstart[b]] * width;
            const int64_t nr = cl_size[c];
            auto release = [&] {
                if (remaining[b].fetch_sub(1) == 1) {  // slot drained: back to the free list
                    std::lock_guard<std::mutex> lk(mu);
                    free_slots.push_back(slot_of[b]);
                    cv.notify_all();
                }
            };
            // a small cluster works on its matrix in the slot (done in well
            // under a millisecond; its copy would cost a fifth of its ACA); a
            // large one copies it out first, so that its long ACA does not
            // hold the slot
            const bool inplace = nr <= INPLACE_ROWS;
            if (!inplace) {
                Aown.assign(A, A + nr * nsrc * width);
                release();
            }
            int amb = 0;
            int rc = gca_operator(equation == 1, inplace ? A : Aown.data(), nr, nsrc, epsilon,
                                  G->rows[c], G->V[c], &amb);
            if (inplace) release();
            if (rc == 0 && amb) {
                // a decision inside the tie window: redo this cluster on
                // entries evaluated in the reference's own arithmetic
                GreenExact ge;
                ge.charts = mesh->charts_host.data();
                ge.panels = perm32.data() + cl_first[c];
                ge.nr = nr;
                ge.equation = equation;
                ge.kappa = kappa;
                ge.duffy = duffy;
                ge.nq = (int)nduffy;
                ge.m = m;
                ge.sources(boxes[c], gauss_pts, gauss_wts);
                rc = gca_operator_exact(equation == 1, ge, epsilon, G->rows[c], G->V[c]);
                n_exact.fetch_add(1);
            }
            G->ambiguous[c] = (char)amb;
            n_host.fetch_add(1);
            if (rc != 0) fail(c, rc);
            busy[tid] += since(t0);
            last_at[tid] = since(t_start);
        }
    };
    double t_wait = 0.0;
    const auto t_pipe = clk::now();
    std::vector<std::thread> th;
    if (e == cudaSuccess) {
        for (int t = 0; t < nthreads; ++t) th.emplace_back(worker, t);
    }
    int64_t issued = 0, completed = 0;
    while (e == cudaSuccess && completed < nb) {
        for (;;) {
            int k = -1;
            {
                std::lock_guard<std::mutex> lk(mu);
                if (issued < nb && !free_slots.empty()) {
                    k = free_slots.back();
                    free_slots.pop_back();
                }
            }
            if (k < 0) break;
            e = enqueue(issued++, k);
            if (e != cudaSuccess) break;
        }
        if (e != cudaSuccess) break;
        if (completed < issued) {
            // publish the oldest batch once its D2H has landed; meanwhile a
            // slot freed by the workers is refilled at once (a blocking wait
            // on the event would leave it empty until the batch lands)
            const auto t0 = clk::now();
            const cudaError_t q = cudaEventQuery(done[slot_of[completed]]);
            if (q == cudaErrorNotReady) {
                std::unique_lock<std::mutex> lk(mu);
                cv.wait_for(lk, std::chrono::microseconds(100),
                            [&] { return !free_slots.empty() && issued < nb; });
                t_wait += since(t0);
                continue;
            }
            e = q;
            t_wait += since(t0);
            std::lock_guard<std::mutex> lk(mu);
            ready[completed++] = 1;
            cv.notify_all();
        } else {
            std::unique_lock<std::mutex> lk(mu);
            cv.wait(lk, [&] { return !free_slots.empty(); });
        }
    }
    if (e != cudaSuccess) {
        std::lock_guard<std::mutex> lk(mu);
        abort = true;
        cv.notify_all();
    }
    for (auto &t : th) t.join();
    tr.mark("pipeline");
    if (tr.on) {
        int64_t namb = 0;
        for (char x : G->ambiguous) namb += x;
        std::fprintf(stderr, "[gca] %lld clusters, %lld with a decision inside the tie window\n",
                     (long long)n_host.load(), (long long)namb);
    }
    if (tr.on && nthreads > 0)
        std::fprintf(stderr, "[gca] workers: first cluster %.1f-%.1f ms, last done %.1f-%.1f ms, "
                     "waiting for Green batches %.1f ms (all threads)\n",
                     1e3 * *std::min_element(first_at.begin(), first_at.end()),
                     1e3 * *std::max_element(first_at.begin(), first_at.end()),
                     1e3 * *std::min_element(last_at.begin(), last_at.end()),
                     1e3 * *std::max_element(last_at.begin(), last_at.end()),
                     1e3 * std::accumulate(starved.begin(), starved.end(), 0.0));
    double t_host = 0.0;
    for (double x : busy) t_host += x;
    G->phase[1] = since(t_pipe);
    cudaStreamSynchronize(s);
    for (auto &d : done)
        if (d) cudaEventDestroy(d);
    tr.mark("sync+events");
    if (e != cudaSuccess) {
        delete G;
        return gcabem_internal_error(GCABEM_ERR_CUDA,
                                     (std::string("gca build: ") + cudaGetErrorString(e)).c_str());
    }
    if (err_code.load() != 0) {
        const int64_t c = err_cluster.load();
        const std::string id = std::to_string(cl_ids ? cl_ids[c] : c);
        const std::string msg =
            err_code.load() == 1
                ? "cluster " + id + ": zero Green matrix"
                : "cluster " + id + ": singular ACA pivot block (condition above 1e+14)";
        delete G;
        return gcabem_internal_error(GCABEM_ERR_GCA, msg.c_str());
    }
    d_first.release();
    d_at.release();
    d_size.release();
    d_perm.release();
    d_box.release();
    d_gq.release();
    d_duffy.release();
    d_task.release();
    tr.mark("finish");
    G->phase[0] = t_wait;
    G->phase[2] = since(t_all);
    G->phase[3] = (double)nb;
    G->phase[4] = t_host;
    G->phase[5] = (double)nthreads;
    tr.mark("return");
    *out = G;
    return GCABEM_OK;
}

int gcabem_gca_sizes(gcabem_gca_t G, int64_t *ranks, double *phase4) {
    if (!G) return gcabem_internal_error(GCABEM_ERR_ARG, "null handle");
    for (int64_t c = 0; c < G->ncl; ++c) ranks[c] = (int64_t)G->rows[c].size();
    if (phase4)
        for (int k = 0; k < 6; ++k) phase4[k] = G->phase[k];
    return GCABEM_OK;
}

int gcabem_gca_flags(gcabem_gca_t G, int8_t *ambiguous) {
    if (!G || !ambiguous) return gcabem_internal_error(GCABEM_ERR_ARG, "null argument");
    for (int64_t c = 0; c < G->ncl; ++c) ambiguous[c] = (int8_t)G->ambiguous[c];
    return GCABEM_OK;
}

int gcabem_gca_fetch(gcabem_gca_t G, int64_t *rows, double *V) {
    if (!G) return gcabem_internal_error(GCABEM_ERR_ARG, "null handle");
    // offsets, then a threaded copy (the caller's fresh buffer is
    // page-faulted by the copying threads in parallel)
    std::vector<int64_t> ro(G->ncl + 1, 0), vo(G->ncl + 1, 0);
    for (int64_t c = 0; c < G->ncl; ++c) {
        ro[c + 1] = ro[c] + (int64_t)G->rows[c].size();
        vo[c + 1] = vo[c] + (int64_t)G->V[c].size();
    }
    const int nt = (int)std::min<int64_t>(16, std::max<int64_t>(1, G->ncl / 256));
    std::atomic<int64_t> next{0};
    auto work = [&]() {
        for (;;) {
            const int64_t c0 = next.fetch_add(64);
            if (c0 >= G->ncl) return;
            for (int64_t c = c0; c < std::min<int64_t>(G->ncl, c0 + 64); ++c) {
                std::copy(G->rows[c].begin(), G->rows[c].end(), rows + ro[c]);
                std::copy(G->V[c].begin(), G->V[c].end(), V + vo[c]);
            }
        }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < nt; ++t) th.emplace_back(work);
    work();
    for (auto &t : th) t.join();
    return GCABEM_OK;
}

int gcabem_gca_free(gcabem_gca_t G) {
    // hundreds of MB in thousands of blocks: release them off the caller's path
    if (G) std::thread([G]() { delete G; }).detach();
    return GCABEM_OK;
}

}  // extern "C"
