// Device V solves of the GCA pipeline (gca_pipeline.cu): the workers hand
// each cluster's pivot block and pivot columns to the pack being filled
// (gathered straight into its pinned buffer); one launcher thread sends full
// packs to the device (vsolve.cu) and harvests the finished ones into the
// build's rows / V. Workers never wait on the device for a small cluster:
// with no pack free they solve on the host; large clusters (whose host solve
// costs more than the wait) wait for a pack. Clusters the device hands back
// (singular pivot block, condition bracket ambiguous) are listed for the
// host's exact decision.
#pragma once
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <vector>

#include "internal.h"

namespace gcabem {
namespace gca_detail {

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

constexpr int VPACKS = 8;
constexpr int64_t VS_PACK_BYTES = int64_t(8) << 20;  // input bytes per launch
constexpr int64_t VS_WAIT_WORK = 256 * 32;           // nr x k from which a worker waits for a pack

enum VState { V_FREE, V_FILLING, V_SEALED, V_INFLIGHT };

struct VItem {
    int64_t c, out_off, nr, k;
    std::vector<int64_t> rows;
};

template <typename T>
cudaError_t pool_reserve(PoolBuf<T> &b, size_t n, cudaStream_t s) {
    return (b.p && b.n >= n) ? cudaSuccess : b.alloc(std::max<size_t>(n, 1), s);
}

struct VPack {
    // hin: the pivot blocks and columns the workers gather, H2D at launch;
    // V comes back into the same buffer (stream order: the H2D is done
    // before the kernels, V is never larger than the input)
    Pinned hin, haux, htk;
    PoolBuf<double> din, dout, dscr;
    PoolBuf<VAux> daux;
    PoolBuf<VTask> dtk;
    PoolBuf<int2> dch;
    cudaEvent_t ev = nullptr;
    VState state = V_FREE;
    int64_t seq = 0;
    int writers = 0;
    std::vector<VItem> items;
    std::vector<VTask> tasks;
    std::vector<int2> chunks;
    int64_t in_len = 0, out_len = 0, scr_len = 0;
    int kmax = 0;
    void reset() {
        items.clear();
        tasks.clear();
        chunks.clear();
        in_len = out_len = scr_len = 0;
        kmax = 0;
        writers = 0;
    }
};

// the packs and their stream, kept per device across builds
struct VRing {
    cudaStream_t s = nullptr;
    VPack pack[VPACKS];
    cudaError_t init() {
        cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
        for (auto &p : pack)
            if (e == cudaSuccess)
                e = cudaEventCreateWithFlags(&p.ev, cudaEventDisableTiming | cudaEventBlockingSync);
        return e;
    }
    ~VRing() {
        for (auto &p : pack) {
            p.din.release();
            p.dout.release();
            p.dscr.release();
            p.daux.release();
            p.dtk.release();
            p.dch.release();
            if (p.ev) cudaEventDestroy(p.ev);
        }
        if (s) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    }
};

// One build's use of the ring. offload() from the workers, run() on the
// launcher thread until workers_finished() and every pack is harvested.
class VSolveQueue {
  public:
    VSolveQueue(VRing &ring, int device, bool is_complex, int64_t nsrc,
                std::vector<std::vector<int64_t>> &rows, std::vector<std::vector<double>> &V)
        : r_(ring), device_(device), cplx_(is_complex), width_(is_complex ? 2 : 1), nsrc_(nsrc),
          rows_(rows), V_(V) {
        // test hooks: every device solve handed back (the retry pass); every
        // cluster solved on the host from its pivots (the no-pack path)
        force_retry_ = std::getenv("GCABEM_GCA_FORCE_RETRY") != nullptr;
        force_fallback_ = std::getenv("GCABEM_GCA_FORCE_FALLBACK") != nullptr;
    }

    // hand cluster c (Green matrix A, nr x nsrc; ACA pivots) to the device;
    // false: solve it on the host
    bool offload(int64_t c, const double *A, int64_t nr, int64_t k, const int64_t *prow,
                 const int64_t *pcol) {
        if (force_fallback_) return false;
        const int64_t need = (k * k + k * nr) * width_;
        VPack *p = nullptr;
        int64_t in_off = 0;
        {
            std::unique_lock<std::mutex> lk(mu_);
            for (;;) {
                if (cur_ && cur_->in_len + need > (int64_t)(cur_->hin.n / 8)) {
                    cur_->state = V_SEALED;  // full: to the launcher
                    cur_ = nullptr;
                    cv_.notify_all();
                }
                if (!cur_) {
                    VPack *f = take_pack();
                    // room for a full pack plus one more cluster (packs seal
                    // at VS_PACK_BYTES rather than on the first cluster that
                    // misses); the pinned allocation happens outside the lock
                    // with the pack private to this worker, so the others
                    // keep going (first build of a process)
                    if (f && (int64_t)(f->hin.n / 8) < std::max(need, VS_PACK_BYTES / 8)) {
                        lk.unlock();
                        const cudaError_t e =
                            f->hin.reserve((size_t)std::max(need * 8, 2 * VS_PACK_BYTES));
                        lk.lock();
                        if (e != cudaSuccess || cur_) {  // failed, or another pack took over
                            f->state = V_FREE;
                            if (e != cudaSuccess) return false;
                            continue;
                        }
                    }
                    cur_ = f;
                }
                if (cur_) break;
                if (nr * k < VS_WAIT_WORK || err_.load() != 0) return false;
                cv_.wait(lk);
            }
            p = cur_;
            in_off = p->in_len;
            VTask tk;
            tk.in_off = in_off;
            tk.out_off = p->out_len;
            tk.scr_off = p->scr_len;
            tk.nr = (int32_t)nr;
            tk.k = (int32_t)k;
            for (int64_t q0 = 0; q0 < nr; q0 += VS_ROWS)
                p->chunks.push_back(make_int2((int)p->tasks.size(), (int)q0));
            p->tasks.push_back(tk);
            p->items.push_back(VItem{c, p->out_len, nr, k, std::vector<int64_t>(prow, prow + k)});
            p->in_len += need;
            p->out_len += nr * k * width_;
            p->scr_len += vsolve_scratch(k, nr, width_);
            p->kmax = std::max(p->kmax, (int)k);
            ++p->writers;
            if (p->in_len * 8 >= VS_PACK_BYTES) {
                p->state = V_SEALED;
                cur_ = nullptr;
            }
        }
        // B = A[rows, cols] and A[:, cols]^T, gathered into the pinned buffer
        double *dst = static_cast<double *>(p->hin.p) + in_off;
        for (int64_t a = 0; a < k; ++a)
            for (int64_t b = 0; b < k; ++b) {
                const double *src = A + (prow[a] * nsrc_ + pcol[b]) * width_;
                for (int t = 0; t < width_; ++t) *dst++ = src[t];
            }
        for (int64_t b = 0; b < k; ++b)
            for (int64_t q = 0; q < nr; ++q) {
                const double *src = A + (q * nsrc_ + pcol[b]) * width_;
                for (int t = 0; t < width_; ++t) *dst++ = src[t];
            }
        std::lock_guard<std::mutex> lk(mu_);
        if (--p->writers == 0 && p->state == V_SEALED) cv_.notify_all();
        return true;
    }

    // launcher thread: sealed packs (all writers done) to the device, oldest
    // first; finished packs harvested; after the workers the partial pack too
    void run() {
        cudaSetDevice(device_);
        for (;;) {
            VPack *todo = nullptr;
            bool inflight = false, pending = false;
            {
                std::unique_lock<std::mutex> lk(mu_);
                if (done_ && cur_ && cur_->writers == 0) {
                    cur_->state = cur_->items.empty() ? V_FREE : V_SEALED;
                    cur_ = nullptr;
                }
                for (auto &p : r_.pack) {
                    if (p.state == V_SEALED && p.writers == 0 && (!todo || p.seq < todo->seq))
                        todo = &p;
                    inflight = inflight || p.state == V_INFLIGHT;
                    pending = pending || p.state == V_SEALED || p.state == V_FILLING;
                }
                if (todo) todo->state = V_INFLIGHT;
                if (!todo && !inflight) {
                    if (done_ && !pending) return;
                    cv_.wait_for(lk, std::chrono::microseconds(500));
                    continue;
                }
            }
            const auto t0 = std::chrono::steady_clock::now();
            if (todo) {
                const cudaError_t e = err_.load() == 0 ? launch(*todo) : cudaErrorUnknown;
                if (e != cudaSuccess) {  // not on the device: the build fails, nothing to harvest
                    fail(e);
                    std::lock_guard<std::mutex> lk(mu_);
                    for (auto &it : todo->items) back_.push_back(it.c);
                    todo->reset();
                    todo->state = V_FREE;
                    cv_.notify_all();
                }
            }
            bool harvested = false;
            for (auto &p : r_.pack) {
                {
                    std::lock_guard<std::mutex> lk(mu_);
                    if (p.state != V_INFLIGHT) continue;
                }
                const cudaError_t q = cudaEventQuery(p.ev);
                if (q == cudaErrorNotReady) continue;
                if (q != cudaSuccess) fail(q);
                harvest(p);
                harvested = true;
            }
            busy_s_ += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            if (!todo && !harvested) std::this_thread::sleep_for(std::chrono::microseconds(100));
        }
    }

    void workers_finished() {
        std::lock_guard<std::mutex> lk(mu_);
        done_ = true;
        cv_.notify_all();
    }

    // after run() returned
    std::vector<int64_t> &handed_back() { return back_; }
    int64_t device_solves() const { return n_dev_; }
    double busy_s() const { return busy_s_; }
    cudaError_t error() const { return (cudaError_t)err_.load(); }

  private:
    // a FREE pack as the one being filled (mu_ held); nullptr if none
    VPack *take_pack() {
        for (auto &p : r_.pack)
            if (p.state == V_FREE) {
                p.reset();
                p.state = V_FILLING;
                p.seq = seq_++;
                return &p;
            }
        return nullptr;
    }

    void fail(cudaError_t e) {
        std::lock_guard<std::mutex> lk(mu_);
        if (err_.load() == 0) err_ = (int)e;
        cv_.notify_all();  // waiting workers fall back to the host
    }

    cudaError_t launch(VPack &p) {
        const size_t nt = p.tasks.size(), nch = p.chunks.size();
        const size_t tk_bytes = nt * sizeof(VTask), ch_bytes = nch * sizeof(int2);
        cudaStream_t s = r_.s;
        // pinned buffers grow in steps of at least a pack (cudaHostAlloc /
        // FreeHost cost milliseconds and FreeHost synchronises)
        cudaError_t e = p.htk.reserve(std::max<size_t>(tk_bytes + ch_bytes, size_t(256) << 10));
        if (e == cudaSuccess) e = p.haux.reserve(std::max<size_t>(nt * sizeof(VAux), 64 << 10));
        if (e == cudaSuccess) e = pool_reserve(p.din, (size_t)p.in_len, s);
        if (e == cudaSuccess) e = pool_reserve(p.dout, (size_t)p.out_len, s);
        if (e == cudaSuccess) e = pool_reserve(p.dscr, (size_t)p.scr_len, s);
        if (e == cudaSuccess) e = pool_reserve(p.daux, nt, s);
        if (e == cudaSuccess) e = pool_reserve(p.dtk, nt, s);
        if (e == cudaSuccess) e = pool_reserve(p.dch, nch, s);
        if (e != cudaSuccess) return e;
        char *hb = static_cast<char *>(p.htk.p);
        std::copy(p.tasks.begin(), p.tasks.end(), reinterpret_cast<VTask *>(hb));
        std::copy(p.chunks.begin(), p.chunks.end(), reinterpret_cast<int2 *>(hb + tk_bytes));
        e = cudaMemcpyAsync(p.dtk.p, hb, tk_bytes, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(p.dch.p, hb + tk_bytes, ch_bytes, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(p.din.p, p.hin.p, (size_t)p.in_len * 8, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess)
            e = launch_vsolve(cplx_, p.dtk.p, (int)nt, p.dch.p, (int)nch, p.kmax, p.din.p,
                              p.dout.p, p.dscr.p, p.daux.p, s);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(p.hin.p, p.dout.p, (size_t)p.out_len * 8, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(p.haux.p, p.daux.p, nt * sizeof(VAux), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaEventRecord(p.ev, s);
        return e;
    }

    void harvest(VPack &p) {
        const VAux *ax = static_cast<const VAux *>(p.haux.p);
        const double *o = static_cast<const double *>(p.hin.p);  // V, over the input
        std::vector<int64_t> back;
        for (size_t i = 0; i < p.items.size(); ++i) {
            VItem &it = p.items[i];
            if (ax[i].status == 0 && !force_retry_) {
                rows_[it.c] = std::move(it.rows);
                V_[it.c].assign(o + it.out_off, o + it.out_off + it.nr * it.k * width_);
                ++n_dev_;
            } else {
                back.push_back(it.c);
            }
        }
        std::lock_guard<std::mutex> lk(mu_);
        back_.insert(back_.end(), back.begin(), back.end());
        p.reset();
        p.state = V_FREE;
        cv_.notify_all();  // workers waiting for a pack
    }

    VRing &r_;
    const int device_;
    const bool cplx_;
    const int width_;
    const int64_t nsrc_;
    std::vector<std::vector<int64_t>> &rows_;
    std::vector<std::vector<double>> &V_;
    bool force_retry_ = false, force_fallback_ = false;
    std::mutex mu_;
    std::condition_variable cv_;
    VPack *cur_ = nullptr;  // the pack being filled
    int64_t seq_ = 0;
    bool done_ = false;
    std::atomic<int> err_{0};
    std::vector<int64_t> back_;
    int64_t n_dev_ = 0;      // launcher thread only
    double busy_s_ = 0.0;   // launcher thread only
};

}  // namespace gca_detail
}  // namespace gcabem
