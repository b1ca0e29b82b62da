// C ABI of gcabem_b200 (declared in include/gcabem_b200.h). Host-side
// ownership, uploads, task decomposition and error mapping; no compute here.
#include <cuda_runtime.h>
#include <sched.h>
#include <emmintrin.h>

#include <algorithm>
#include <map>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <cmath>
#include <cstring>
#include <mutex>
#include <thread>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "gcabem_b200.h"
#include "gcabem_common.cuh"
#include "internal.h"

using namespace gcabem;

namespace {

thread_local std::string g_error;


int set_error(int code, const std::string &msg) {
    g_error = msg;
    return code;
}

#define GC_CUDA(call)                                                                     \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return set_error(GCABEM_ERR_CUDA, std::string(#call) + ": " +                 \
                                                  cudaGetErrorString(e_));                \
    } while (0)

#define GC_ARG(cond, msg)                                             \
    do {                                                              \
        if (!(cond)) return set_error(GCABEM_ERR_ARG, (msg));         \
    } while (0)

std::mutex g_rule_mutex;
std::set<std::pair<int, int>> g_rules_loaded;  // (device, order)

// Constant-memory disjoint rule of `order` on `device` (idempotent: the
// tables are functions of the Gauss rule only).
int ensure_disjoint_rule(int device, int order, const double *g, const double *gw) {
    std::lock_guard<std::mutex> lock(g_rule_mutex);
    if (g_rules_loaded.count({device, order})) return GCABEM_OK;
    GC_CUDA(upload_disjoint_rule(order, g, gw));
    GC_CUDA(cudaDeviceSynchronize());
    g_rules_loaded.insert({device, order});
    return GCABEM_OK;
}

int check_kind(int equation, int layer, double kappa) {
    GC_ARG(equation == 0 || equation == 1, "unknown equation");
    GC_ARG(layer == 0 || layer == 1, "unknown layer");
    GC_ARG(!(equation == 1 && kappa < 0.0), "kappa must be >= 0");
    return GCABEM_OK;
}

// Pack an (n,5) generic rule {xs, xt, ys, yt, w} from (q,2),(q,2),(q,) arrays.
std::vector<double> pack_rule(int64_t q, const double *xs, const double *ys, const double *w) {
    std::vector<double> r(5 * q);
    for (int64_t k = 0; k < q; ++k) {
        r[5 * k] = xs[2 * k];
        r[5 * k + 1] = xs[2 * k + 1];
        r[5 * k + 2] = ys[2 * k];
        r[5 * k + 3] = ys[2 * k + 1];
        r[5 * k + 4] = w[k];
    }
    return r;
}

}  // namespace

namespace gcabem {
cudaError_t pool_init(int device) {
    static std::mutex mu;
    static std::set<int> done;
    std::lock_guard<std::mutex> lock(mu);
    if (done.count(device)) return cudaSuccess;
    cudaMemPool_t pool;
    cudaError_t e = cudaDeviceGetDefaultMemPool(&pool, device);
    if (e != cudaSuccess) return e;
    uint64_t keep = UINT64_MAX;
    e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    if (e == cudaSuccess) done.insert(device);
    return e;
}
}  // namespace gcabem

// Error hook for the other translation units (packaging.cpp).
int gcabem_internal_error(int code, const char *msg) { return set_error(code, msg); }


namespace {
// TaskDesc lists of a layout (defined below, next to the other layout kernels)
cudaError_t build_task_descs(gcabem_layout_s *L, cudaStream_t s);
}  // namespace

struct gcabem_plan_s {
    gcabem_mesh_t mesh = nullptr;
    gcabem_layout_t L = nullptr;
    int kind = 0, order = 0;
    double kappa = 0.0;
    int64_t payload_len = 0;
    PoolBuf<double2> payload;
    PoolBuf<double2> payload2;  // pair kinds: the double layer
    PoolBuf<double> srule[3];
    int64_t sq[3] = {0, 0, 0};
    // x-grouped vertex and edge rules (kernels.cu generic_pair_grouped)
    PoolBuf<double> grows[3], ggroups[3];
    PoolBuf<int4> gchunks[3];
    int gn[3] = {0, 0, 0};
    // identical rule: its base half when the terms come in swapped pairs
    PoolBuf<double> hrule;
    int64_t hq = 0;
    cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
    std::vector<cudaEvent_t> chunk_ev;
    cudaStream_t stream = nullptr;  // kernels (own_stream, or the caller's)
    cudaStream_t own_stream = nullptr;
    cudaStream_t copy = nullptr;    // D2H, overlapping later chunks' kernels
    bool executed = false;
    // the layout's mirrored blocks run on the mirrored kernel (orders up to
    // MAX_MIRROR_ORDER; gcabem_plan_set_mirror can turn it off)
    bool mirrored = false;
    // symmetric download of the single layer (gcabem_layout_s::hf_lo): the
    // gathered singular entries of the host-filled leaves (device, pinned
    // host), one event per chunk after its copies, the host thread that
    // fills the leaves chunk by chunk, and the bytes the last download moved
    bool sym = false;
    PoolBuf<double2> patch_vals;
    double2 *patch_host = nullptr;
    size_t patch_host_bytes = 0;
    std::vector<cudaEvent_t> copy_ev;
    std::thread filler;
    int fill_rc = 0;
    std::string fill_msg;
    int64_t d2h_bytes = 0;
};

extern "C" {

int gcabem_version(void) { return 100; }

const char *gcabem_last_error(void) { return g_error.c_str(); }

int gcabem_device_count(int *count) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *count = 0;
        return set_error(GCABEM_ERR_NODEV, std::string("no CUDA device: ") + cudaGetErrorString(e));
    }
    *count = n;
    return GCABEM_OK;
}

int gcabem_device_info(int device, char *name, int *sm_count, int *clock_khz) {
    cudaDeviceProp prop;
    GC_CUDA(cudaGetDeviceProperties(&prop, device));
    if (name) {
        std::strncpy(name, prop.name, 255);
        name[255] = 0;
    }
    if (sm_count) *sm_count = prop.multiProcessorCount;
    if (clock_khz) {
        int clk = 0;
        cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, device);
        *clock_khz = clk;
    }
    return GCABEM_OK;
}

int gcabem_host_alloc(int64_t nbytes, void **ptr) {
    GC_ARG(nbytes >= 0 && ptr, "bad host_alloc arguments");
    *ptr = nullptr;
    if (nbytes == 0) return GCABEM_OK;
    GC_CUDA(cudaHostAlloc(ptr, (size_t)nbytes, cudaHostAllocPortable));
    return GCABEM_OK;
}

int gcabem_host_free(void *ptr) {
    if (ptr) GC_CUDA(cudaFreeHost(ptr));
    return GCABEM_OK;
}

int gcabem_pair_values(int device, int equation, int layer, double kappa, int64_t n,
                       const double *ox, const double *e1x, const double *e2x,
                       const double *gx, const double *oy, const double *e1y,
                       const double *e2y, const double *gy, const double *ny, int64_t nq,
                       const double *xs, const double *ys, const double *w, double *out) {
    if (int rc = check_kind(equation, layer, kappa)) return rc;
    GC_ARG(n >= 0 && nq >= 0, "negative size");
    if (n == 0) return GCABEM_OK;
    GC_CUDA(cudaSetDevice(device));
    std::vector<double> packed(24 * (size_t)n, 0.0);
    for (int64_t i = 0; i < n; ++i) {
        double *p = packed.data() + 24 * i;
        for (int c = 0; c < 3; ++c) {
            p[c] = ox[3 * i + c];
            p[3 + c] = e1x[3 * i + c];
            p[6 + c] = e2x[3 * i + c];
            p[9 + c] = oy[3 * i + c];
            p[12 + c] = e1y[3 * i + c];
            p[15 + c] = e2y[3 * i + c];
            p[18 + c] = ny ? ny[3 * i + c] : 0.0;
        }
        p[21] = gx[i];
        p[22] = gy[i];
    }
    std::vector<double> rule = pack_rule(nq, xs, ys, w);
    cudaStream_t s;
    GC_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    DevBuf<double> dp, dr;
    DevBuf<double2> dout;
    cudaError_t e = dp.upload(packed.data(), packed.size(), s);
    if (e == cudaSuccess) e = dr.upload(rule.data(), rule.size(), s);
    if (e == cudaSuccess) e = dout.alloc(n);
    if (e == cudaSuccess)
        e = launch_raw(kind_of(equation, layer), dp.p, n, dr.p, nq, dout.p, kappa, s);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(out, dout.p, sizeof(double2) * n, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    GC_CUDA(e);
    return GCABEM_OK;
}

int gcabem_mesh_create(int device, int64_t nv, const double *vertices, int64_t nt,
                       const int64_t *triangles, const double *normals, const double *gramians,
                       gcabem_mesh_t *out) {
    GC_ARG(out && nv > 0 && nt > 0, "empty mesh");
    GC_ARG(nv < (int64_t(1) << 31) && nt < (int64_t(1) << 31), "mesh too large for int32 indices");
    *out = nullptr;
    GC_CUDA(cudaSetDevice(device));
    std::vector<int32_t> T(3 * nt);
    std::vector<Chart> charts(nt);
    for (int64_t t = 0; t < nt; ++t) {
        const int64_t i0 = triangles[3 * t], i1 = triangles[3 * t + 1], i2 = triangles[3 * t + 2];
        GC_ARG(i0 >= 0 && i0 < nv && i1 >= 0 && i1 < nv && i2 >= 0 && i2 < nv,
               "triangle index out of range");
        T[3 * t] = (int32_t)i0;
        T[3 * t + 1] = (int32_t)i1;
        T[3 * t + 2] = (int32_t)i2;
        Chart &c = charts[t];
        for (int k = 0; k < 3; ++k) {
            c.o[k] = vertices[3 * i0 + k];
            c.e1[k] = vertices[3 * i1 + k] - vertices[3 * i0 + k];
            c.e2[k] = vertices[3 * i2 + k] - vertices[3 * i1 + k];
            c.n[k] = normals[3 * t + k];
        }
        c.gram = gramians[t];
        // bounding sphere about the centroid (relative to v0: (2 e1 + e2) / 3)
        // and |e1| + |e2|, for the kernels' per-pair guards
        double cen[3], r = 0.0;
        for (int k = 0; k < 3; ++k) cen[k] = (2.0 * c.e1[k] + c.e2[k]) / 3.0;
        auto nrm = [](double x, double y, double z) { return std::sqrt(x * x + y * y + z * z); };
        r = std::max(r, nrm(cen[0], cen[1], cen[2]));
        r = std::max(r, nrm(cen[0] - c.e1[0], cen[1] - c.e1[1], cen[2] - c.e1[2]));
        r = std::max(r, nrm(cen[0] - c.e1[0] - c.e2[0], cen[1] - c.e1[1] - c.e2[1],
                            cen[2] - c.e1[2] - c.e2[2]));
        c.radius = r * (1.0 + 1e-12);  // rounding-safe upper bound
        c.enorm = (nrm(c.e1[0], c.e1[1], c.e1[2]) + nrm(c.e2[0], c.e2[1], c.e2[2])) *
                  (1.0 + 1e-12);
        c.pad = 0.0;
    }
    auto *m = new gcabem_mesh_s();
    m->device = device;
    m->nv = nv;
    m->nt = nt;
    cudaError_t e = cudaStreamCreateWithFlags(&m->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = m->V.upload(vertices, 3 * nv, m->stream);
    if (e == cudaSuccess) e = m->T.upload(T.data(), T.size(), m->stream);
    if (e == cudaSuccess) e = m->charts.upload(charts.data(), charts.size(), m->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(m->stream);
    if (e != cudaSuccess) {
        gcabem_mesh_destroy(m);
        GC_CUDA(e);
    }
    m->charts_host = std::move(charts);  // host evaluations (GCA tie redo)
    *out = m;
    return GCABEM_OK;
}

int gcabem_mesh_destroy(gcabem_mesh_t mesh) {
    if (!mesh) return GCABEM_OK;
    cudaSetDevice(mesh->device);
    if (mesh->stream) cudaStreamSynchronize(mesh->stream);
    mesh->V.release();
    mesh->T.release();
    mesh->charts.release();
    if (mesh->stream) cudaStreamDestroy(mesh->stream);
    delete mesh;
    return GCABEM_OK;
}

int gcabem_batch_quadrature(gcabem_mesh_t mesh, int equation, int layer, double kappa,
                            int64_t n, const int64_t *tri_x, const int64_t *tri_y,
                            const uint8_t *perm_x, const uint8_t *perm_y, int64_t nq,
                            const double *xs, const double *ys, const double *w, double *out) {
    GC_ARG(mesh, "null mesh");
    if (int rc = check_kind(equation, layer, kappa)) return rc;
    if (n == 0) return GCABEM_OK;
    GC_CUDA(cudaSetDevice(mesh->device));
    std::vector<SingItem> items(n);
    for (int64_t i = 0; i < n; ++i) {
        GC_ARG(tri_x[i] >= 0 && tri_x[i] < mesh->nt && tri_y[i] >= 0 && tri_y[i] < mesh->nt,
               "triangle index out of range");
        SingItem &it = items[i];
        std::memset(&it, 0, sizeof it);
        it.out = i;
        it.tri_x = (int32_t)tri_x[i];
        it.tri_y = (int32_t)tri_y[i];
        for (int k = 0; k < 3; ++k) {
            it.px[k] = perm_x ? perm_x[3 * i + k] : (uint8_t)k;
            it.py[k] = perm_y ? perm_y[3 * i + k] : (uint8_t)k;
            GC_ARG(it.px[k] < 3 && it.py[k] < 3, "bad permutation");
        }
    }
    std::vector<double> rule = pack_rule(nq, xs, ys, w);
    DevBuf<SingItem> di;
    DevBuf<double> dr;
    DevBuf<double2> dout;
    cudaStream_t s = mesh->stream;
    GC_CUDA(di.upload(items.data(), n, s));
    GC_CUDA(dr.upload(rule.data(), rule.size(), s));
    GC_CUDA(dout.alloc(n));
    bool same = true;
    for (int64_t i = 0; i < n && same; ++i)
        same = items[i].tri_x == items[i].tri_y && items[i].px[0] == items[i].py[0] &&
               items[i].px[1] == items[i].py[1] && items[i].px[2] == items[i].py[2];
    GC_CUDA(launch_generic(kind_of(equation, layer), same, mesh->V.p, mesh->T.p, mesh->charts.p,
                           di.p, n, dr.p, nq, dout.p, nullptr, kappa, s));
    GC_CUDA(cudaMemcpyAsync(out, dout.p, sizeof(double2) * n, cudaMemcpyDeviceToHost, s));
    GC_CUDA(cudaStreamSynchronize(s));
    return GCABEM_OK;
}

int gcabem_layout_create(gcabem_mesh_t mesh, int64_t payload_len, int64_t nblocks,
                         const int64_t *blocks, int64_t npanels, const int64_t *panels,
                         int64_t nitems, const int64_t *items, const uint8_t *perms,
                         gcabem_layout_t *out) {
    GC_ARG(mesh && out, "null argument");
    *out = nullptr;
    GC_ARG(payload_len >= 0 && nblocks >= 0 && npanels >= 0 && nitems >= 0, "negative size");
    GC_ARG(nblocks < (int64_t(1) << 31), "too many blocks");
    GC_CUDA(cudaSetDevice(mesh->device));
    Trace tr("layout");
    auto *L = new gcabem_layout_s();
    L->mesh = mesh;
    L->payload_len = payload_len;
    auto fail = [&](const char *msg) {
        delete L;
        return set_error(GCABEM_ERR_ARG, msg);
    };
    // WorkBlocks -> descriptors + fixed-size tasks (DISJOINT_TPB pairs each)
    std::vector<BlockDesc> bd(nblocks);
    L->block_task_at.assign(nblocks + 1, 0);
    L->block_leaf.resize(nblocks);
    L->block_base.resize(nblocks);
    L->block_pairs.resize(nblocks);
    int64_t ntasks = 0;
    for (int64_t b = 0; b < nblocks; ++b) {
        const int64_t *r = blocks + 7 * b;
        const int64_t base = r[0], ld = r[1], nr = r[2], nc = r[3], ra = r[4], ca = r[5];
        if (!(nr >= 0 && nc >= 0 && nr * nc < (int64_t(1) << 31)) ||
            !(ra >= 0 && ra + nr <= npanels && ca >= 0 && ca + nc <= npanels) ||
            !(nr == 0 || nc == 0 || (base >= 0 && base + (nr - 1) * ld + nc <= payload_len)) ||
            (b > 0 && r[6] < blocks[7 * (b - 1) + 6]))
            return fail("block descriptor out of bounds or out of order");
        bd[b] = BlockDesc{base, ra, ca, (int32_t)ld, (int32_t)nr, (int32_t)nc, ROLE_NORMAL, 0, 0, 0};
        L->block_task_at[b] = ntasks;
        L->block_leaf[b] = r[6];
        L->block_base[b] = base;
        L->block_pairs[b] = nr * nc;
        ntasks += (nr * nc + DISJOINT_TPB - 1) / DISJOINT_TPB;
    }
    L->block_task_at[nblocks] = ntasks;
    std::vector<int2> tasks(ntasks);
    for (int64_t b = 0; b < nblocks; ++b) {
        int64_t t = L->block_task_at[b];
        for (int64_t k0 = 0; k0 < L->block_pairs[b]; k0 += DISJOINT_TPB)
            tasks[t++] = make_int2((int)b, (int)k0);
    }
    tr.mark("blocks+tasks");
    std::vector<int32_t> pan(npanels);
    for (int64_t k = 0; k < npanels; ++k) {
        if (panels[k] < 0 || panels[k] >= mesh->nt) return fail("panel index out of range");
        pan[k] = (int32_t)panels[k];
    }
    // singular items: grouped by case 1..3, sorted by payload index inside a
    // case (chunked execution looks chunks up by payload range); the common
    // input (device_items order) already is, which is checked in O(n)
    int64_t counts[4] = {0, 0, 0, 0};
    bool sorted = true;
    for (int64_t k = 0; k < nitems; ++k) {
        const int64_t c = items[4 * k];
        if (c < 1 || c > 3) return fail("singular item case must be vertex/edge/identical");
        counts[c]++;
        if (k > 0) {
            const int64_t pc = items[4 * (k - 1)];
            sorted = sorted && (pc < c || (pc == c && items[4 * (k - 1) + 3] <= items[4 * k + 3]));
        }
    }
    std::vector<int64_t> order(nitems);
    for (int64_t k = 0; k < nitems; ++k) order[k] = k;
    if (!sorted)
        std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
            return items[4 * a] != items[4 * b] ? items[4 * a] < items[4 * b]
                                                : items[4 * a + 3] < items[4 * b + 3];
        });
    std::vector<SingItem> si(nitems);
    L->item_out.resize(nitems);
    for (int64_t q = 0; q < nitems; ++q) {
        const int64_t k = order[q];
        const int64_t c = items[4 * k];
        SingItem &it = si[q];
        std::memset(&it, 0, sizeof it);
        it.out = items[4 * k + 3];
        bool ok = it.out >= 0 && it.out < payload_len && items[4 * k + 1] >= 0 &&
                  items[4 * k + 1] < mesh->nt && items[4 * k + 2] >= 0 &&
                  items[4 * k + 2] < mesh->nt;
        it.tri_x = (int32_t)items[4 * k + 1];
        it.tri_y = (int32_t)items[4 * k + 2];
        for (int j = 0; j < 3; ++j) {
            it.px[j] = perms[6 * k + j];
            it.py[j] = perms[6 * k + 3 + j];
            ok = ok && it.px[j] < 3 && it.py[j] < 3;
        }
        ok = ok && (c != 3 || (it.tri_x == it.tri_y && it.px[0] == it.py[0] &&
                               it.px[1] == it.py[1] && it.px[2] == it.py[2]));
        if (!ok) return fail("bad singular item (index, permutation or chart)");
        L->item_out[q] = it.out;
    }
    tr.mark("items");
    L->ntasks = ntasks;
    L->case_at[0] = 0;
    for (int c = 1; c <= 3; ++c) L->case_at[c] = L->case_at[c - 1] + counts[c];
    cudaStream_t s = mesh->stream;
    cudaError_t e = pool_init(mesh->device);
    if (e == cudaSuccess) e = L->blocks.upload(bd.data(), bd.size(), s);
    if (e == cudaSuccess) e = L->tasks.upload(tasks.data(), tasks.size(), s);
    if (e == cudaSuccess) e = build_task_descs(L, s);
    if (e == cudaSuccess) e = L->panels.upload(pan.data(), pan.size(), s);
    if (e == cudaSuccess) e = L->items.upload(si.data(), si.size(), s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // host vectors die here
    tr.mark("upload");
    if (e != cudaSuccess) {
        delete L;
        GC_CUDA(e);
    }
    *out = L;
    return GCABEM_OK;
}

}  // extern "C"

namespace {

// this process's share of the host CPUs: its affinity set divided among the
// ranks of a node (torchrun LOCAL_WORLD_SIZE), as packaging.host_threads
unsigned host_cpus() {
    static const unsigned n = [] {
        cpu_set_t set;
        unsigned c = std::max(1u, std::thread::hardware_concurrency());
        if (sched_getaffinity(0, sizeof(set), &set) == 0) c = (unsigned)CPU_COUNT(&set);
        const char *lw = std::getenv("LOCAL_WORLD_SIZE");
        const int ranks = lw ? std::max(1, std::atoi(lw)) : 1;
        return std::max(1u, c / (unsigned)ranks);
    }();
    return n;
}

// split [0, n) over up to `max_threads` std::threads (inline below `grain`)
template <typename F>
void par_for(int64_t n, int64_t grain, F fn, unsigned max_threads = 8) {
    const int maxt = (int)std::min<unsigned>(max_threads, host_cpus());
    const int nt = (int)std::min<int64_t>(maxt, std::max<int64_t>(1, n / std::max<int64_t>(grain, 1)));
    if (nt <= 1) {
        fn(0, n, 0);
        return;
    }
    std::vector<std::thread> th;
    const int64_t chunk = (n + nt - 1) / nt;
    for (int t = 1; t < nt; ++t) {
        const int64_t lo = t * chunk, hi = std::min(n, lo + chunk);
        if (lo < hi) th.emplace_back(fn, lo, hi, t);
    }
    fn(0, std::min(n, chunk), 0);
    for (auto &x : th) x.join();
}

// pinned host blocks reused across plans (cudaHostAlloc costs milliseconds):
// a free list by size
std::mutex g_pin_mutex;
std::multimap<size_t, void *> g_pin_free;

void *pinned_acquire(size_t bytes, size_t *got) {
    {
        std::lock_guard<std::mutex> lk(g_pin_mutex);
        auto it = g_pin_free.lower_bound(bytes);
        if (it != g_pin_free.end() && it->first <= 4 * bytes + (1 << 20)) {
            void *ptr = it->second;
            *got = it->first;
            g_pin_free.erase(it);
            return ptr;
        }
    }
    size_t n = 1 << 16;
    while (n < bytes) n <<= 1;
    void *ptr = nullptr;
    if (cudaHostAlloc(&ptr, n, cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    *got = n;
    return ptr;
}

void pinned_release(void *ptr, size_t bytes) {
    if (!ptr) return;
    std::lock_guard<std::mutex> lk(g_pin_mutex);
    g_pin_free.emplace(bytes, ptr);
}

// TaskDesc records of a task list (block descriptor copied next to the task)
__global__ void task_desc_kernel(const BlockDesc *__restrict__ blocks,
                                 const int2 *__restrict__ tasks, int64_t n,
                                 TaskDesc *__restrict__ out) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int2 tk = tasks[t];
    TaskDesc d;
    d.b = blocks[tk.x];
    d.k0 = tk.y;
    d.pad = 0;
    out[t] = d;
}

// the layout's three TaskDesc lists from its blocks and int2 task lists
cudaError_t build_task_descs(gcabem_layout_s *L, cudaStream_t s) {
    struct List {
        const int2 *src;
        int64_t n;
        PoolBuf<TaskDesc> *dst;
    } lists[3] = {{L->tasks.p, L->ntasks, &L->tdesc},
                  {L->mtasks.p, L->nmtasks, &L->mtdesc},
                  {L->rtasks.p, L->nrtasks, &L->rtdesc}};
    for (const List &l : lists) {
        if (l.n <= 0 || !l.src) continue;
        cudaError_t e = l.dst->alloc(l.n, s);
        if (e != cudaSuccess) return e;
        task_desc_kernel<<<(unsigned)((l.n + 255) / 256), 256, 0, s>>>(L->blocks.p, l.src, l.n,
                                                                        l.dst->p);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

// task lists of a layout from their per-block prefixes (block b's tasks are
// (b, 0), (b, DISJOINT_TPB), ...): all blocks, mirrored (PRIMARY / SELF)
// blocks, plain (NORMAL) blocks; a block has mirrored or plain tasks or none
__global__ void expand_tasks_kernel(const int32_t *__restrict__ at,
                                    const int32_t *__restrict__ at_m,
                                    const int32_t *__restrict__ at_r, int2 *__restrict__ tasks,
                                    int2 *__restrict__ mtasks, int2 *__restrict__ rtasks) {
    const int b = blockIdx.x;
    for (int t = threadIdx.x; t < at[b + 1] - at[b]; t += blockDim.x)
        tasks[at[b] + t] = make_int2(b, t * DISJOINT_TPB);
    if (mtasks)
        for (int t = threadIdx.x; t < at_m[b + 1] - at_m[b]; t += blockDim.x)
            mtasks[at_m[b] + t] = make_int2(b, t * DISJOINT_TPB);
    if (rtasks)
        for (int t = threadIdx.x; t < at_r[b + 1] - at_r[b]; t += blockDim.x)
            rtasks[at_r[b] + t] = make_int2(b, t * DISJOINT_TPB);
}

__global__ void gather_entries_kernel(const double2 *__restrict__ src,
                                      const int64_t *__restrict__ idx, int64_t n,
                                      double2 *__restrict__ dst) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[idx[i]];
}

// host threads writing the skipped leaves of a symmetric download (memory
// bound: a few threads saturate the copy; more would take cores from the
// packaging threads); GCABEM_FILL_THREADS overrides
unsigned fill_threads() {
    static const unsigned n = [] {
        const char *e = std::getenv("GCABEM_FILL_THREADS");
        return e ? (unsigned)std::max(1, std::atoi(e)) : std::min(8u, host_cpus());
    }();
    return n;
}

// SKIP leaf s of the host-filled list: its entries as the transpose of its
// PRIMARY (already in `host`), written with streaming stores (the rows are
// contiguous; no read-for-ownership of the target lines), then its singular
// entries from the patch
void host_fill_leaf(const gcabem_layout_s *L, int64_t s, double2 *host, const double2 *patch) {
    const int64_t nr = L->hf_nr[s], nc = L->hf_nc[s];
    double *dst = reinterpret_cast<double *>(host + L->hf_lo[s]);
    const double *src = reinterpret_cast<const double *>(host + L->hf_m[s]);  // nc x nr
    constexpr int64_t TB = 16;
    for (int64_t i0 = 0; i0 < nr; i0 += TB)
        for (int64_t j0 = 0; j0 < nc; j0 += TB) {
            const int64_t i1 = std::min(nr, i0 + TB), j1 = std::min(nc, j0 + TB);
            for (int64_t i = i0; i < i1; ++i)
                for (int64_t j = j0; j < j1; ++j)
                    _mm_stream_pd(dst + 2 * (i * nc + j), _mm_loadu_pd(src + 2 * (j * nr + i)));
        }
    _mm_sfence();
    for (int64_t q = L->hf_item_at[s]; q < L->hf_item_at[s + 1]; ++q)
        host[L->patch_out[q]] = patch[q];
}

}  // namespace

extern "C" {

int gcabem_layout_from_packages(gcabem_mesh_t mesh, int64_t leaf_lo, int64_t leaf_hi,
                                int64_t nleaves, const int64_t *leaf_shape,
                                const int64_t *leaf_base, const int64_t *leaf_rows_at,
                                const int64_t *leaf_cols_at, int64_t npanels,
                                const int64_t *panels, int64_t nblocks, const int64_t *blk_leaf,
                                const int64_t *blk_r0, const int64_t *blk_nr,
                                const int64_t *blk_c0, const int64_t *blk_nc, int64_t nitems,
                                const int8_t *item_case, const int64_t *item_tri_x,
                                const int64_t *item_tri_y, const int64_t *item_leaf,
                                const int64_t *item_offset, const uint8_t *perms,
                                const int64_t *leaf_mirror, gcabem_layout_t *out) {
    GC_ARG(mesh && out, "null argument");
    *out = nullptr;
    GC_ARG(0 <= leaf_lo && leaf_lo <= leaf_hi && leaf_hi <= nleaves, "bad leaf range");
    GC_ARG(npanels >= 0 && nblocks >= 0 && nitems >= 0, "negative size");
    GC_CUDA(cudaSetDevice(mesh->device));
    Trace tr("from_pk");
    const int64_t base0 = leaf_base[leaf_lo], plen = leaf_base[leaf_hi] - base0;
    // blocks are in leaf order: the range is one contiguous run
    for (int64_t b = 1; b < nblocks; ++b)
        GC_ARG(blk_leaf[b] >= blk_leaf[b - 1], "block leaves out of order");
    GC_ARG(nblocks == 0 || (blk_leaf[0] >= 0 && blk_leaf[nblocks - 1] < nleaves),
           "block leaf out of range");
    const int64_t b0 = std::lower_bound(blk_leaf, blk_leaf + nblocks, leaf_lo) - blk_leaf;
    const int64_t b1 = std::lower_bound(blk_leaf, blk_leaf + nblocks, leaf_hi) - blk_leaf;
    const int64_t B = b1 - b0;
    auto *L = new gcabem_layout_s();
    L->mesh = mesh;
    L->payload_len = plen;
    L->block_task_at.resize(B + 1);
    L->block_leaf.resize(B);
    L->block_base.resize(B);
    L->block_pairs.resize(B);
    // leaf roles of the mirrored evaluation: a leaf whose mirror (the leaf of
    // the transposed cluster pair) lies in this range is PRIMARY if it comes
    // first in the preorder, SKIP if it comes second (its entries are written
    // by the primary: chunked execution in leaf order sees the primary first),
    // SELF if it is its own mirror; every other leaf is NORMAL
    std::vector<int8_t> leaf_role;
    bool any_mirror = false;
    if (leaf_mirror) {
        leaf_role.assign(leaf_hi - leaf_lo, ROLE_NORMAL);
        for (int64_t lf = leaf_lo; lf < leaf_hi; ++lf) {
            const int64_t m = leaf_mirror[lf];
            if (m < leaf_lo || m >= leaf_hi) continue;
            if (leaf_mirror[m] != lf || leaf_shape[2 * m] != leaf_shape[2 * lf + 1] ||
                leaf_shape[2 * m + 1] != leaf_shape[2 * lf]) {
                delete L;
                return set_error(GCABEM_ERR_ARG, "leaf mirror is not a transposed leaf");
            }
            leaf_role[lf - leaf_lo] = m == lf ? ROLE_SELF : m > lf ? ROLE_PRIMARY : ROLE_SKIP;
            any_mirror = true;
        }
    }
    auto role_of = [&](int64_t lf) -> int {
        return any_mirror ? leaf_role[lf - leaf_lo] : ROLE_NORMAL;
    };
    int64_t ntasks = 0, nmt = 0, nrt = 0;
    if (any_mirror) {
        L->block_mtask_at.resize(B + 1);
        L->block_rtask_at.resize(B + 1);
    }
    {
        // task offsets of the blocks (all / mirrored / plain): exclusive
        // prefix sums, per block chunk on the pool, then the chunk offsets
        constexpr int NP = 16;
        int64_t tot[NP + 1][3] = {};
        auto pass = [&](bool write) {
            par_for(NP, 1, [&](int64_t t0, int64_t t1, int) {
                for (int64_t t = t0; t < t1; ++t) {
                    // first pass: chunk sums from 0 (tot[t] is another
                    // chunk's output then); second pass: from the offsets
                    int64_t a = write ? tot[t][0] : 0, m = write ? tot[t][1] : 0,
                            n = write ? tot[t][2] : 0;
                    for (int64_t b = t * B / NP; b < (t + 1) * B / NP; ++b) {
                        const int64_t np = blk_nr[b0 + b] * blk_nc[b0 + b];
                        const int64_t nt = (np + DISJOINT_TPB - 1) / DISJOINT_TPB;
                        const int r = any_mirror ? role_of(blk_leaf[b0 + b]) : ROLE_NORMAL;
                        if (write) {
                            L->block_task_at[b] = a;
                            L->block_pairs[b] = np;
                            if (any_mirror) {
                                L->block_mtask_at[b] = m;
                                L->block_rtask_at[b] = n;
                            }
                        }
                        a += nt;
                        if (r == ROLE_PRIMARY || r == ROLE_SELF) m += nt;
                        if (r == ROLE_NORMAL) n += nt;
                    }
                    if (!write) {
                        tot[t + 1][0] = a;
                        tot[t + 1][1] = m;
                        tot[t + 1][2] = n;
                    }
                }
            });
        };
        pass(false);  // chunk totals at tot[t + 1]
        for (int t = 0; t < NP; ++t)
            for (int c = 0; c < 3; ++c) tot[t + 1][c] += tot[t][c];
        pass(true);   // offsets from tot[t]
        ntasks = tot[NP][0];
        nmt = any_mirror ? tot[NP][1] : 0;
        nrt = any_mirror ? tot[NP][2] : 0;
    }
    L->block_task_at[B] = ntasks;
    if (any_mirror) {
        L->block_mtask_at[B] = nmt;
        L->block_rtask_at[B] = nrt;
    }
    // singular items of the range: per-chunk case counts (stable counting sort)
    constexpr int MAXT = 8;
    int64_t cnt[MAXT][4] = {};
    std::atomic<bool> bad{false};
    const int64_t ichunk = std::max<int64_t>(1, (nitems + MAXT - 1) / MAXT);
    // fixed item slots [slot * ichunk, (slot + 1) * ichunk): thread-count independent
    const int64_t slot_grain = nitems < (1 << 16) ? MAXT : 1;
    par_for(MAXT, slot_grain, [&](int64_t slo, int64_t shi, int) {
        for (int64_t slot = slo; slot < shi; ++slot) {
            const int64_t c0 = slot * ichunk, c1 = std::min(nitems, c0 + ichunk);
            for (int64_t k = c0; k < c1; ++k) {
                const int c = item_case[k];
                const int64_t lf = item_leaf[k];
                if (c < 1 || c > 3 || lf < 0 || lf >= nleaves) {
                    bad = true;
                    continue;
                }
                if (lf >= leaf_lo && lf < leaf_hi) cnt[slot][c]++;
            }
        }
    });
    if (bad) {
        delete L;
        return set_error(GCABEM_ERR_ARG, "bad singular item");
    }
    int64_t chunk_at[MAXT][4] = {};
    L->case_at[0] = 0;
    {
        int64_t run = 0;
        for (int c = 1; c <= 3; ++c) {
            for (int s = 0; s < MAXT; ++s) {
                chunk_at[s][c] = run;
                run += cnt[s][c];
            }
            L->case_at[c] = run;
        }
    }
    const int64_t S = L->case_at[3];
    L->item_out.resize(S);
    tr.mark("counts");
    // one pinned arena: [BlockDesc B | int32 task prefixes 3 (B + 1) | int32 npanels |
    // SingItem S]; the task lists themselves are expanded on the device
    // (expand_tasks_kernel: 32-pair tasks would be 4x the bytes to write and upload)
    auto align = [](size_t x) { return (x + 255) & ~size_t(255); };
    const size_t off_t = align(sizeof(BlockDesc) * B),
                 off_p = off_t + 3 * align(sizeof(int32_t) * (B + 1)),
                 off_s = off_p + align(sizeof(int32_t) * npanels),
                 total = off_s + align(sizeof(SingItem) * S);
    // from the pinned pool (no lock held while filling: layouts of several
    // leaf ranges may be built concurrently); returned after the stream sync
    struct PinnedBlock {
        void *p = nullptr;
        size_t n = 0;
        ~PinnedBlock() { pinned_release(p, n); }
    } arena_blk;
    arena_blk.p = pinned_acquire(total, &arena_blk.n);
    if (!arena_blk.p) {
        delete L;
        return set_error(GCABEM_ERR_CUDA, "pinned staging allocation failed");
    }
    char *arena = static_cast<char *>(arena_blk.p);
    BlockDesc *bd = reinterpret_cast<BlockDesc *>(arena);
    int32_t *at3 = reinterpret_cast<int32_t *>(arena + off_t);  // all / mirrored / plain
    const size_t at_stride = align(sizeof(int32_t) * (B + 1)) / sizeof(int32_t);
    if (ntasks >= (int64_t(1) << 31)) {
        delete L;
        return set_error(GCABEM_ERR_ARG, "too many disjoint tasks for one layout");
    }
    int32_t *pan = reinterpret_cast<int32_t *>(arena + off_p);
    SingItem *si = reinterpret_cast<SingItem *>(arena + off_s);
    par_for(B, 1 << 14, [&](int64_t lo, int64_t hi, int) {
        for (int64_t b = lo; b < hi; ++b) {
            const int64_t g = b0 + b, lf = blk_leaf[g];
            const int64_t ld = leaf_shape[2 * lf + 1], nr = blk_nr[g], nc = blk_nc[g];
            const int64_t base = leaf_base[lf] - base0 + blk_r0[g] * ld + blk_c0[g];
            const int64_t ra = leaf_rows_at[lf] + blk_r0[g], ca = leaf_cols_at[lf] + blk_c0[g];
            if (!(nr >= 0 && nc >= 0 && nr * nc < (int64_t(1) << 31)) ||
                !(ra >= 0 && ra + nr <= npanels && ca >= 0 && ca + nc <= npanels) ||
                !(nr == 0 || nc == 0 || (base >= 0 && base + (nr - 1) * ld + nc <= plen)))
                bad = true;
            const int role = role_of(lf);
            int64_t mbase = 0, mld = 0, dr = 0;
            if (role == ROLE_PRIMARY || role == ROLE_SELF) {
                // entry (i, j) of this block is leaf entry (r0 + i, c0 + j); the
                // transposed pair is entry (c0 + j, r0 + i) of the mirror leaf
                const int64_t m = leaf_mirror[lf];
                mld = leaf_shape[2 * m + 1];
                mbase = leaf_base[m] - base0 + blk_c0[g] * mld + blk_r0[g];
                dr = blk_r0[g] - blk_c0[g];
                if (!(nr == 0 || nc == 0 || (mbase >= 0 && mbase + (nc - 1) * mld + nr <= plen)))
                    bad = true;
            }
            bd[b] = BlockDesc{base, ra, ca, (int32_t)ld, (int32_t)nr, (int32_t)nc, role, mbase,
                              (int32_t)mld, (int32_t)dr};
            L->block_leaf[b] = lf;
            L->block_base[b] = base;
            at3[b] = (int32_t)L->block_task_at[b];
            at3[at_stride + b] = any_mirror ? (int32_t)L->block_mtask_at[b] : 0;
            at3[2 * at_stride + b] = any_mirror ? (int32_t)L->block_rtask_at[b] : 0;
        }
    });
    at3[B] = (int32_t)ntasks;
    at3[at_stride + B] = (int32_t)nmt;
    at3[2 * at_stride + B] = (int32_t)nrt;
    par_for(npanels, 1 << 16, [&](int64_t lo, int64_t hi, int) {
        for (int64_t k = lo; k < hi; ++k) {
            if (panels[k] < 0 || panels[k] >= mesh->nt) bad = true;
            pan[k] = (int32_t)panels[k];
        }
    });
    par_for(MAXT, slot_grain, [&](int64_t slo, int64_t shi, int) {
        for (int64_t slot = slo; slot < shi; ++slot) {
            const int64_t c0 = slot * ichunk, c1 = std::min(nitems, c0 + ichunk);
            int64_t at[4] = {0, chunk_at[slot][1], chunk_at[slot][2], chunk_at[slot][3]};
            for (int64_t k = c0; k < c1; ++k) {
                const int64_t lf = item_leaf[k];
                if (lf < leaf_lo || lf >= leaf_hi) continue;
                const int c = item_case[k];
                SingItem &it = si[at[c]];
                it.out = leaf_base[lf] - base0 + item_offset[k];
                it.tri_x = (int32_t)item_tri_x[k];
                it.tri_y = (int32_t)item_tri_y[k];
                const uint8_t *pm = perms + 6 * k;
                it.px[0] = pm[0]; it.px[1] = pm[1]; it.px[2] = pm[2];
                it.py[0] = pm[3]; it.py[1] = pm[4]; it.py[2] = pm[5];
                it.pad[0] = it.pad[1] = 0;
                bool ok = it.out >= 0 && it.out < plen && item_tri_x[k] >= 0 &&
                          item_tri_x[k] < mesh->nt && item_tri_y[k] >= 0 &&
                          item_tri_y[k] < mesh->nt && pm[0] < 3 && pm[1] < 3 && pm[2] < 3 &&
                          pm[3] < 3 && pm[4] < 3 && pm[5] < 3;
                ok = ok && (c != 3 || (it.tri_x == it.tri_y && pm[0] == pm[3] &&
                                       pm[1] == pm[4] && pm[2] == pm[5]));
                if (!ok) bad = true;
                L->item_out[at[c]] = it.out;
                ++at[c];
            }
        }
    });
    if (bad) {
        delete L;
        return set_error(GCABEM_ERR_ARG, "bad block, panel or singular item");
    }
    // chunked execution looks items up by payload index inside a case: sort a
    // case only if its generation order is not already ascending (it is,
    // unless a flagged leaf was split by columns)
    for (int c = 0; c < 3; ++c) {
        const int64_t a0 = L->case_at[c], a1 = L->case_at[c + 1];
        if (std::is_sorted(L->item_out.begin() + a0, L->item_out.begin() + a1)) continue;
        std::stable_sort(si + a0, si + a1,
                         [](const SingItem &x, const SingItem &y) { return x.out < y.out; });
        for (int64_t q = a0; q < a1; ++q) L->item_out[q] = si[q].out;
    }
    tr.mark("fill");
    L->ntasks = ntasks;
    L->nmtasks = nmt;
    L->nrtasks = nrt;
    std::vector<SingItem> vm, vp;
    std::vector<int64_t> vm_mout;
    if (any_mirror) {
        // vertex items (case slot 0, sorted by payload index) -> mirrored /
        // plain / written-by-partner, from their leaf's role; in item chunks
        // on the pool (each chunk finds its first leaf by bisection, then
        // walks the leaves alongside), concatenated in chunk order
        const int64_t q0 = L->case_at[0], nv = L->case_at[1] - L->case_at[0];
        constexpr int VCH = 8;
        struct Part {
            std::vector<SingItem> vm, vp;
            std::vector<int64_t> mout;
            int64_t dropped = 0;
        } parts[VCH];
        par_for(VCH, nv < (1 << 15) ? VCH : 1, [&](int64_t c0, int64_t c1, int) {
            for (int64_t ch = c0; ch < c1; ++ch) {
                const int64_t a0 = q0 + ch * nv / VCH, a1 = q0 + (ch + 1) * nv / VCH;
                Part &P = parts[ch];
                if (a1 <= a0) continue;
                int64_t lf = std::upper_bound(leaf_base + leaf_lo, leaf_base + leaf_hi + 1,
                                              si[a0].out + base0) - leaf_base - 1;
                for (int64_t q = a0; q < a1; ++q) {
                    const SingItem &it = si[q];
                    const int64_t g = it.out + base0;
                    while (lf + 1 < leaf_hi && leaf_base[lf + 1] <= g) ++lf;
                    const int r = role_of(lf);
                    const int64_t ncol = leaf_shape[2 * lf + 1], off = g - leaf_base[lf];
                    const int64_t i = off / ncol, j = off % ncol;
                    if (r == ROLE_PRIMARY || (r == ROLE_SELF && i < j)) {
                        const int64_t m = leaf_mirror[lf];
                        P.vm.push_back(it);
                        P.mout.push_back(leaf_base[m] - base0 + j * leaf_shape[2 * m + 1] + i);
                    } else if (r == ROLE_NORMAL) {
                        P.vp.push_back(it);
                    } else {
                        ++P.dropped;
                    }
                }
            }
        });
        int64_t dropped = 0;
        for (const Part &P : parts) {
            dropped += P.dropped;
            vm.insert(vm.end(), P.vm.begin(), P.vm.end());
            vm_mout.insert(vm_mout.end(), P.mout.begin(), P.mout.end());
            vp.insert(vp.end(), P.vp.begin(), P.vp.end());
        }
        L->vertex_mirror = dropped == (int64_t)vm.size();
        if (L->vertex_mirror) {
            L->vm_out.resize(vm.size());
            L->vp_out.resize(vp.size());
            for (size_t k = 0; k < vm.size(); ++k) L->vm_out[k] = vm[k].out;
            for (size_t k = 0; k < vp.size(); ++k) L->vp_out[k] = vp[k].out;
        }
        tr.mark("mirror-split");
    }
    if (any_mirror) {
        // evaluation counts for the roofline: pairs of PRIMARY/SELF(upper)
        // blocks minus their vertex-sharing pairs (one mirrored evaluation
        // each), NORMAL pairs minus theirs
        // per-thread partial sums (integers: the order does not matter)
        constexpr int NP = 16;
        int64_t part[NP][6] = {};
        par_for(NP, 1, [&](int64_t t0, int64_t t1, int) {
            for (int64_t t = t0; t < t1; ++t) {
                int64_t *q = part[t];  // mp, sp, np, up, sh_m, sh_n
                for (int64_t b = t * B / NP; b < (t + 1) * B / NP; ++b) {
                    const int64_t g = b0 + b, lf = blk_leaf[g], nr = blk_nr[g], nc = blk_nc[g];
                    const int r = role_of(lf);
                    if (r == ROLE_PRIMARY) q[0] += nr * nc;
                    else if (r == ROLE_SKIP) q[1] += nr * nc;
                    else if (r == ROLE_NORMAL) q[2] += nr * nc;
                    else {  // SELF: leaf entries (r0 + i, c0 + j) with r0 + i < c0 + j
                        const int64_t dr = blk_r0[g] - blk_c0[g];
                        for (int64_t i = 0; i < nr; ++i)
                            q[3] += std::max<int64_t>(0, nc - std::max<int64_t>(0, i + dr + 1));
                    }
                }
                for (int64_t k = t * nitems / NP; k < (t + 1) * nitems / NP; ++k) {
                    const int64_t lf = item_leaf[k];
                    if (lf < leaf_lo || lf >= leaf_hi) continue;
                    const int r = role_of(lf);
                    if (r == ROLE_PRIMARY) ++q[4];
                    else if (r == ROLE_NORMAL) ++q[5];
                    else if (r == ROLE_SELF) {
                        const int64_t ncol = leaf_shape[2 * lf + 1];
                        const int64_t i = item_offset[k] / ncol, j = item_offset[k] % ncol;
                        if (i < j) ++q[4];
                    }
                }
            }
        });
        int64_t mp = 0, sp = 0, np_ = 0, up = 0, sh_m = 0, sh_n = 0;
        for (const auto &q : part) {
            mp += q[0];
            sp += q[1];
            np_ += q[2];
            up += q[3];
            sh_m += q[4];
            sh_n += q[5];
        }
        L->mirror_info[0] = mp + up - sh_m;
        L->mirror_info[1] = np_ - sh_n;
        L->mirror_info[2] = mp + up;
        L->mirror_info[3] = sp;
        tr.mark("eval-counts");
    }
    if (any_mirror) {
        // host-filled SKIP leaves (symmetric download): runs of consecutive
        // SKIP leaves of at least SYM_MIN_RUN entries (a shorter gap costs
        // less to copy than one more D2H call; GCABEM_SYM_MIN_RUN overrides)
        const char *env_run = std::getenv("GCABEM_SYM_MIN_RUN");
        const int64_t min_run = env_run ? std::max<long long>(1, std::atoll(env_run)) : SYM_MIN_RUN;
        for (int64_t lf = leaf_lo; lf < leaf_hi;) {
            if (role_of(lf) != ROLE_SKIP) {
                ++lf;
                continue;
            }
            int64_t e = lf;
            while (e < leaf_hi && role_of(e) == ROLE_SKIP) ++e;
            if (leaf_base[e] - leaf_base[lf] >= min_run)
                for (int64_t q = lf; q < e; ++q) {
                    L->hf_lo.push_back(leaf_base[q] - base0);
                    L->hf_m.push_back(leaf_base[leaf_mirror[q]] - base0);
                    L->hf_nr.push_back((int32_t)leaf_shape[2 * q]);
                    L->hf_nc.push_back((int32_t)leaf_shape[2 * q + 1]);
                }
            lf = e;
        }
        // their singular entries: per case the item payload indices ascend,
        // so a sweep against the (ascending) leaves finds them; in leaf
        // chunks on the pool (each chunk bisects to its first item), one
        // pass counting, one filling
        const int64_t H = (int64_t)L->hf_lo.size();
        L->hf_item_at.assign(H + 1, 0);
        std::vector<int64_t> hf_hi(H);
        for (int64_t h = 0; h < H; ++h) hf_hi[h] = L->hf_lo[h] + (int64_t)L->hf_nr[h] * L->hf_nc[h];
        constexpr int64_t NCH = 64;
        auto sweep = [&](int64_t ch, auto &&visit) {
            const int64_t h0 = ch * H / NCH, h1 = (ch + 1) * H / NCH;
            if (h0 >= h1) return;
            for (int c = 0; c < 3; ++c) {
                const int64_t *b = L->item_out.data() + L->case_at[c];
                const int64_t *e = L->item_out.data() + L->case_at[c + 1];
                int64_t h = h0;
                for (const int64_t *it = std::lower_bound(b, e, L->hf_lo[h0]);
                     it != e && *it < hf_hi[h1 - 1]; ++it) {
                    while (hf_hi[h] <= *it) ++h;
                    if (*it >= L->hf_lo[h]) visit(h, *it);
                }
            }
        };
        if (H) {
            par_for(NCH, 1, [&](int64_t c0, int64_t c1, int) {
                for (int64_t ch = c0; ch < c1; ++ch)
                    sweep(ch, [&](int64_t h, int64_t) { ++L->hf_item_at[h + 1]; });
            });
            for (int64_t h = 0; h < H; ++h) L->hf_item_at[h + 1] += L->hf_item_at[h];
            L->patch_out.resize(L->hf_item_at[H]);
            std::vector<int64_t> cur(L->hf_item_at.begin(), L->hf_item_at.end() - 1);
            par_for(NCH, 1, [&](int64_t c0, int64_t c1, int) {
                for (int64_t ch = c0; ch < c1; ++ch)
                    sweep(ch, [&](int64_t h, int64_t off) { L->patch_out[cur[h]++] = off; });
            });
        }
        tr.mark("sym-leaves");
    }
    cudaStream_t s = mesh->stream;
    cudaError_t e = pool_init(mesh->device);
    if (e == cudaSuccess) e = L->blocks.alloc(B, s);
    if (e == cudaSuccess) e = L->tasks.alloc(ntasks, s);
    if (e == cudaSuccess && nmt) e = L->mtasks.alloc(nmt, s);
    if (e == cudaSuccess && nrt) e = L->rtasks.alloc(nrt, s);
    if (e == cudaSuccess) e = L->panels.alloc(npanels, s);
    if (e == cudaSuccess) e = L->items.alloc(S, s);
    if (e == cudaSuccess && B) e = cudaMemcpyAsync(L->blocks.p, bd, sizeof(BlockDesc) * B, cudaMemcpyHostToDevice, s);
    PoolBuf<int32_t> d_at;   // the three task prefixes, for the expansion below
    if (e == cudaSuccess && B) e = d_at.alloc(3 * at_stride, s);
    if (e == cudaSuccess && B)
        e = cudaMemcpyAsync(d_at.p, at3, sizeof(int32_t) * 3 * at_stride, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && B && ntasks) {
        expand_tasks_kernel<<<(unsigned)B, 32, 0, s>>>(d_at.p, d_at.p + at_stride,
                                                       d_at.p + 2 * at_stride, L->tasks.p,
                                                       L->mtasks.p, L->rtasks.p);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess && npanels) e = cudaMemcpyAsync(L->panels.p, pan, sizeof(int32_t) * npanels, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && S) e = cudaMemcpyAsync(L->items.p, si, sizeof(SingItem) * S, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && L->vertex_mirror) {
        e = L->vm_items.upload(vm.data(), vm.size(), s);
        if (e == cudaSuccess) e = L->vm_mout.upload(vm_mout.data(), vm_mout.size(), s);
        if (e == cudaSuccess) e = L->vp_items.upload(vp.data(), vp.size(), s);
    }
    if (e == cudaSuccess && !L->patch_out.empty())
        e = L->patch_dev.upload(L->patch_out.data(), L->patch_out.size(), s);
    if (e == cudaSuccess) e = build_task_descs(L, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // the arena is reused after this
    tr.mark("upload");
    if (e != cudaSuccess) {
        delete L;
        GC_CUDA(e);
    }
    *out = L;
    return GCABEM_OK;
}

int gcabem_layout_info(gcabem_layout_t L, int64_t *info8) {
    GC_ARG(L && info8, "null argument");
    int64_t pairs = 0;
    for (int64_t v : L->block_pairs) pairs += v;
    info8[0] = L->payload_len;
    info8[1] = (int64_t)L->block_pairs.size();
    info8[2] = L->ntasks;
    info8[3] = pairs;
    for (int c = 0; c < 3; ++c) info8[4 + c] = L->case_at[c + 1] - L->case_at[c];
    info8[7] = (int64_t)(L->blocks.n * sizeof(BlockDesc) +
                         (L->tasks.n + L->mtasks.n + L->rtasks.n) * sizeof(int2) +
                         L->panels.n * sizeof(int32_t) + L->items.n * sizeof(SingItem));
    return GCABEM_OK;
}

int gcabem_layout_mirror_info(gcabem_layout_t L, int64_t *info6) {
    GC_ARG(L && info6, "null argument");
    for (int k = 0; k < 4; ++k) info6[k] = L->mirror_info[k];
    info6[4] = L->nmtasks;
    info6[5] = L->nrtasks;
    return GCABEM_OK;
}

int gcabem_layout_release(gcabem_layout_t L) {
    if (!L) return GCABEM_OK;
    if (--L->refs > 0) return GCABEM_OK;
    cudaSetDevice(L->mesh->device);
    cudaStreamSynchronize(L->mesh->stream);
    delete L;  // DevBuf destructors free the device buffers
    return GCABEM_OK;
}

}  // extern "C"

namespace {
// Group the points of a staged singular rule (rows {xs, xt, ys, yt, w}) by
// the point of one side, term by term (`nterms` terms of equal size, in rule
// order): per term the side with fewer distinct points is held fixed (a
// vertex term has 25 distinct x points for 625 points, an edge term as few
// as 25 on one side and 385 on the other). Groups in first-appearance order,
// packed into chunks of at most RULE_CHUNK rows and groups (a group larger
// than a chunk is split). Group record {a, b, first row, rows, side}: side 0
// = x point (a, b) fixed, rows {ys, yt, w}; side 1 = y point fixed, rows
// {xs, xt, w}.
void group_rule(const double *r5, int64_t q, int nterms, std::vector<double> &rows,
                std::vector<double> &groups, std::vector<int4> &chunks) {
    rows.clear();
    groups.clear();
    chunks.clear();
    if (nterms < 1 || q % nterms) nterms = 1;
    const int64_t tq = q / nterms;
    int r0 = 0, g0 = 0, nr = 0, ng = 0;
    for (int term = 0; term < nterms; ++term) {
        const int64_t k0 = term * tq, k1 = k0 + tq;
        std::vector<std::pair<std::pair<double, double>, std::vector<int64_t>>> order[2];
        for (int side = 0; side < 2; ++side) {
            std::map<std::pair<uint64_t, uint64_t>, size_t> at;
            for (int64_t k = k0; k < k1; ++k) {
                uint64_t a, b;
                std::memcpy(&a, r5 + 5 * k + 2 * side, 8);
                std::memcpy(&b, r5 + 5 * k + 2 * side + 1, 8);
                auto it = at.find({a, b});
                if (it == at.end()) {
                    at.emplace(std::make_pair(a, b), order[side].size());
                    order[side].push_back({{r5[5 * k + 2 * side], r5[5 * k + 2 * side + 1]}, {k}});
                } else {
                    order[side][it->second].second.push_back(k);
                }
            }
        }
        const int side = order[1].size() < order[0].size() ? 1 : 0;
        const int other = 2 - 2 * side;   // column of the varying point
        for (auto &grp : order[side]) {
            const auto &idx = grp.second;
            for (size_t p0 = 0; p0 < idx.size(); p0 += RULE_CHUNK) {
                const int piece = (int)std::min<size_t>(RULE_CHUNK, idx.size() - p0);
                if (nr + piece > RULE_CHUNK || ng + 1 > RULE_CHUNK) {
                    chunks.push_back(make_int4(r0, r0 + nr, g0, g0 + ng));
                    r0 += nr;
                    g0 += ng;
                    nr = ng = 0;
                }
                groups.insert(groups.end(), {grp.first.first, grp.first.second,
                                             (double)(r0 + nr), (double)piece, (double)side});
                for (int j = 0; j < piece; ++j) {
                    const double *r = r5 + 5 * idx[p0 + j];
                    rows.insert(rows.end(), {r[other], r[other + 1], r[4]});
                }
                nr += piece;
                ++ng;
            }
        }
    }
    if (nr > 0) chunks.push_back(make_int4(r0, r0 + nr, g0, g0 + ng));
}

int plan_create_kind(gcabem_layout_t L, int kind, double kappa, int disjoint_n,
                     const double *gauss_pts, const double *gauss_wts, const int64_t *sq,
                     const double *const *srule, gcabem_plan_t *out);
}  // namespace

extern "C" {

int gcabem_plan_create_on(gcabem_layout_t L, int equation, int layer, double kappa,
                          int disjoint_n, const double *gauss_pts, const double *gauss_wts,
                          const int64_t *sq, const double *const *srule, gcabem_plan_t *out) {
    GC_ARG(L && out, "null argument");
    *out = nullptr;
    if (int rc = check_kind(equation, layer, kappa)) return rc;
    return plan_create_kind(L, kind_of(equation, layer), kappa, disjoint_n, gauss_pts, gauss_wts,
                            sq, srule, out);
}

int gcabem_plan_create_pair(gcabem_layout_t L, int equation, double kappa, int disjoint_n,
                            const double *gauss_pts, const double *gauss_wts, const int64_t *sq,
                            const double *const *srule, gcabem_plan_t *out) {
    GC_ARG(L && out, "null argument");
    *out = nullptr;
    if (int rc = check_kind(equation, 1, kappa)) return rc;
    return plan_create_kind(L, equation == 0 ? L_PAIR : H_PAIR, kappa, disjoint_n, gauss_pts,
                            gauss_wts, sq, srule, out);
}

}  // extern "C"

namespace {
int plan_create_kind(gcabem_layout_t L, int kind, double kappa, int disjoint_n,
                     const double *gauss_pts, const double *gauss_wts, const int64_t *sq,
                     const double *const *srule, gcabem_plan_t *out) {
    GC_ARG(disjoint_n >= 1 && disjoint_n <= MAX_ORDER, "disjoint order outside [1, 12]");
    gcabem_mesh_t mesh = L->mesh;
    GC_CUDA(cudaSetDevice(mesh->device));
    if (int rc = ensure_disjoint_rule(mesh->device, disjoint_n, gauss_pts, gauss_wts)) return rc;
    for (int c = 0; c < 3; ++c)
        GC_ARG(L->case_at[c + 1] == L->case_at[c] || (sq && sq[c] > 0),
               "singular items without a rule");
    auto *p = new gcabem_plan_s();
    p->mesh = mesh;
    p->L = L;
    ++L->refs;
    p->kind = kind;
    p->order = disjoint_n;
    p->kappa = kappa;
    p->mirrored = L->nmtasks > 0 && disjoint_n <= MAX_MIRROR_ORDER;
    p->payload_len = L->payload_len;
    cudaError_t e = cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->copy, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = pool_init(mesh->device);
    Trace tr("plan_create");
    if (e == cudaSuccess) e = p->payload.alloc(p->payload_len, p->stream);
    if (e == cudaSuccess && kind_pair(kind)) e = p->payload2.alloc(p->payload_len, p->stream);
    tr.mark("alloc");
    for (int c = 0; c < 3 && e == cudaSuccess; ++c) {
        p->sq[c] = sq ? sq[c] : 0;
        if (p->sq[c] > 0 && L->case_at[c + 1] > L->case_at[c])
            e = p->srule[c].upload(srule[c], 5 * p->sq[c], p->stream);
        // vertex and edge items: the x-grouped rule (the identical case keeps
        // its exact-difference form); GCABEM_NO_GROUPED=1 turns it off
        static const bool no_grouped = std::getenv("GCABEM_NO_GROUPED") != nullptr;
        static const bool no_grouped_edge = std::getenv("GCABEM_NO_GROUPED_EDGE") != nullptr;
        if (e == cudaSuccess && c < 2 && !no_grouped && !(c == 1 && no_grouped_edge) &&
            p->sq[c] > 0 &&
            L->case_at[c + 1] > L->case_at[c]) {
            std::vector<double> rows, groups;
            std::vector<int4> chunks;
            group_rule(srule[c], p->sq[c], c == 0 ? 2 : 5, rows, groups, chunks);
            e = p->grows[c].upload(rows.data(), rows.size(), p->stream);
            if (e == cudaSuccess) e = p->ggroups[c].upload(groups.data(), groups.size(), p->stream);
            if (e == cudaSuccess) e = p->gchunks[c].upload(chunks.data(), chunks.size(), p->stream);
            p->gn[c] = (int)chunks.size();
        }
        // identical items: the 6 terms of the rule are 3 base terms each
        // followed by its x <-> y swap with the same weights (quadrature.py:
        // 132-143); verified point by point, the base half is kept
        static const bool no_half = std::getenv("GCABEM_NO_SYM_HALF") != nullptr;
        if (e == cudaSuccess && c == 2 && !no_half && p->sq[2] > 0 && p->sq[2] % 6 == 0 &&
            L->case_at[3] > L->case_at[2]) {
            const double *r = srule[2];
            const int64_t n4 = p->sq[2] / 6;
            bool ok = true;
            for (int m = 0; m < 3 && ok; ++m)
                for (int64_t k = 2 * m * n4; k < (2 * m + 1) * n4 && ok; ++k) {
                    const double *a = r + 5 * k, *b = r + 5 * (k + n4);
                    ok = a[0] == b[2] && a[1] == b[3] && a[2] == b[0] && a[3] == b[1] &&
                         a[4] == b[4];
                }
            if (ok) {
                std::vector<double> half;
                half.reserve(15 * n4);
                for (int m = 0; m < 3; ++m)
                    half.insert(half.end(), r + 5 * (2 * m * n4), r + 5 * ((2 * m + 1) * n4));
                e = p->hrule.upload(half.data(), half.size(), p->stream);
                p->hq = 3 * n4;
            }
        }
    }
    for (int k = 0; k < 3 && e == cudaSuccess; ++k) e = cudaEventCreate(&p->ev[k]);
    if (e == cudaSuccess) e = cudaStreamSynchronize(p->stream);
    tr.mark("rules+sync");
    if (e != cudaSuccess) {
        gcabem_plan_destroy(p);
        GC_CUDA(e);
    }
    *out = p;
    return GCABEM_OK;
}
}  // namespace

extern "C" {

int gcabem_plan_create(gcabem_mesh_t mesh, int equation, int layer, double kappa, int disjoint_n,
                       const double *gauss_pts, const double *gauss_wts, int64_t payload_len,
                       int64_t nblocks, const int64_t *blocks, int64_t npanels,
                       const int64_t *panels, int64_t nitems, const int64_t *items,
                       const uint8_t *perms, const int64_t *sq, const double *const *srule,
                       gcabem_plan_t *out) {
    GC_ARG(out, "null argument");
    if (int rc = check_kind(equation, layer, kappa)) return rc;
    gcabem_layout_t L = nullptr;
    if (int rc = gcabem_layout_create(mesh, payload_len, nblocks, blocks, npanels, panels,
                                      nitems, items, perms, &L))
        return rc;
    const int rc = gcabem_plan_create_on(L, equation, layer, kappa, disjoint_n, gauss_pts,
                                         gauss_wts, sq, srule, out);
    gcabem_layout_release(L);  // the plan holds its own reference
    return rc;
}

namespace {

// Launch the kernels of blocks [b0, b1) and of the singular items whose
// payload index lies in [p0, p1) on the plan stream.
GroupedRule grouped_of(gcabem_plan_t p, int c) {
    GroupedRule g;
    if (c == 2 && p->hq > 0) g.sym_half = 1;
    if (p->gn[c] > 0) {
        g.rows = p->grows[c].p;
        g.groups = p->ggroups[c].p;
        g.chunks = p->gchunks[c].p;
        g.nchunks = p->gn[c];
    }
    return g;
}

// vertex items on the mirrored path: a mirrored plan whose layout split the
// vertex items and whose vertex rule is x-grouped
bool vertex_mirrored(gcabem_plan_t p) {
    return p->mirrored && p->L->vertex_mirror && p->gn[0] > 0;
}

// Disjoint kernels of blocks [b0, b1): the plain kernel over every task, or
// (mirrored plan) the plain kernel over the NORMAL blocks' tasks and the
// mirrored kernel over the PRIMARY/SELF blocks' tasks (SKIP blocks: none).
int enqueue_disjoint(gcabem_plan_t p, int64_t b0, int64_t b1) {
    gcabem_mesh_t m = p->mesh;
    gcabem_layout_t L = p->L;
    cudaStream_t s = p->stream;
    if (!p->mirrored) {
        const int64_t t0 = L->block_task_at[b0], t1 = L->block_task_at[b1];
        GC_CUDA(launch_disjoint(p->kind, p->order, m->charts.p, m->T.p, L->tdesc.p + t0, t1 - t0,
                                L->panels.p, p->payload.p, p->payload2.p, p->kappa, s));
        return GCABEM_OK;
    }
    const int64_t r0 = L->block_rtask_at[b0], r1 = L->block_rtask_at[b1];
    const int64_t q0 = L->block_mtask_at[b0], q1 = L->block_mtask_at[b1];
    GC_CUDA(launch_disjoint(p->kind, p->order, m->charts.p, m->T.p, L->rtdesc.p + r0, r1 - r0,
                            L->panels.p, p->payload.p, p->payload2.p, p->kappa, s));
    GC_CUDA(launch_disjoint(p->kind + MIRRORED, p->order, m->charts.p, m->T.p,
                            L->mtdesc.p + q0, q1 - q0, L->panels.p, p->payload.p, p->payload2.p,
                            p->kappa, s));
    return GCABEM_OK;
}

// The singular lists of the items whose payload index lies in [p0, p1), as
// one fused launch (launch_singular_fused): mirrored vertex items, vertex
// items alone, edge items, identical items (half rule when available).
int enqueue_singular(gcabem_plan_t p, int64_t p0, int64_t p1) {
    gcabem_mesh_t m = p->mesh;
    gcabem_layout_t L = p->L;
    SingularBatch sb;
    int k = 0;
    auto add = [&](const SingItem *items, const int64_t *mout, int64_t n, const double *rule,
                   int64_t q, int same, GroupedRule g) {
        if (n <= 0) return;
        SingularSeg &seg = sb.seg[k];
        seg.items = items;
        seg.mout = mout;
        seg.n = n;
        seg.rule = rule;
        seg.q = q;
        seg.same = same;
        seg.grouped = g;
        sb.cta_at[k + 1] = sb.cta_at[k] + (n + GENERIC_TPB - 1) / GENERIC_TPB;
        ++k;
    };
    auto range = [&](const std::vector<int64_t> &v, int64_t a0, int64_t a1) {
        const int64_t lo = std::lower_bound(v.begin() + a0, v.begin() + a1, p0) - v.begin();
        const int64_t hi = std::lower_bound(v.begin() + a0, v.begin() + a1, p1) - v.begin();
        return std::make_pair(lo, hi);
    };
    if (vertex_mirrored(p)) {
        auto r = range(L->vm_out, 0, (int64_t)L->vm_out.size());
        add(L->vm_items.p + r.first, L->vm_mout.p + r.first, r.second - r.first, nullptr, 0, 0,
            grouped_of(p, 0));
        r = range(L->vp_out, 0, (int64_t)L->vp_out.size());
        add(L->vp_items.p + r.first, nullptr, r.second - r.first, p->srule[0].p, p->sq[0], 0,
            grouped_of(p, 0));
    } else {
        auto r = range(L->item_out, L->case_at[0], L->case_at[1]);
        add(L->items.p + r.first, nullptr, r.second - r.first, p->srule[0].p, p->sq[0], 0,
            grouped_of(p, 0));
    }
    {
        auto r = range(L->item_out, L->case_at[1], L->case_at[2]);
        add(L->items.p + r.first, nullptr, r.second - r.first, p->srule[1].p, p->sq[1], 0,
            grouped_of(p, 1));
    }
    {
        auto r = range(L->item_out, L->case_at[2], L->case_at[3]);
        const bool half = p->hq > 0;
        add(L->items.p + r.first, nullptr, r.second - r.first,
            half ? p->hrule.p : p->srule[2].p, half ? p->hq : p->sq[2], 1, grouped_of(p, 2));
    }
    for (int e = k + 1; e <= 4; ++e) sb.cta_at[e] = sb.cta_at[k];
    GC_CUDA(launch_singular_fused(p->kind, m->V.p, m->T.p, m->charts.p, sb, p->payload.p,
                                  p->payload2.p, p->kappa, p->stream));
    return GCABEM_OK;
}

int enqueue_range(gcabem_plan_t p, int64_t b0, int64_t b1, int64_t p0, int64_t p1) {
    if (int rc = enqueue_disjoint(p, b0, b1)) return rc;
    return enqueue_singular(p, p0, p1);
}

}  // namespace

int gcabem_plan_execute(gcabem_plan_t p) {
    GC_ARG(p, "null plan");
    gcabem_mesh_t m = p->mesh;
    GC_CUDA(cudaSetDevice(m->device));
    cudaStream_t s = p->stream;
    // no memset: the blocks tile every leaf and the disjoint kernels write
    // every entry (pairs sharing a vertex as 0, SKIP blocks by their primary)
    GC_CUDA(cudaEventRecord(p->ev[0], s));
    if (int rc = enqueue_disjoint(p, 0, (int64_t)p->L->block_leaf.size())) return rc;
    GC_CUDA(cudaEventRecord(p->ev[1], s));
    if (int rc = enqueue_singular(p, 0, p->payload_len)) return rc;
    GC_CUDA(cudaEventRecord(p->ev[2], s));
    p->executed = true;
    return GCABEM_OK;
}

int gcabem_plan_singular_evals(gcabem_plan_t p, int64_t *out5) {
    GC_ARG(p && out5, "null argument");
    gcabem_layout_t L = p->L;
    const bool vm = vertex_mirrored(p);
    out5[0] = vm ? (int64_t)L->vm_out.size() : 0;
    out5[1] = vm ? (int64_t)L->vp_out.size() : L->case_at[1] - L->case_at[0];
    out5[2] = L->case_at[2] - L->case_at[1];
    out5[3] = L->case_at[3] - L->case_at[2];
    out5[4] = p->hq > 0 ? p->hq : p->sq[2];   // rule points per identical item evaluated
    return GCABEM_OK;
}

int gcabem_plan_set_mirror(gcabem_plan_t p, int enable) {
    GC_ARG(p, "null plan");
    p->mirrored = enable && p->L->nmtasks > 0 && p->order <= MAX_MIRROR_ORDER;
    return GCABEM_OK;
}

int gcabem_plan_mirrored(gcabem_plan_t p, int *out) {
    GC_ARG(p && out, "null argument");
    *out = p->mirrored ? 1 : 0;
    return GCABEM_OK;
}

int gcabem_plan_execute_download(gcabem_plan_t p, double *host, int nchunks) {
    GC_ARG(p && !kind_pair(p->kind), "pair plans download with gcabem_plan_execute_download2");
    return gcabem_plan_execute_download2(p, host, nullptr, nchunks);
}

namespace {
int join_filler(gcabem_plan_t p) {
    if (p->filler.joinable()) p->filler.join();
    const int rc = p->fill_rc;
    p->fill_rc = 0;
    return rc ? set_error(rc, p->fill_msg) : GCABEM_OK;
}
}  // namespace

int gcabem_plan_set_symmetric_download(gcabem_plan_t p, int enable) {
    GC_ARG(p, "null plan");
    // the first payload is a single layer: symmetric under the mirror
    p->sym = enable && (p->kind == L_SLP || p->kind == H_SLP || kind_pair(p->kind));
    return GCABEM_OK;
}

int gcabem_plan_d2h_bytes(gcabem_plan_t p, int64_t *out) {
    GC_ARG(p && out, "null argument");
    *out = p->d2h_bytes;
    return GCABEM_OK;
}

int gcabem_plan_execute_download2(gcabem_plan_t p, double *host, double *host2, int nchunks) {
    GC_ARG(p && (host || p->payload_len == 0), "null argument");
    GC_ARG(!kind_pair(p->kind) || host2 || p->payload_len == 0,
           "pair plan: the double-layer target is missing");
    GC_CUDA(cudaSetDevice(p->mesh->device));
    if (int rc = join_filler(p)) return rc;
    gcabem_layout_t L = p->L;
    // symmetric download: host-filled SKIP leaves are not copied (see
    // gcabem_layout_s::hf_lo); needs the mirrored kernels to have written
    // their values (one value to both entries of a mirrored pair)
    const bool sym = p->sym && p->mirrored && !L->hf_lo.empty();
    const int64_t npatch = sym ? (int64_t)L->patch_out.size() : 0;
    if (npatch > 0) {
        // kept across executes (the previous execute's copies from it are
        // done: join_filler waited for them)
        if (p->patch_vals.n < (size_t)npatch) GC_CUDA(p->patch_vals.alloc(npatch, p->stream));
        if (p->patch_host_bytes < sizeof(double2) * npatch) {
            pinned_release(p->patch_host, p->patch_host_bytes);
            p->patch_host = (double2 *)pinned_acquire(sizeof(double2) * npatch,
                                                      &p->patch_host_bytes);
            if (!p->patch_host) {
                p->patch_host_bytes = 0;
                return set_error(GCABEM_ERR_CUDA, "pinned patch staging allocation failed");
            }
        }
    }
    p->d2h_bytes = 0;
    const int64_t B = (int64_t)p->L->block_leaf.size();
    if (nchunks < 1) nchunks = 1;
    // leaf-aligned chunk boundaries balanced by pairs
    std::vector<int64_t> cut{0};
    int64_t total = 0;
    for (int64_t b = 0; b < B; ++b) total += p->L->block_pairs[b];
    int64_t acc = 0, next = 1;
    for (int64_t b = 0; b < B && next < nchunks; ++b) {
        if (b > 0 && p->L->block_leaf[b] != p->L->block_leaf[b - 1] && acc * nchunks >= next * total) {
            cut.push_back(b);
            ++next;
        }
        acc += p->L->block_pairs[b];
    }
    cut.push_back(B);
    cudaStream_t s = p->stream;
    GC_CUDA(cudaEventRecord(p->ev[0], s));
    while ((int64_t)p->chunk_ev.size() < (int64_t)cut.size()) {
        cudaEvent_t e;
        GC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        p->chunk_ev.push_back(e);
    }
    if (sym)
        while (p->copy_ev.size() < p->chunk_ev.size()) {
            cudaEvent_t e;
            GC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            p->copy_ev.push_back(e);
        }
    double2 *h1 = reinterpret_cast<double2 *>(host);
    std::vector<std::pair<int64_t, int64_t>> fill;  // host-filled leaves per chunk
    auto copy = [&](double2 *dst, const double2 *src, int64_t n) -> cudaError_t {
        p->d2h_bytes += (int64_t)sizeof(double2) * n;
        return cudaMemcpyAsync(dst, src, sizeof(double2) * n, cudaMemcpyDeviceToHost, p->copy);
    };
    for (size_t k = 0; k + 1 < cut.size(); ++k) {
        const int64_t b0 = cut[k], b1 = cut[k + 1];
        const int64_t p0 = b0 < B ? L->block_base[b0] : p->payload_len;
        const int64_t p1 = b1 < B ? L->block_base[b1] : p->payload_len;
        // chunks run in leaf order, so every SKIP entry of this chunk was
        // written by its PRIMARY in this or an earlier chunk before this D2H
        if (int rc = enqueue_range(p, b0, b1, p0, p1)) return rc;
        int64_t s0 = 0, s1 = 0, q0 = 0, q1 = 0;
        if (sym) {
            s0 = std::lower_bound(L->hf_lo.begin(), L->hf_lo.end(), p0) - L->hf_lo.begin();
            s1 = std::lower_bound(L->hf_lo.begin(), L->hf_lo.end(), p1) - L->hf_lo.begin();
            q0 = L->hf_item_at[s0];
            q1 = L->hf_item_at[s1];
            if (q1 > q0)
                gather_entries_kernel<<<(unsigned)((q1 - q0 + 255) / 256), 256, 0, s>>>(
                    p->payload.p, L->patch_dev.p + q0, q1 - q0, p->patch_vals.p + q0);
            GC_CUDA(cudaGetLastError());
        }
        GC_CUDA(cudaEventRecord(p->chunk_ev[k], s));
        if (p1 > p0) {
            GC_CUDA(cudaStreamWaitEvent(p->copy, p->chunk_ev[k], 0));
            if (sym) {  // the chunk's payload minus its host-filled leaves
                int64_t cur = p0;
                for (int64_t h = s0; h < s1; ++h) {
                    if (L->hf_lo[h] > cur)
                        GC_CUDA(copy(h1 + cur, p->payload.p + cur, L->hf_lo[h] - cur));
                    cur = L->hf_lo[h] + (int64_t)L->hf_nr[h] * L->hf_nc[h];
                }
                if (cur < p1) GC_CUDA(copy(h1 + cur, p->payload.p + cur, p1 - cur));
                if (q1 > q0)
                    GC_CUDA(copy(p->patch_host + q0, p->patch_vals.p + q0, q1 - q0));
            } else {
                GC_CUDA(copy(h1 + p0, p->payload.p + p0, p1 - p0));
            }
            if (kind_pair(p->kind))
                GC_CUDA(copy(reinterpret_cast<double2 *>(host2) + p0, p->payload2.p + p0,
                             p1 - p0));
        }
        if (sym) {
            GC_CUDA(cudaEventRecord(p->copy_ev[k], p->copy));
            fill.emplace_back(s0, s1);
        }
    }
    GC_CUDA(cudaEventRecord(p->ev[1], s));
    GC_CUDA(cudaEventRecord(p->ev[2], s));
    p->executed = true;
    if (sym) {
        // the host side: chunk by chunk (copies complete in chunk order, so a
        // leaf's PRIMARY, in this or an earlier chunk, has arrived), the
        // chunk's host-filled leaves on the pool
        const int dev = p->mesh->device;
        std::vector<cudaEvent_t> evs(p->copy_ev.begin(), p->copy_ev.begin() + fill.size());
        double2 *patch = p->patch_host;
        p->filler = std::thread([p, L, h1, patch, dev, evs, fill]() {
            cudaSetDevice(dev);
            Trace tr("sym-fill");
            for (size_t k = 0; k < fill.size(); ++k) {
                if (cudaEventSynchronize(evs[k]) != cudaSuccess) {
                    p->fill_msg = std::string("symmetric download: ") +
                                  cudaGetErrorString(cudaGetLastError());
                    p->fill_rc = GCABEM_ERR_CUDA;
                    return;
                }
                tr.mark("copied");
                const int64_t s0 = fill[k].first, n = fill[k].second - fill[k].first;
                par_for(n, 32, [&](int64_t a, int64_t b, int) {
                    for (int64_t h = a; h < b; ++h) host_fill_leaf(L, s0 + h, h1, patch);
                }, fill_threads());
                tr.mark("filled");
            }
        });
    }
    return GCABEM_OK;
}

int gcabem_plan_download(gcabem_plan_t p, double *host) {
    return gcabem_plan_download2(p, host, nullptr);
}

int gcabem_plan_download2(gcabem_plan_t p, double *host, double *host2) {
    GC_ARG(p && (host || p->payload_len == 0), "null argument");
    GC_CUDA(cudaSetDevice(p->mesh->device));
    if (int rc = join_filler(p)) return rc;
    if (p->payload_len > 0)
        GC_CUDA(cudaMemcpyAsync(host, p->payload.p, sizeof(double2) * p->payload_len,
                                cudaMemcpyDeviceToHost, p->stream));
    if (p->payload_len > 0 && kind_pair(p->kind) && host2)
        GC_CUDA(cudaMemcpyAsync(host2, p->payload2.p, sizeof(double2) * p->payload_len,
                                cudaMemcpyDeviceToHost, p->stream));
    GC_CUDA(cudaStreamSynchronize(p->stream));
    return GCABEM_OK;
}

int gcabem_plan_synchronize(gcabem_plan_t p) {
    GC_ARG(p, "null plan");
    GC_CUDA(cudaSetDevice(p->mesh->device));
    GC_CUDA(cudaStreamSynchronize(p->stream));
    GC_CUDA(cudaStreamSynchronize(p->copy));
    return join_filler(p);
}

int gcabem_plan_timing(gcabem_plan_t p, float *ms3) {
    GC_ARG(p && ms3, "null argument");
    GC_ARG(p->executed, "plan not executed");
    GC_CUDA(cudaSetDevice(p->mesh->device));
    GC_CUDA(cudaEventSynchronize(p->ev[2]));
    GC_CUDA(cudaEventElapsedTime(&ms3[0], p->ev[0], p->ev[1]));
    GC_CUDA(cudaEventElapsedTime(&ms3[1], p->ev[1], p->ev[2]));
    GC_CUDA(cudaEventElapsedTime(&ms3[2], p->ev[0], p->ev[2]));
    return GCABEM_OK;
}

int gcabem_plan_set_stream(gcabem_plan_t p, void *stream) {
    GC_ARG(p, "null plan");
    GC_CUDA(cudaSetDevice(p->mesh->device));
    GC_CUDA(cudaStreamSynchronize(p->stream));
    if (p->own_stream == nullptr) p->own_stream = p->stream;
    p->stream = stream ? (cudaStream_t)stream : p->own_stream;
    return GCABEM_OK;
}

int gcabem_plan_payload(gcabem_plan_t p, void **dev_ptr) {
    GC_ARG(p && dev_ptr, "null argument");
    *dev_ptr = p->payload.p;
    return GCABEM_OK;
}

int gcabem_plan_destroy(gcabem_plan_t p) {
    if (!p) return GCABEM_OK;
    Trace tr("plan_destroy");
    cudaSetDevice(p->mesh->device);
    if (p->stream) cudaStreamSynchronize(p->stream);
    if (p->copy) cudaStreamSynchronize(p->copy);
    join_filler(p);
    for (auto &e : p->ev)
        if (e) cudaEventDestroy(e);
    for (auto &e : p->chunk_ev) cudaEventDestroy(e);
    for (auto &e : p->copy_ev) cudaEventDestroy(e);
    pinned_release(p->patch_host, p->patch_host_bytes);
    p->patch_vals.release();
    tr.mark("sync+events");
    p->payload.release();
    p->payload2.release();
    tr.mark("free");
    for (auto &r : p->srule) r.release();
    for (auto &r : p->grows) r.release();
    for (auto &r : p->ggroups) r.release();
    for (auto &r : p->gchunks) r.release();
    p->hrule.release();
    cudaStream_t mine = p->own_stream ? p->own_stream : p->stream;
    if (mine) cudaStreamDestroy(mine);
    if (p->copy) cudaStreamDestroy(p->copy);
    tr.mark("streams");
    gcabem_layout_release(p->L);
    delete p;
    tr.mark("layout");
    return GCABEM_OK;
}

int gcabem_green_matrices(gcabem_mesh_t mesh, int equation, double kappa, int64_t nclusters,
                          const int64_t *panel_at, const int64_t *panels, int64_t nsrc,
                          const double *src, int64_t nduffy, const double *duffy,
                          const int64_t *out_at, int64_t out_len, double *out_host) {
    GC_ARG(mesh, "null mesh");
    if (int rc = check_kind(equation, 0, kappa)) return rc;
    GC_ARG(nclusters >= 0 && nsrc > 0 && nduffy > 0, "bad sizes");
    if (nclusters == 0) return GCABEM_OK;
    GC_ARG(nclusters < (int64_t(1) << 31), "too many clusters");
    GC_CUDA(cudaSetDevice(mesh->device));
    const int64_t npan = panel_at[nclusters];
    std::vector<int32_t> pan(npan);
    for (int64_t k = 0; k < npan; ++k) {
        GC_ARG(panels[k] >= 0 && panels[k] < mesh->nt, "panel index out of range");
        pan[k] = (int32_t)panels[k];
    }
    std::vector<int2> tasks;
    for (int64_t c = 0; c < nclusters; ++c) {
        const int64_t ne = (panel_at[c + 1] - panel_at[c]) * nsrc;
        GC_ARG(ne >= 0 && ne < (int64_t(1) << 31), "cluster too large");
        GC_ARG(out_at[c] >= 0 && out_at[c] + ne <= out_len, "output range out of bounds");
        for (int64_t e0 = 0; e0 < ne; e0 += GREEN_TPB) tasks.push_back(make_int2((int)c, (int)e0));
    }
    const int64_t width = equation == 0 ? 1 : 2;
    cudaStream_t s = mesh->stream;
    DevBuf<int64_t> dpa, doa;
    DevBuf<int32_t> dpan;
    DevBuf<double> dsrc, dduf, dout;
    DevBuf<int2> dtask;
    GC_CUDA(dpa.upload(panel_at, nclusters + 1, s));
    GC_CUDA(doa.upload(out_at, nclusters, s));
    GC_CUDA(dpan.upload(pan.data(), pan.size(), s));
    GC_CUDA(dsrc.upload(src, (size_t)(nclusters * nsrc * 8), s));
    GC_CUDA(dduf.upload(duffy, (size_t)(3 * nduffy), s));
    GC_CUDA(dtask.upload(tasks.data(), tasks.size(), s));
    GC_CUDA(dout.alloc((size_t)(out_len * width)));
    GC_CUDA(launch_green(equation, mesh->charts.p, dtask.p, (int64_t)tasks.size(), dpa.p, dpan.p,
                         doa.p, (int)nsrc, dsrc.p, dduf.p, (int)nduffy, dout.p, kappa, s));
    GC_CUDA(cudaMemcpyAsync(out_host, dout.p, sizeof(double) * out_len * width,
                            cudaMemcpyDeviceToHost, s));
    GC_CUDA(cudaStreamSynchronize(s));
    return GCABEM_OK;
}

int gcabem_potential(gcabem_mesh_t mesh, int equation, int layer, double kappa, int order,
                     const double *gauss_pts, const double *gauss_wts, int64_t npts,
                     const double *points, double *out) {
    GC_ARG(mesh && out && (points || npts == 0), "null argument");
    if (int rc = check_kind(equation, layer, kappa)) return rc;
    GC_ARG(order >= 1 && order <= 8, "potential order outside [1, 8]");
    GC_ARG(npts >= 0, "negative size");
    if (npts == 0) return GCABEM_OK;
    GC_CUDA(cudaSetDevice(mesh->device));
    if (int rc = ensure_disjoint_rule(mesh->device, order, gauss_pts, gauss_wts)) return rc;
    // sum of the x-side Duffy weights (gx = 2 cancels the reference-triangle area)
    double xw = 0.0;
    for (int a = 0; a < order; ++a)
        for (int b = 0; b < order; ++b) xw += (gauss_wts[a] * gauss_wts[b]) * gauss_pts[a];
    cudaStream_t s = mesh->stream;
    DevBuf<double> dp;
    DevBuf<double2> dout;
    GC_CUDA(dp.upload(points, 3 * npts, s));
    GC_CUDA(dout.alloc(npts * mesh->nt));
    GC_CUDA(launch_potential(kind_of(equation, layer), order, mesh->charts.p, mesh->nt, dp.p, npts,
                             xw, dout.p, kappa, s));
    GC_CUDA(cudaMemcpyAsync(out, dout.p, sizeof(double2) * npts * mesh->nt,
                            cudaMemcpyDeviceToHost, s));
    GC_CUDA(cudaStreamSynchronize(s));
    return GCABEM_OK;
}

int gcabem_release_cached(int device) {
    GC_CUDA(cudaSetDevice(device));
    GC_CUDA(cudaDeviceSynchronize());
    gca_release_staging(device);
    {
        std::lock_guard<std::mutex> lock(g_pin_mutex);
        for (auto &kv : g_pin_free) cudaFreeHost(kv.second);
        g_pin_free.clear();
    }
    cudaMemPool_t pool;
    GC_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    GC_CUDA(cudaMemPoolTrimTo(pool, 0));
    return GCABEM_OK;
}

int gcabem_fp64_probe(int device, double *tflops) {
    GC_ARG(tflops, "null argument");
    GC_CUDA(cudaSetDevice(device));
    int sms = 0;
    GC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    DevBuf<double> sink;
    GC_CUDA(sink.alloc(1));
    cudaEvent_t a, b;
    GC_CUDA(cudaEventCreate(&a));
    GC_CUDA(cudaEventCreate(&b));
    const int iters = 1 << 14, blocks = sms * 8;
    GC_CUDA(launch_fp64_probe(sink.p, iters, blocks, 0));  // warm-up
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        GC_CUDA(cudaEventRecord(a, 0));
        GC_CUDA(launch_fp64_probe(sink.p, iters, blocks, 0));
        GC_CUDA(cudaEventRecord(b, 0));
        GC_CUDA(cudaEventSynchronize(b));
        float ms = 0.f;
        GC_CUDA(cudaEventElapsedTime(&ms, a, b));
        best = std::min(best, ms);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    const double flops = 2.0 * 8.0 * iters * (double)blocks * 256.0;
    *tflops = flops / (best * 1e-3) / 1e12;
    return GCABEM_OK;
}

}  // extern "C"
