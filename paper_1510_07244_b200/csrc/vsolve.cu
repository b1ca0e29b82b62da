// GCA interpolation-operator solves on the device: the part of the
// reference's build_interpolation_operator (gca.py:248-282) after ACA, for
// many clusters per launch (the pivots themselves stay on the CPU):
//
//   cond check  np.linalg.cond(B) <= 1e14, decided by the Frobenius bracket
//               kF / k <= cond2 <= kF (kF = |B|_F |B^-1|_F): accept below
//               0.5e14, reject above 2e14 k, else hand back to the host (its
//               exact Jacobi SVD decides);
//   V           = A[:, cols] B^-1 by LU with partial pivoting of B^T (pivot
//               choice |re| + |im| as LAPACK izamax, first maximum wins) and
//               the reference's two refinement sweeps with their early exit.
//
// Same operations in the same order as the host solve (aca.cpp solve_one),
// with explicit roundings (no FMA contraction): V is bitwise the host's except
// where a residual maximum lands on the early-exit threshold. One CTA per
// cluster factors the pivot block; the right-hand sides (rows of V) spread
// over CTAs of VS_ROWS rows, the early exit decided from per-cluster maxima.
#include <cuda_runtime.h>

#include "internal.h"

namespace gcabem {
namespace {

constexpr int VS_TPB = VS_ROWS;

struct Cx {
    double re, im;
};
__device__ __forceinline__ double mul_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_(double a, double b) { return __dsub_rn(a, b); }

template <typename T>
struct Ops;
template <>
struct Ops<double> {
    __device__ static double mul(double a, double b) { return mul_(a, b); }
    __device__ static double sub(double a, double b) { return sub_(a, b); }
    __device__ static double add(double a, double b) { return add_(a, b); }
    __device__ static double div(double a, double b) { return a / b; }
    __device__ static double abs1(double a) { return fabs(a); }
    __device__ static double mag(double a) { return fabs(a); }
    __device__ static double norm2(double a) { return mul_(a, a); }
    __device__ static double zero() { return 0.0; }
    __device__ static double one() { return 1.0; }
};
template <>
struct Ops<Cx> {
    __device__ static Cx mul(Cx a, Cx b) {
        return {sub_(mul_(a.re, b.re), mul_(a.im, b.im)), add_(mul_(a.re, b.im), mul_(a.im, b.re))};
    }
    __device__ static Cx sub(Cx a, Cx b) { return {sub_(a.re, b.re), sub_(a.im, b.im)}; }
    __device__ static Cx add(Cx a, Cx b) { return {add_(a.re, b.re), add_(a.im, b.im)}; }
    __device__ static Cx div(Cx a, Cx b) {  // numpy CDOUBLE_divide (Smith)
        if (fabs(b.re) >= fabs(b.im)) {
            const double rat = b.im / b.re, scl = 1.0 / add_(b.re, mul_(b.im, rat));
            return {mul_(add_(a.re, mul_(a.im, rat)), scl), mul_(sub_(a.im, mul_(a.re, rat)), scl)};
        }
        const double rat = b.re / b.im, scl = 1.0 / add_(b.im, mul_(b.re, rat));
        return {mul_(add_(mul_(a.re, rat), a.im), scl), mul_(sub_(mul_(a.im, rat), a.re), scl)};
    }
    __device__ static double abs1(Cx a) { return fabs(a.re) + fabs(a.im); }
    __device__ static double mag(Cx a) { return hypot(a.re, a.im); }
    __device__ static double norm2(Cx a) { return add_(mul_(a.re, a.re), mul_(a.im, a.im)); }
    __device__ static Cx zero() { return {0.0, 0.0}; }
    __device__ static Cx one() { return {1.0, 0.0}; }
};

// x (k values at stride ld) <- M^-1 x with the LU factors in shared memory,
// in the order of the host LU<T>::solve
template <typename T>
__device__ __forceinline__ void lu_solve(const T *m, const int *piv, int k, T *x, int64_t ld) {
    using O = Ops<T>;
    for (int i = 0; i < k; ++i)
        if (piv[i] != i) {
            const T t = x[i * ld];
            x[i * ld] = x[piv[i] * ld];
            x[piv[i] * ld] = t;
        }
    for (int i = 1; i < k; ++i) {
        T s = x[i * ld];
        for (int j = 0; j < i; ++j) s = O::sub(s, O::mul(m[i * k + j], x[j * ld]));
        x[i * ld] = s;
    }
    for (int i = k - 1; i >= 0; --i) {
        T s = x[i * ld];
        for (int j = i + 1; j < k; ++j) s = O::sub(s, O::mul(m[i * k + j], x[j * ld]));
        x[i * ld] = O::div(s, m[i * k + i]);
    }
}

// fixed-shape tree: deterministic for the fixed block size
__device__ __forceinline__ double block_sum(double v, double *red) {
    red[threadIdx.x] = v;
    __syncthreads();
    for (int s = VS_TPB / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    const double r = red[0];
    __syncthreads();
    return r;
}

// scratch of one task (doubles from scr_off): LU factors F (k x k), pivots
// (k int32), X = V^T (k x nr, [b][q]), R (k x nr; (B^T)^-1 columns in the
// factor kernel)
template <typename T>
struct TaskView {
    const T *B, *Ct;
    T *V, *F, *X, *R;
    int *piv;
    int k, nr;
    __device__ TaskView(const VTask &tk, const double *in, double *out, double *scratch) {
        k = tk.k;
        nr = tk.nr;
        B = reinterpret_cast<const T *>(in + tk.in_off);  // k x k: B[a][b] = A[rows[a], cols[b]]
        Ct = B + (int64_t)k * k;                           // k x nr: A[q, cols[b]] at [b][q]
        V = reinterpret_cast<T *>(out + tk.out_off);      // nr x k
        F = reinterpret_cast<T *>(scratch + tk.scr_off);
        piv = reinterpret_cast<int *>(F + (int64_t)k * k);
        X = reinterpret_cast<T *>(reinterpret_cast<double *>(F + (int64_t)k * k) + (k + 1) / 2);
        R = X + (int64_t)k * nr;
    }
};

// nonnegative doubles order like their bit patterns: atomicMax on the bits
__device__ __forceinline__ void atomic_max_nonneg(unsigned long long *slot, double v) {
    atomicMax(slot, (unsigned long long)__double_as_longlong(v));
}
__device__ __forceinline__ double load_max(const unsigned long long *slot) {
    return __longlong_as_double((long long)*slot);
}

// One CTA per task: LU with partial pivoting of M = B^T, then the Frobenius
// condition bracket from (B^T)^-1.
template <typename T>
__global__ void __launch_bounds__(VS_TPB)
vs_factor_kernel(const VTask *__restrict__ tasks, const double *__restrict__ in,
                 double *__restrict__ out, double *__restrict__ scratch, VAux *__restrict__ aux) {
    using O = Ops<T>;
    extern __shared__ double smem_raw[];
    T *m = reinterpret_cast<T *>(smem_raw);
    __shared__ int piv[VS_KMAX];
    __shared__ double red[VS_TPB];
    __shared__ int flag;
    const TaskView<T> tv(tasks[blockIdx.x], in, out, scratch);
    const int k = tv.k;
    for (int e = threadIdx.x; e < k * k; e += VS_TPB) {
        const int b = e / k, a = e - b * k;
        m[b * k + a] = tv.B[a * k + b];
    }
    if (threadIdx.x == 0) flag = 0;
    __syncthreads();
    for (int kk = 0; kk < k; ++kk) {
        if (threadIdx.x < 32) {  // pivot: first maximum of |re| + |im| in column kk
            double best = -1.0;
            int p = kk;
            for (int i = kk + threadIdx.x; i < k; i += 32) {
                const double v = O::abs1(m[i * k + kk]);
                if (v > best) {
                    best = v;
                    p = i;
                }
            }
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int op = __shfl_xor_sync(0xffffffffu, p, o);
                if (ob > best || (ob == best && op < p)) {
                    best = ob;
                    p = op;
                }
            }
            if (threadIdx.x == 0) {
                piv[kk] = p;
                if (!(best > 0.0)) flag = 2;  // exactly singular: cond = inf
            }
        }
        __syncthreads();
        if (flag) break;
        const int p = piv[kk];
        if (p != kk)
            for (int j = threadIdx.x; j < k; j += VS_TPB) {
                const T t = m[kk * k + j];
                m[kk * k + j] = m[p * k + j];
                m[p * k + j] = t;
            }
        __syncthreads();
        const T d = m[kk * k + kk];
        for (int i = kk + 1 + threadIdx.x; i < k; i += VS_TPB) m[i * k + kk] = O::div(m[i * k + kk], d);
        __syncthreads();
        const int w = k - kk - 1;
        for (int e = threadIdx.x; e < w * w; e += VS_TPB) {
            const int i = kk + 1 + e / w, j = kk + 1 + e % w;
            m[i * k + j] = O::sub(m[i * k + j], O::mul(m[i * k + kk], m[kk * k + j]));
        }
        __syncthreads();
    }
    if (flag) {
        if (threadIdx.x == 0) aux[blockIdx.x].status = flag;
        return;
    }
    for (int e = threadIdx.x; e < k * k; e += VS_TPB) tv.F[e] = m[e];
    for (int i = threadIdx.x; i < k; i += VS_TPB) tv.piv[i] = piv[i];
    double fb = 0.0, fi = 0.0;
    for (int e = threadIdx.x; e < k * k; e += VS_TPB) fb = add_(fb, O::norm2(tv.B[e]));
    for (int col = threadIdx.x; col < k; col += VS_TPB) {
        T *y = tv.R + col;
        for (int i = 0; i < k; ++i) y[i * k] = O::zero();
        y[col * k] = O::div(O::one(), O::one());
        lu_solve<T>(m, piv, k, y, k);
        for (int i = 0; i < k; ++i) fi = add_(fi, O::norm2(y[i * k]));
    }
    fb = block_sum(fb, red);
    fi = block_sum(fi, red);
    const double kf = sqrt(fb) * sqrt(fi);
    int decision;
    if (!(kf == kf)) decision = 2;
    else if (kf <= 0.5e14) decision = 0;
    else if (kf >= 2e14 * (double)k) decision = 2;
    else decision = 3;
    if (threadIdx.x == 0) aux[blockIdx.x].status = decision;
}

// One CTA per (task, VS_ROWS right-hand sides); thread = one row q of V.
//   STEP 0    X = M^-1 A_cols^T, amax = max |A_cols|
//   STEP 1/2  residual of sweep STEP-1 (sweep 1 only after sweep 0 missed the
//             limit), rmax[sweep]
//   STEP 3/4  correction of sweep STEP-3 when its rmax is above the limit;
//             STEP 4 also stores V = X^T
template <typename T, int STEP>
__global__ void __launch_bounds__(VS_TPB)
vs_rhs_kernel(const VTask *__restrict__ tasks, const int2 *__restrict__ chunks,
              const double *__restrict__ in, double *__restrict__ out,
              double *__restrict__ scratch, VAux *__restrict__ aux) {
    using O = Ops<T>;
    extern __shared__ double smem_raw[];
    T *m = reinterpret_cast<T *>(smem_raw);
    __shared__ int piv[VS_KMAX];
    const int2 ch = chunks[blockIdx.x];
    VAux &ax = aux[ch.x];
    if (ax.status != 0) return;
    const TaskView<T> tv(tasks[ch.x], in, out, scratch);
    const int k = tv.k, nr = tv.nr;
    const int q = ch.y + threadIdx.x;
    const double lim = STEP > 0 ? 1e-15 * fmax(load_max(&ax.amax), 1.0) : 0.0;
    bool solve = true;
    if (STEP == 2 || STEP == 3) solve = load_max(&ax.rmax[0]) > lim;
    if (STEP == 4) solve = load_max(&ax.rmax[0]) > lim && load_max(&ax.rmax[1]) > lim;
    if (STEP == 1 || STEP == 2) {
        if (!solve) return;
        // R = A_cols^T - M X, per row q: r_b = Ct[b][q] - sum_l B[l][b] x_l
        double rmax = 0.0;
        if (q < nr)
            for (int b = 0; b < k; ++b) {
                T s = tv.Ct[(int64_t)b * nr + q];
                for (int l = 0; l < k; ++l)
                    s = O::sub(s, O::mul(tv.B[l * k + b], tv.X[(int64_t)l * nr + q]));
                tv.R[(int64_t)b * nr + q] = s;
                rmax = fmax(rmax, O::mag(s));
            }
        for (int o = 16; o > 0; o >>= 1) rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
        if ((threadIdx.x & 31) == 0) atomic_max_nonneg(&ax.rmax[STEP - 1], rmax);
        return;
    }
    if (solve) {
        for (int e = threadIdx.x; e < k * k; e += VS_TPB) m[e] = tv.F[e];
        for (int i = threadIdx.x; i < k; i += VS_TPB) piv[i] = tv.piv[i];
        __syncthreads();
    }
    if (q >= nr) return;
    if (STEP == 0) {
        double amax = 0.0;
        for (int b = 0; b < k; ++b) {
            const T v = tv.Ct[(int64_t)b * nr + q];
            tv.X[(int64_t)b * nr + q] = v;
            amax = fmax(amax, O::mag(v));
        }
        lu_solve<T>(m, piv, k, tv.X + q, nr);
        atomic_max_nonneg(&ax.amax, amax);
        return;
    }
    if (solve) {
        T *r = tv.R + q;
        lu_solve<T>(m, piv, k, r, nr);
        for (int b = 0; b < k; ++b)
            tv.X[(int64_t)b * nr + q] = O::add(tv.X[(int64_t)b * nr + q], r[(int64_t)b * nr]);
    }
    if (STEP == 4)
        for (int b = 0; b < k; ++b) tv.V[(int64_t)q * k + b] = tv.X[(int64_t)b * nr + q];
}

template <typename T>
cudaError_t vsolve_all(const VTask *tasks, int ntasks, const int2 *chunks, int nchunks, int kmax,
                       const double *in, double *out, double *scratch, VAux *aux, cudaStream_t s) {
    const size_t smem = (size_t)kmax * kmax * sizeof(T);
    const int cap = VS_KMAX * VS_KMAX * (int)sizeof(T);
    // per call: the attribute belongs to the current device
    cudaFuncSetAttribute(vs_factor_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
    cudaFuncSetAttribute(vs_rhs_kernel<T, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
    cudaFuncSetAttribute(vs_rhs_kernel<T, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
    cudaFuncSetAttribute(vs_rhs_kernel<T, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
    cudaError_t e = cudaMemsetAsync(aux, 0, sizeof(VAux) * ntasks, s);
    if (e != cudaSuccess) return e;
    vs_factor_kernel<T><<<ntasks, VS_TPB, smem, s>>>(tasks, in, out, scratch, aux);
    vs_rhs_kernel<T, 0><<<nchunks, VS_TPB, smem, s>>>(tasks, chunks, in, out, scratch, aux);
    vs_rhs_kernel<T, 1><<<nchunks, VS_TPB, 0, s>>>(tasks, chunks, in, out, scratch, aux);
    vs_rhs_kernel<T, 3><<<nchunks, VS_TPB, smem, s>>>(tasks, chunks, in, out, scratch, aux);
    vs_rhs_kernel<T, 2><<<nchunks, VS_TPB, 0, s>>>(tasks, chunks, in, out, scratch, aux);
    vs_rhs_kernel<T, 4><<<nchunks, VS_TPB, smem, s>>>(tasks, chunks, in, out, scratch, aux);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_vsolve(bool is_complex, const VTask *tasks, int ntasks, const int2 *chunks,
                          int nchunks, int kmax, const double *in, double *out, double *scratch,
                          VAux *aux, cudaStream_t s) {
    if (ntasks <= 0) return cudaSuccess;
    if (is_complex)
        return vsolve_all<Cx>(tasks, ntasks, chunks, nchunks, kmax, in, out, scratch, aux, s);
    return vsolve_all<double>(tasks, ntasks, chunks, nchunks, kmax, in, out, scratch, aux, s);
}

}  // namespace gcabem
