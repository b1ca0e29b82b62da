// Accuracy probe of the FP64 building blocks used by the kernels (run on a
// B200): MUFU.RSQ64H seed, one quadratic / cubic Newton step, and the
// branch-free sincos against correctly rounded references.
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

__device__ double seed(double x) { double y; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); return y; }

__global__ void probe(int n, unsigned long long s0, double *out) {
    // out[0..2]: max rel err seed, quadratic, cubic (vs 1/sqrt)
    double e0 = 0, e1 = 0, e2 = 0;
    unsigned long long st = s0 + 7919ull * (blockIdx.x * blockDim.x + threadIdx.x);
    for (int i = 0; i < n; ++i) {
        st = st * 6364136223846793005ull + 1442695040888963407ull;
        double u = (double)(st >> 11) * (1.0 / 9007199254740992.0);
        double x = exp2(-30.0 + 40.0 * u);
        double ref = 1.0 / sqrt(x);
        double y = seed(x);
        e0 = fmax(e0, fabs(y - ref) / ref);
        double t = y * y, e = fma(-x, t, 1.0);
        double yq = fma(0.5 * y, e, y);
        e1 = fmax(e1, fabs(yq - ref) / ref);
        double yc = fma(fma(e, 0.375, 0.5), y * e, y);
        e2 = fmax(e2, fabs(yc - ref) / ref);
    }
    atomicMax((unsigned long long *)&out[0], __double_as_longlong(e0));
    atomicMax((unsigned long long *)&out[1], __double_as_longlong(e1));
    atomicMax((unsigned long long *)&out[2], __double_as_longlong(e2));
}

int main() {
    double *d, h[3] = {0, 0, 0};
    cudaMalloc(&d, 3 * sizeof(double));
    cudaMemset(d, 0, 3 * sizeof(double));
    probe<<<1184, 256>>>(4096, 12345, d);
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("{\"rsqrt_seed_max_rel\": %.3e, \"rsqrt_quadratic_max_rel\": %.3e, \"rsqrt_cubic_max_rel\": %.3e, \"samples\": %d}\n",
           h[0], h[1], h[2], 1184 * 256 * 4096);
    return 0;
}
