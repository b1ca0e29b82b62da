// disjoint_kernel<N, KIND> for orders 5..8 (see disjoint.cuh)
#include "disjoint.cuh"

namespace gcabem {

cudaError_t upload_disjoint_rule_o5_8(int n, const double *g, const double *gw) {
    return upload_tables(n, g, gw);
}

cudaError_t launch_disjoint_o5_8(int kind, int order, const Chart *charts, const int32_t *T,
                                const TaskDesc *tasks, int64_t ntasks,
                                const int32_t *panels, double2 *payload, double2 *payload2,
                                double kappa, cudaStream_t s) {
    switch (order) {
        case 5: return launch_disjoint_n<5>(kind, charts, T, tasks, ntasks, panels, payload, payload2, kappa, s);
        case 6: return launch_disjoint_n<6>(kind, charts, T, tasks, ntasks, panels, payload, payload2, kappa, s);
        case 7: return launch_disjoint_n<7>(kind, charts, T, tasks, ntasks, panels, payload, payload2, kappa, s);
        case 8: return launch_disjoint_n<8>(kind, charts, T, tasks, ntasks, panels, payload, payload2, kappa, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace gcabem
