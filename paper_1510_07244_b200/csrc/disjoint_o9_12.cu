// disjoint_kernel<N, KIND> for orders 9..12 (see disjoint.cuh)
#include "disjoint.cuh"

namespace gcabem {

cudaError_t upload_disjoint_rule_o9_12(int n, const double *g, const double *gw) {
    return upload_tables(n, g, gw);
}

cudaError_t launch_disjoint_o9_12(int kind, int order, const Chart *charts, const int32_t *T,
                                const TaskDesc *tasks, int64_t ntasks,
                                const int32_t *panels, double2 *payload, double2 *payload2,
                                double kappa, cudaStream_t s) {
    switch (order) {
        case 9: return launch_disjoint_n<9>(kind, charts, T, tasks, ntasks, panels, payload, payload2, kappa, s);
        case 10: return launch_disjoint_n<10>(kind, charts, T, tasks, ntasks, panels, payload, payload2, kappa, s);
        case 11: return launch_disjoint_n<11>(kind, charts, T, tasks, ntasks, panels, payload, payload2, kappa, s);
        case 12: return launch_disjoint_n<12>(kind, charts, T, tasks, ntasks, panels, payload, payload2, kappa, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace gcabem
