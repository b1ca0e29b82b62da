// disjoint_kernel<N, KIND> for orders 1..4 (see disjoint.cuh)
#include "disjoint.cuh"

namespace gcabem {

cudaError_t upload_disjoint_rule_o1_4(int n, const double *g, const double *gw) {
    return upload_tables(n, g, gw);
}

cudaError_t launch_disjoint_o1_4(int kind, int order, const Chart *charts, const int32_t *T,
                                const TaskDesc *tasks, int64_t ntasks,
                                const int32_t *panels, double2 *payload, double2 *payload2,
                                double kappa, cudaStream_t s) {
    switch (order) {
        case 1: return launch_disjoint_n<1>(kind, charts, T, tasks, ntasks, panels, payload, payload2, kappa, s);
        case 2: return launch_disjoint_n<2>(kind, charts, T, tasks, ntasks, panels, payload, payload2, kappa, s);
        case 3: return launch_disjoint_n<3>(kind, charts, T, tasks, ntasks, panels, payload, payload2, kappa, s);
        case 4: return launch_disjoint_n<4>(kind, charts, T, tasks, ntasks, panels, payload, payload2, kappa, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace gcabem
