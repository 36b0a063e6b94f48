// tcgen05 tensor-core NUDFT (placeholder until the tensor-core GEMMs land).
#pragma once

#include <vector>

#include "common.cuh"

namespace csr {

struct TcPlan {
    bool enabled = false;
    int split = 1;
    float2 *ws = nullptr;
    int fwd_launches = 0, adj_launches = 0;
};

inline int tc_plan_build(TcPlan &tc, int, int, int, int, int64_t, const float2 *,
                         const float2 *, cudaStream_t, int64_t *, int64_t *,
                         std::vector<void *> &) {
    tc.enabled = false;
    return 0;
}
inline int tc_forward(TcPlan &, const float2 *, const float2 *, float2 *, cudaStream_t,
                      const int *) {
    return 3;
}
inline int tc_adjoint(TcPlan &, const float2 *, float2 *, cudaStream_t, const int *) {
    return 3;
}

}  // namespace csr
