// Hot-column gather plan: shared declarations (hotcols.cu builds the plan,
// segwarp.cuh seg8_hot_kernel consumes it).
#pragma once

#include "common.cuh"

namespace wk {

// Gather plan view (hotcols.cu): nhot cached columns (<= kHotMax), their ids,
// and the rewritten column array (col2[k] = ~slot for cached columns).
constexpr int kHotMax = 8192;
constexpr int kHotThreads = 1024;

struct GatherPlan {
    const int* nhot;  // device scalar
    const int* hot;   // [kHotMax] column ids
    const int* col2;  // [nnz]
};
GatherPlan gather_plan_view(const void* plan);  // hotcols.cu

}  // namespace wk
