// fast_kernels.cuh -- specialised kernels for the hot inner shapes.
#pragma once
#include <cuda_runtime.h>

#include "../../include/nsdgt.h"
#include "cplx.cuh"

namespace nsdgt {

struct FastPlan {
    int kind = 0;  // 0 = none (generic path)
    const char* name = "none";
};

template <typename T>
int build_fast(FastPlan* fp, const dgt_lattice_info&, void*, void*, void*, int*, bool, cudaStream_t) {
    fp->kind = 0;
    return DGT_OK;
}
inline void free_fast(FastPlan*) {}
inline size_t fast_workspace_bytes(const FastPlan*, int64_t) { return 0; }
inline int64_t fast_chunk(const FastPlan*) { return 1; }
template <typename T>
int launch_fast(FastPlan*, const void*, int, void*, void*, int64_t, cudaStream_t) { return DGT_EUNSUPPORTED; }
inline int64_t fast_launches_per_chunk(const FastPlan*) { return 2; }

}  // namespace nsdgt
