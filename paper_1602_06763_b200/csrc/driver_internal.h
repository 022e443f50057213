// driver_internal.h — shared between driver.cu and dist.cu (not part of the ABI).
#pragma once
#include <cuda_runtime.h>

#include <functional>
#include <string>
#include <vector>

#include "plan.h"

namespace relapack {
void set_error(const std::string& s);
int cuda_fail(cudaError_t e, const char* what);
PlanParams current_params();
int trsm_base_cols();
// Enqueue the whole recursive factorization of the device L-view matrix A on st.
// With `host` (pinned), A is the device staging buffer and the H2D/D2H copies
// of the uplo triangle are part of the captured DAG.
// blocked_nb > 0: the blocked right-looking algorithm (relapack_dpotrf_blocked).
int enqueue_potrf(int dev, double* A, int n, int64_t ld, int layout, int* d_info, cudaStream_t st,
                  const double* host = nullptr, int64_t hld = 0, int blocked_nb = 0);
struct UpdateOp;
// Graph capture of a plan as its footprint-dependency DAG (driver.cu), shared
// with the multi-GPU executor: launch(i, st) issues op i on the capturing stream.
cudaError_t capture_plan_dag(const std::vector<PlanOp>& ops, const std::vector<std::vector<int>>& deps,
                             cudaStream_t st, const std::function<cudaError_t(size_t, cudaStream_t)>& launch,
                             std::vector<cudaGraphNode_t>& nodes, std::vector<char>& cls);
cudaError_t set_node_priorities(const std::vector<cudaGraphNode_t>& nodes, const std::vector<char>& cls);
cudaError_t setup_splitk_ops(const std::vector<PlanOp>& ops, std::vector<UpdateOp>& upd,
                             const std::vector<uint64_t>* anc, double** ws, int** cnt, size_t* cnt_bytes);
// The stream set with relapack_set_stream, or `fallback` if none was set.
cudaStream_t current_stream_or(cudaStream_t fallback);
}  // namespace relapack
