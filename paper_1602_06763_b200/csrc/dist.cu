// dist.cu — multi-GPU mode (north_star subsystem (4)): one
// process per GPU, the top recursion levels' TRSM and SYRK/GEMM trailing
// updates sharded by row blocks of the L-view (block-cyclic, block nb; for
// uplo 'U' these are memory block-columns), the freshly solved panel rows
// all-gathered with NCCL over NVLink/NVSwitch, and nodes below dist_min
// factored redundantly on every rank.  The schedule is plan.cpp's
// build_dist_plan; this file executes it:
//   OP_PACK      this rank's owned rows of a block -> contiguous send buffer
//   OP_TRSM/GEMM the recursive TRSM on the packed rows (BUF_SEND)
//   OP_ALLGATHER ncclAllGather(send, recv)
//   OP_UNPACK    every rank's rows -> the matrix (replicated L21)
//   OP_SYRK/GEMM the owned row blocks of the trailing update
// NCCL is loaded with dlopen (the torch-bundled libnccl.so.2 in the process),
// so the library has no link-time NCCL dependency.  A loopback executor runs
// P virtual ranks on one GPU (collectives emulated with device copies between
// the ranks' buffers, ranks executed one after another between collectives:
// no kernel ever waits on another rank) for tests.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdio>
#include <cstring>
#include <chrono>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../include/relapack.h"
#include "common.cuh"
#include "driver_internal.h"
#include "kernels.h"
#include "plan.h"

// ---------------------------------------------------------------- NCCL (dlopen)
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;  // ncclSuccess == 0
enum { ncclDouble_ = 8, ncclInt32_ = 2, ncclMax_ = 2 };

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok() const { return h && GetUniqueId && CommInitRank && CommDestroy && AllGather && AllReduce; }
};

static NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  const char* env = getenv("RELAPACK_NCCL_LIB");
  const char* names[] = {env ? env : "libnccl.so.2", "libnccl.so.2", "libnccl.so"};
  for (const char* nm : names) {
    if (!nm) continue;
    api.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    if (api.h) break;
  }
  if (!api.h) return api;
  api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(api.h, "ncclGetUniqueId");
  api.CommInitRank = (decltype(api.CommInitRank))dlsym(api.h, "ncclCommInitRank");
  api.CommDestroy = (decltype(api.CommDestroy))dlsym(api.h, "ncclCommDestroy");
  api.AllGather = (decltype(api.AllGather))dlsym(api.h, "ncclAllGather");
  api.AllReduce = (decltype(api.AllReduce))dlsym(api.h, "ncclAllReduce");
  api.GetErrorString = (decltype(api.GetErrorString))dlsym(api.h, "ncclGetErrorString");
  api.CommGetAsyncError = (decltype(api.CommGetAsyncError))dlsym(api.h, "ncclCommGetAsyncError");
  api.CommAbort = (decltype(api.CommAbort))dlsym(api.h, "ncclCommAbort");
  return api;
}

namespace relapack {
struct DistPlan;
void destroy_dist_plan(DistPlan* p);
}  // namespace relapack

struct relapack_comm {
  int nranks = 1, rank = 0, device = 0;
  ncclComm_t nccl = nullptr;
  cudaStream_t stream = nullptr;
  cudaStream_t capture = nullptr;  // graph capture of the distributed plan
  int* d_info = nullptr;  // 2 ints: local info, reduced info
  bool aborted = false;
  // single-entry schedule cache (key: n, lda, layout, nb, dist_min, c, T, A)
  relapack::DistPlan* plan = nullptr;
  std::string key;
};

namespace relapack {

namespace {

// ---------------------------------------------------------------- pack / unpack
// Row tables: rows[s * rows_pad + r] = global L-view row of rank s's r-th owned
// row in [lo, hi), -1 for padding.
std::vector<int> row_table(int lo, int hi, const DistParams& d, int rows_pad) {
  std::vector<int> t((size_t)d.nranks * rows_pad, -1);
  for (int s = 0; s < d.nranks; ++s) {
    int r = 0;
    for (int b = lo / d.nb; b * d.nb < hi; ++b) {
      if (dist_owner_block(b, d) != s) continue;
      const int g0 = b * d.nb > lo ? b * d.nb : lo;
      const int g1 = (b + 1) * d.nb < hi ? (b + 1) * d.nb : hi;
      for (int g = g0; g < g1; ++g) t[(size_t)s * rows_pad + r++] = g;
    }
  }
  return t;
}

// Packed chunk layout (L-view, same layout as the matrix): element (r, c) at
// chunk + r + c * rows_pad (layout N) or chunk + c + r * ncols (layout T).
__global__ void k_pack_rows(const double* __restrict__ A, int64_t lda, int layout, const int* __restrict__ rows,
                            int rows_pad, int c0, int ncols, double* __restrict__ W, const int* d_info) {
  if (ld_info(d_info) != 0) return;
  const int64_t total = (int64_t)rows_pad * ncols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int r, c;
    if (layout == kLayoutN) {
      r = (int)(e % rows_pad);
      c = (int)(e / rows_pad);
    } else {
      c = (int)(e % ncols);
      r = (int)(e / ncols);
    }
    const int g = rows[r];
    const double v = g >= 0 ? A[lv_off(layout, g, c0 + c, lda)] : 0.0;
    W[layout == kLayoutN ? r + (int64_t)c * rows_pad : c + (int64_t)r * ncols] = v;
  }
}

__global__ void k_unpack_rows(double* __restrict__ A, int64_t lda, int layout, const int* __restrict__ rows,
                              int rows_pad, int nranks, int c0, int ncols, const double* __restrict__ R,
                              const int* d_info) {
  if (ld_info(d_info) != 0) return;
  const int64_t per = (int64_t)rows_pad * ncols;
  const int64_t total = per * nranks;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int s = (int)(e / per);
    const int64_t q = e - s * per;
    int r, c;
    if (layout == kLayoutN) {
      r = (int)(q % rows_pad);
      c = (int)(q / rows_pad);
    } else {
      c = (int)(q % ncols);
      r = (int)(q / ncols);
    }
    const int g = rows[(int64_t)s * rows_pad + r];
    if (g >= 0) A[lv_off(layout, g, c0 + c, lda)] = R[s * per + q];
  }
}

int grid_for(int64_t total) {
  int64_t b = (total + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  return (int)(b < 1 ? 1 : b);
}

}  // namespace

// ---------------------------------------------------------------- executor
struct DistPlan {
  std::vector<PlanOp> ops;
  std::vector<UpdateOp> upd;           // GEMM/SYRK descriptors (by op index)
  std::vector<int*> d_rows;            // PACK/UNPACK row tables (by op index)
  std::vector<int> rows_pad;           // by op index (PACK/UNPACK/ALLGATHER/TRSM on send)
  std::vector<int> ncols;              // columns of the current packed chunk (by op index)
  double* send = nullptr;
  double* recv = nullptr;
  int64_t send_elems = 0;
  double* splitk_ws = nullptr;         // split-K partials (graph executor)
  int* splitk_cnt = nullptr;
  size_t cnt_bytes = 0;
  cudaGraphExec_t exec = nullptr;      // the whole distributed plan, collectives included
  ~DistPlan() {
    if (exec) cudaGraphExecDestroy(exec);
    for (int* p : d_rows)
      if (p) cudaFree(p);
    if (send) cudaFree(send);
    if (recv) cudaFree(recv);
    if (splitk_ws) cudaFree(splitk_ws);
    if (splitk_cnt) cudaFree(splitk_cnt);
  }
};

namespace {

int build_exec(DistPlan& dp, int n, int layout, const PlanParams& pp, const DistParams& d) {
  int max_rows = 0, max_cols = 0;
  build_dist_plan(n, pp, d, dp.ops, &dp.send_elems, &max_rows, &max_cols);
  // packed rows are padded to a multiple of 8 so packed blocks stay TMA-aligned
  const size_t nops = dp.ops.size();
  dp.upd.resize(nops);
  dp.d_rows.assign(nops, nullptr);
  dp.rows_pad.assign(nops, 0);
  int64_t send_elems = 0;
  int cur_pad = 0, cur_cols = 0;
  cudaError_t e;
  for (size_t i = 0; i < nops; ++i) {
    PlanOp& op = dp.ops[i];
    if (op.kind == OP_PACK || op.kind == OP_UNPACK) {
      // op.c_i = lo, op.m = hi - lo, op.k = ncols, op.n = rows_max (unpadded)
      int rows_max = 0;
      for (int s = 0; s < d.nranks; ++s) {
        const int c = dist_owned_rows(op.c_i, op.c_i + op.m, s, d);
        rows_max = c > rows_max ? c : rows_max;
      }
      const int pad = (rows_max + 7) / 8 * 8;
      std::vector<int> tab = row_table(op.c_i, op.c_i + op.m, d, pad);
      if ((e = cudaMalloc(&dp.d_rows[i], tab.size() * sizeof(int))) != cudaSuccess) return cuda_fail(e, "row table");
      if ((e = cudaMemcpy(dp.d_rows[i], tab.data(), tab.size() * sizeof(int), cudaMemcpyHostToDevice)) != cudaSuccess)
        return cuda_fail(e, "row table");
      dp.rows_pad[i] = pad;
      cur_pad = pad;
      cur_cols = op.k;
      const int64_t el = (int64_t)pad * op.k;
      send_elems = el > send_elems ? el : send_elems;
    } else if (op.kind == OP_ALLGATHER) {
      dp.rows_pad[i] = cur_pad;
      op.k = cur_cols;
    } else {
      dp.rows_pad[i] = cur_pad;  // geometry of BUF_SEND for TRSM/GEMM on packed rows
    }
  }
  dp.send_elems = send_elems;
  if (send_elems > 0) {
    if ((e = cudaMalloc(&dp.recv, send_elems * d.nranks * sizeof(double))) != cudaSuccess)
      return cuda_fail(e, "recv buffer");
  }
  return 0;
}

}  // namespace

void destroy_dist_plan(DistPlan* p) { delete p; }

// This rank's packed chunk of op i: its slot inside the receive buffer, so the
// all-gather runs in place (NCCL: sendbuff == recvbuff + rank * count) and the
// own rows are never copied send -> recv.
static inline double* send_ptr(const DistPlan& dp, size_t i, int rank, int ncols) {
  return dp.recv + (size_t)rank * (size_t)dp.rows_pad[i] * (size_t)ncols;
}

// Pointer + ld of an op operand (matrix or the current packed send chunk).
static inline double* operand(int buf, int ri, int ci, int layout, double* A, int64_t lda, double* send, int rows_pad,
                              int ncols, int64_t* ld) {
  if (buf == BUF_A) {
    *ld = lda;
    return A + lv_off(layout, ri, ci, lda);
  }
  *ld = layout == kLayoutN ? rows_pad : ncols;
  return send + lv_off(layout, ri, ci, *ld);
}

// Enqueue rank-local work of ops [beg, end) (no collectives) on st.
static int run_local(DistPlan& dp, size_t beg, size_t end, int layout, double* A, int64_t lda, int* d_info,
                     const DistParams& d, int rank, cudaStream_t st, std::vector<int>& ncols_of) {
  cudaError_t e = cudaSuccess;
  for (size_t i = beg; i < end; ++i) {
    const PlanOp& op = dp.ops[i];
    const int pad = dp.rows_pad[i], nc = ncols_of[i];
    int64_t ldc = 0, lda_ = 0, ldb = 0;
    switch (op.kind) {
      case OP_POTF2:
        e = launch_potf2(A + lv_off(layout, op.c_i, op.c_j, lda), lda, layout, op.n, d_info, op.info_base, st);
        break;
      case OP_TRSM: {
        double* B = operand(op.c_buf, op.c_i, op.c_j, layout, A, lda, send_ptr(dp, i, rank, nc), pad, nc, &ldc);
        e = launch_trsm_any(A + lv_off(layout, op.a_i, op.a_j, lda), lda, B, ldc, layout, op.m, op.k, d_info, st);
        break;
      }
      case OP_GEMM:
      case OP_SYRK: {
        UpdateOp& u = dp.upd[i];
        const bool syrk = op.kind == OP_SYRK;
        double* sp = send_ptr(dp, i, rank, nc);
        double* C = operand(op.c_buf, op.c_i, op.c_j, layout, A, lda, sp, pad, nc, &ldc);
        const double* Ap = operand(op.a_buf, op.a_i, op.a_j, layout, A, lda, sp, pad, nc, &lda_);
        const double* Bp = operand(op.b_buf, op.b_i, op.b_j, layout, A, lda, sp, pad, nc, &ldb);
        init_update(u, C, ldc, layout, Ap, lda_, layout, Bp, ldb, layout, syrk ? op.n : op.m, op.n, op.k, -1.0,
                    syrk ? 1 : 0);
        u.args.d_info = d_info;
        e = launch_update(u, st);
        break;
      }
      case OP_PACK: {
        const int64_t total = (int64_t)pad * op.k;
        k_pack_rows<<<grid_for(total), 256, 0, st>>>(A, lda, layout, dp.d_rows[i] + (size_t)rank * pad, pad, op.c_j,
                                                     op.k, send_ptr(dp, i, rank, op.k), d_info);
        e = cudaGetLastError();
        break;
      }
      case OP_UNPACK: {
        const int64_t total = (int64_t)pad * op.k * d.nranks;
        k_unpack_rows<<<grid_for(total), 256, 0, st>>>(A, lda, layout, dp.d_rows[i], pad, d.nranks, op.c_j, op.k,
                                                       dp.recv, d_info);
        e = cudaGetLastError();
        break;
      }
      default:
        break;
    }
    if (e != cudaSuccess) return cuda_fail(e, "dist launch");
  }
  return 0;
}

// One op of the graph executor: kernels as run_local (update descriptors built
// once, with split-K), the all-gather as an NCCL call on the capturing stream.
static cudaError_t launch_dist_op(DistPlan& dp, size_t i, int layout, double* A, int64_t lda, int* d_info,
                                  const DistParams& d, relapack_comm* comm, cudaStream_t st) {
  const PlanOp& op = dp.ops[i];
  const int pad = dp.rows_pad[i], nc = dp.ncols[i];
  int64_t ldc = 0;
  switch (op.kind) {
    case OP_POTF2:
      return launch_potf2(A + lv_off(layout, op.c_i, op.c_j, lda), lda, layout, op.n, d_info, op.info_base, st);
    case OP_TRSM: {
      double* B = operand(op.c_buf, op.c_i, op.c_j, layout, A, lda, send_ptr(dp, i, d.rank, nc), pad, nc, &ldc);
      return launch_trsm_any(A + lv_off(layout, op.a_i, op.a_j, lda), lda, B, ldc, layout, op.m, op.k, d_info, st);
    }
    case OP_GEMM:
    case OP_SYRK:
      return launch_update(dp.upd[i], st);
    case OP_PACK: {
      const int64_t total = (int64_t)pad * op.k;
      k_pack_rows<<<grid_for(total), 256, 0, st>>>(A, lda, layout, dp.d_rows[i] + (size_t)d.rank * pad, pad, op.c_j,
                                                   op.k, send_ptr(dp, i, d.rank, op.k), d_info);
      return cudaGetLastError();
    }
    case OP_UNPACK: {
      const int64_t total = (int64_t)pad * op.k * d.nranks;
      k_unpack_rows<<<grid_for(total), 256, 0, st>>>(A, lda, layout, dp.d_rows[i], pad, d.nranks, op.c_j, op.k,
                                                     dp.recv, d_info);
      return cudaGetLastError();
    }
    case OP_ALLGATHER: {
      const size_t cnt = (size_t)pad * op.k;
      // in place: this rank's chunk already sits at recv + rank * cnt
      const ncclResult_t r = nccl().AllGather(send_ptr(dp, i, d.rank, op.k), dp.recv, cnt, ncclDouble_, comm->nccl, st);
      if (r != 0) {
        set_error(std::string("ncclAllGather: ") + (nccl().GetErrorString ? nccl().GetErrorString(r) : "error"));
        return cudaErrorUnknown;
      }
      return cudaSuccess;
    }
    default:
      return cudaErrorInvalidValue;
  }
}

// Column count of the current packed chunk for every op (TRSM/GEMM on BUF_SEND).
static std::vector<int> chunk_cols(const DistPlan& dp) {
  std::vector<int> nc(dp.ops.size(), 0);
  int cur = 0;
  for (size_t i = 0; i < dp.ops.size(); ++i) {
    if (dp.ops[i].kind == OP_PACK || dp.ops[i].kind == OP_UNPACK) cur = dp.ops[i].k;
    nc[i] = cur;
  }
  return nc;
}

}  // namespace relapack

using namespace relapack;

static int parse_uplo(const char* uplo, int* layout) {
  if (!uplo) return -1;
  if (*uplo == 'L' || *uplo == 'l') {
    *layout = kLayoutN;
    return 0;
  }
  if (*uplo == 'U' || *uplo == 'u') {
    *layout = kLayoutT;
    return 0;
  }
  return -1;
}

extern "C" {

int relapack_comm_unique_id(char uid[128]) {
  NcclApi& api = nccl();
  if (!api.ok()) {
    set_error("relapack_comm_unique_id: libnccl.so.2 not loadable (set RELAPACK_NCCL_LIB)");
    return -1000;
  }
  ncclUniqueId id;
  ncclResult_t r = api.GetUniqueId(&id);
  if (r != 0) {
    set_error(std::string("ncclGetUniqueId: ") + (api.GetErrorString ? api.GetErrorString(r) : "error"));
    return -1000 - r;
  }
  memcpy(uid, id.internal, 128);
  return 0;
}

int relapack_comm_init(relapack_comm_t** comm, const char uid[128], int nranks, int rank, int device) {
  if (!comm || nranks < 1 || rank < 0 || rank >= nranks) return -1;
  auto* c = new relapack_comm();
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete c;
    return cuda_fail(e, "comm init");
  }
  if ((e = cudaStreamCreateWithFlags(&c->capture, cudaStreamNonBlocking)) != cudaSuccess) {
    delete c;
    return cuda_fail(e, "comm init");
  }
  {  // the communicator exists at every world size (world 1 included: the same path)
    NcclApi& api = nccl();
    if (!api.ok()) {
      set_error("relapack_comm_init: libnccl.so.2 not loadable (set RELAPACK_NCCL_LIB)");
      delete c;
      return -1000;
    }
    ncclUniqueId id;
    memcpy(id.internal, uid, 128);
    ncclResult_t r = api.CommInitRank(&c->nccl, nranks, id, rank);
    if (r != 0) {
      set_error(std::string("ncclCommInitRank: ") + (api.GetErrorString ? api.GetErrorString(r) : "error"));
      delete c;
      return -1000 - r;
    }
  }
  *comm = c;
  return 0;
}

void relapack_comm_destroy(relapack_comm_t* comm) {
  if (!comm) return;
  if (comm->plan) destroy_dist_plan(comm->plan);
  if (comm->d_info) cudaFree(comm->d_info);
  if (comm->nccl && nccl().ok()) (comm->aborted ? 0 : nccl().CommDestroy(comm->nccl));
  if (comm->stream) cudaStreamDestroy(comm->stream);
  if (comm->capture) cudaStreamDestroy(comm->capture);
  delete comm;
}

void relapack_dpotrf_dist(const char* uplo, const int* n_, double* A, const int* lda_, int nb, int dist_min,
                          relapack_comm_t* comm, int* info) {
  if (!info) return;
  int layout = 0;
  if (parse_uplo(uplo, &layout) != 0) {
    *info = -1;
    return;
  }
  if (!n_ || *n_ < 0) {
    *info = -2;
    return;
  }
  const int n = *n_;
  if (n > 0 && !A) {
    *info = -3;
    return;
  }
  if (!lda_ || *lda_ < (n > 1 ? n : 1)) {
    *info = -4;
    return;
  }
  if (!comm || nb < 64 || nb % 64 != 0 || dist_min < 1) {
    *info = -5;
    return;
  }
  if (n == 0) {
    *info = 0;
    return;
  }
  const int64_t lda = *lda_;
  DistParams d;
  d.nranks = comm->nranks;
  d.rank = comm->rank;
  d.nb = nb;
  d.dist_min = dist_min;
  PlanParams pp = current_params();
  cudaStream_t st = current_stream_or(comm->stream);
  cudaError_t e;
  if (!comm->d_info && (e = cudaMalloc(&comm->d_info, 2 * sizeof(int))) != cudaSuccess) {
    *info = cuda_fail(e, "dist info");
    return;
  }
  int* d_info = comm->d_info;
  if ((e = configure_kernels()) != cudaSuccess) {
    *info = cuda_fail(e, "configure");
    return;
  }
  if (comm->aborted) {
    set_error("relapack_dpotrf_dist: the communicator was aborted after an earlier NCCL failure / timeout");
    *info = -1000;
    return;
  }
  char kb[256];
  snprintf(kb, sizeof(kb), "n%d ld%lld l%d nb%d dm%d c%d T%d tb%d la%d ld%d b21%d A%p", n, (long long)lda, layout,
           nb, dist_min, pp.crossover, pp.split_tile, pp.trsm_base, (int)pp.lookahead, pp.lookahead_depth,
           pp.b21_chunks, (void*)A);
  if (!comm->plan || comm->key != kb) {
    if (comm->plan) destroy_dist_plan(comm->plan);
    comm->plan = new DistPlan();
    comm->key = kb;
    DistPlan& dp = *comm->plan;
    int r0 = build_exec(dp, n, layout, pp, d);
    cudaGraph_t g = nullptr;
    if (r0 == 0) {
      dp.ncols = chunk_cols(dp);
      // update descriptors (the packed send buffer or the matrix), split-K
      // slots from the DAG's ancestor sets, then one capture of the whole plan
      dp.upd.assign(dp.ops.size(), UpdateOp{});
      for (size_t i = 0; i < dp.ops.size(); ++i) {
        const PlanOp& op = dp.ops[i];
        if (op.kind != OP_GEMM && op.kind != OP_SYRK) continue;
        int64_t ldc = 0, lda_ = 0, ldb = 0;
        const int pad = dp.rows_pad[i], nc = dp.ncols[i];
        double* sp = send_ptr(dp, i, d.rank, nc);
        double* C = operand(op.c_buf, op.c_i, op.c_j, layout, A, lda, sp, pad, nc, &ldc);
        const double* Ap = operand(op.a_buf, op.a_i, op.a_j, layout, A, lda, sp, pad, nc, &lda_);
        const double* Bp = operand(op.b_buf, op.b_i, op.b_j, layout, A, lda, sp, pad, nc, &ldb);
        const bool syrk = op.kind == OP_SYRK;
        init_update(dp.upd[i], C, ldc, layout, Ap, lda_, layout, Bp, ldb, layout, syrk ? op.n : op.m, op.n, op.k,
                    -1.0, syrk ? 1 : 0);
        dp.upd[i].args.d_info = d_info;
      }
      std::vector<std::vector<int>> deps;
      std::vector<uint64_t> anc;
      compute_deps(dp.ops, deps, &anc);
      if ((e = setup_splitk_ops(dp.ops, dp.upd, &anc, &dp.splitk_ws, &dp.splitk_cnt, &dp.cnt_bytes)) != cudaSuccess)
        r0 = cuda_fail(e, "dist split-K");
      if (r0 == 0 && (e = cudaStreamBeginCapture(comm->capture, cudaStreamCaptureModeThreadLocal)) != cudaSuccess)
        r0 = cuda_fail(e, "dist capture");
      if (r0 == 0) {
        cudaError_t er = cudaMemsetAsync(d_info, 0, 2 * sizeof(int), comm->capture);
        if (er == cudaSuccess && dp.splitk_cnt) er = cudaMemsetAsync(dp.splitk_cnt, 0, dp.cnt_bytes, comm->capture);
        std::vector<cudaGraphNode_t> nodes;
        std::vector<char> cls;
        if (er == cudaSuccess)
          er = capture_plan_dag(
              dp.ops, deps, comm->capture,
              [&](size_t i, cudaStream_t s2) { return launch_dist_op(dp, i, layout, A, lda, d_info, d, comm, s2); },
              nodes, cls);
        // info identical on every rank (every rank computes the same replicated
        // leaves; this all-reduce(max) is the guard the ABI promises)
        if (er == cudaSuccess &&
            nccl().AllReduce(d_info, d_info + 1, 1, ncclInt32_, ncclMax_, comm->nccl, comm->capture) != 0)
          er = cudaErrorUnknown;
        if (er == cudaSuccess)
          er = cudaMemcpyAsync(d_info, d_info + 1, sizeof(int), cudaMemcpyDeviceToDevice, comm->capture);
        e = cudaStreamEndCapture(comm->capture, &g);
        if (er == cudaSuccess && e == cudaSuccess && (e = set_node_priorities(nodes, cls)) == cudaSuccess)
          e = cudaGraphInstantiateWithFlags(&dp.exec, g, cudaGraphInstantiateFlagUseNodePriority);
        if (er != cudaSuccess) r0 = cuda_fail(er, "dist capture (launch)");
        else if (e != cudaSuccess) r0 = cuda_fail(e, "dist graph");
      }
      if (g) cudaGraphDestroy(g);
    }
    if (r0 != 0) {
      destroy_dist_plan(comm->plan);
      comm->plan = nullptr;
      comm->key.clear();
      *info = r0;
      return;
    }
  }
  DistPlan& dp = *comm->plan;
  if ((e = cudaGraphLaunch(dp.exec, st)) != cudaSuccess) {
    *info = cuda_fail(e, "dist launch");
    return;
  }
  // wait, polling NCCL's asynchronous error state and a timeout (SURVEY §5:
  // a peer that died must not hang the caller forever)
  const char* tv = getenv("RELAPACK_DIST_TIMEOUT_S");
  const double timeout_s = tv ? atof(tv) : 600.0;
  const auto t0 = std::chrono::steady_clock::now();
  int r = 0;
  for (;;) {
    const cudaError_t q = cudaStreamQuery(st);
    if (q == cudaSuccess) break;
    if (q != cudaErrorNotReady) {
      r = cuda_fail(q, "dist wait");
      break;
    }
    ncclResult_t ae = 0;
    if (nccl().CommGetAsyncError && nccl().CommGetAsyncError(comm->nccl, &ae) == 0 && ae != 0 && ae != 7 /*inProgress*/) {
      set_error(std::string("NCCL asynchronous error: ") + (nccl().GetErrorString ? nccl().GetErrorString(ae) : "?"));
      r = -1000 - (int)ae;
    }
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (r == 0 && el > timeout_s) {
      set_error("relapack_dpotrf_dist: timed out waiting for the collectives (RELAPACK_DIST_TIMEOUT_S)");
      r = -1999;
    }
    if (r != 0) {
      if (nccl().CommAbort) nccl().CommAbort(comm->nccl);
      comm->aborted = true;
      break;
    }
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
  int h = 0;
  if (r == 0) {
    if ((e = cudaMemcpyAsync(&h, d_info, sizeof(int), cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (e = cudaStreamSynchronize(st)) != cudaSuccess)
      r = cuda_fail(e, "dist sync");
  }
  if (r != 0) {
    *info = r;
    return;
  }
  *info = h;
}

// Test hook: P virtual ranks on the current GPU, rank s owning the matrix
// buffer A_ranks[s] (each a full lda x n copy).  Collectives are emulated with
// device copies between the ranks' buffers; ranks run one after another
// between collectives (no kernel waits on another).  infos[s] = rank s's info.
int relapack_dpotrf_dist_loopback(const char* uplo, int n, double* const* A_ranks, int lda, int nb, int dist_min,
                                  int nranks, int* infos) {
  int layout = 0;
  if (parse_uplo(uplo, &layout) != 0) return -1;
  if (n < 0) return -2;
  if (lda < (n > 1 ? n : 1)) return -4;
  if (nranks < 1 || nb < 64 || nb % 64 != 0 || !A_ranks || !infos) return -5;
  if (n == 0) {
    for (int s = 0; s < nranks; ++s) infos[s] = 0;
    return 0;
  }
  PlanParams pp = current_params();
  cudaError_t e;
  if ((e = configure_kernels()) != cudaSuccess) return cuda_fail(e, "configure");
  cudaStream_t st = nullptr;
  if ((e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)) != cudaSuccess) return cuda_fail(e, "stream");
  int* d_info = nullptr;
  if ((e = cudaMalloc(&d_info, nranks * sizeof(int))) != cudaSuccess) return cuda_fail(e, "info");
  cudaMemsetAsync(d_info, 0, nranks * sizeof(int), st);
  std::vector<std::unique_ptr<DistPlan>> plans(nranks);
  std::vector<std::vector<int>> ncs(nranks);
  int r = 0;
  for (int s = 0; s < nranks && r == 0; ++s) {
    DistParams d;
    d.nranks = nranks;
    d.rank = s;
    d.nb = nb;
    d.dist_min = dist_min;
    plans[s].reset(new DistPlan());
    r = build_exec(*plans[s], n, layout, pp, d);
    ncs[s] = chunk_cols(*plans[s]);
  }
  std::vector<size_t> beg(nranks, 0);
  while (r == 0) {
    // run every rank up to its next collective
    std::vector<size_t> stop(nranks);
    bool any = false;
    for (int s = 0; s < nranks && r == 0; ++s) {
      DistParams d;
      d.nranks = nranks;
      d.rank = s;
      d.nb = nb;
      d.dist_min = dist_min;
      size_t i = beg[s];
      while (i < plans[s]->ops.size() && plans[s]->ops[i].kind != OP_ALLGATHER) ++i;
      stop[s] = i;
      r = run_local(*plans[s], beg[s], i, layout, A_ranks[s], lda, d_info + s, d, s, st, ncs[s]);
      if (i < plans[s]->ops.size()) any = true;
    }
    if (r != 0 || !any) break;
    // emulate the all-gather: recv_d[s] = send_s for every pair
    for (int dst = 0; dst < nranks; ++dst) {
      const size_t i = stop[dst];
      const size_t cnt = (size_t)plans[dst]->rows_pad[i] * plans[dst]->ops[i].k;
      for (int src = 0; src < nranks; ++src)
        if (src != dst)  // in place: the own chunk is already there
          cudaMemcpyAsync(plans[dst]->recv + (size_t)src * cnt, plans[src]->recv + (size_t)src * cnt,
                          cnt * sizeof(double), cudaMemcpyDeviceToDevice, st);
    }
    for (int s = 0; s < nranks; ++s) beg[s] = stop[s] + 1;
  }
  if (r == 0) {
    if ((e = cudaMemcpyAsync(infos, d_info, nranks * sizeof(int), cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (e = cudaStreamSynchronize(st)) != cudaSuccess)
      r = cuda_fail(e, "loopback sync");
  }
  cudaStreamSynchronize(st);
  plans.clear();
  cudaFree(d_info);
  cudaStreamDestroy(st);
  return r;
}

// Host-only: this rank's distributed schedule as 16 int64 per op:
// kind, level, c_i, c_j, a_i, a_j, b_i, b_j, m, n, k, info_base, c_buf, a_buf,
// b_buf, 0.  Returns the op count (or -1 on bad arguments).
int relapack_dist_schedule(int n, int c, int T, int nb, int dist_min, int rank, int nranks, int64_t* out, int max_ops) {
  if (n < 0 || c < 1 || T < 1 || nb < 1 || nranks < 1 || rank < 0 || rank >= nranks) return -1;
  PlanParams p;
  p.crossover = c;
  p.split_tile = T;
  p.trsm_base = trsm_base_cols();
  DistParams d;
  d.nranks = nranks;
  d.rank = rank;
  d.nb = nb;
  d.dist_min = dist_min;
  std::vector<PlanOp> ops;
  int64_t se = 0;
  int mr = 0, mc = 0;
  build_dist_plan(n, p, d, ops, &se, &mr, &mc);
  const int cnt = (int)ops.size();
  for (int i = 0; i < cnt && i < max_ops && out; ++i) {
    const PlanOp& o = ops[i];
    int64_t* w = out + 16 * i;
    w[0] = o.kind; w[1] = o.level; w[2] = o.c_i; w[3] = o.c_j; w[4] = o.a_i; w[5] = o.a_j; w[6] = o.b_i;
    w[7] = o.b_j; w[8] = o.m; w[9] = o.n; w[10] = o.k; w[11] = o.info_base; w[12] = o.c_buf; w[13] = o.a_buf;
    w[14] = o.b_buf; w[15] = 0;
  }
  return cnt;
}

}  // extern "C"
