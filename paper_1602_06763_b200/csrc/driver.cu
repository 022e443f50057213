// driver.cu — C-ABI entry points (include/relapack.h) and the host recursion
// driver: validates LAPACK arguments, maps uplo 'U' onto the L-view (layout
// T), turns the plan (plan.h) into kernel launches, captures them once per
// (device, A, n, lda, uplo, info pointer, knobs) into a CUDA graph and replays
// it.  Every step of the factorization runs in the kernels of update.cu,
// potf2.cu and trsm.cu; there is no CPU fallback.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <list>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/relapack.h"
#include "common.cuh"
#include "driver_internal.h"
#include "kernels.h"
#include "plan.h"

namespace relapack {

// ------------------------------------------------------------------ errors
static thread_local std::string g_last_error;
static std::mutex g_err_mu;
static std::string g_last_error_global;

void set_error(const std::string& s) {
  g_last_error = s;
  std::lock_guard<std::mutex> lk(g_err_mu);
  g_last_error_global = s;
}

int cuda_fail(cudaError_t e, const char* what) {
  set_error(std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
  return -1000 - (int)e;
}

thread_local TraceRec* g_launch_trace = nullptr;

// ------------------------------------------------------------------ knobs
static std::atomic<int> g_crossover{-1}, g_split_tile{-1}, g_graphs{-1};
// relapack_set_stream is per calling thread: a thread's set_stream + call pair
// is never redirected by another thread's set_stream (the Python binding calls
// them back to back, releasing the GIL in between)
static thread_local cudaStream_t g_stream = nullptr;
static thread_local int g_stream_set = 0;

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  if (!v || !*v) return dflt;
  return atoi(v);
}

cudaStream_t current_stream_or(cudaStream_t fallback) { return g_stream_set ? g_stream : fallback; }

// Column width of the TRSM base case (RELAPACK_TRSM_BASE, 64 .. kTrsmFusedMax;
// default 128: the whole L of the base fits shared memory next to the row
// slab, staged once — measured best at n = 4096 and 16384, profiles/).
int trsm_base_cols() {
  int b = env_int("RELAPACK_TRSM_BASE", 128);
  return b < 64 ? 64 : (b > kTrsmFusedMax ? kTrsmFusedMax : b);
}

PlanParams current_params() {
  PlanParams p;
  int c = g_crossover.load();
  if (c < 0) c = env_int("RELAPACK_CROSSOVER", kCrossoverDefault);
  int t = g_split_tile.load();
  if (t < 0) t = env_int("RELAPACK_SPLIT_TILE", 64);
  if (c < 16 || c > kPotf2Max) c = kCrossoverDefault;
  if (t != 8 && t != 16 && t != 32 && t != 64 && t != 128) t = 64;
  p.crossover = c;
  p.split_tile = t;
  p.trsm_base = trsm_base_cols();
  p.lookahead = env_int("RELAPACK_LOOKAHEAD", 1) != 0;
  p.trsm_rows = env_int("RELAPACK_TRSM_ROWS", 0);
  p.lookahead_depth = env_int("RELAPACK_LOOKAHEAD_DEPTH", 1);
  p.defer_b21 = env_int("RELAPACK_DEFER_B21", 1) != 0;
  p.b21_chunks = env_int("RELAPACK_B21_CHUNKS", 1);
  return p;
}

// DAG capture: the graph's edges are the plan's footprint dependencies
// (compute_deps) instead of the serial launch order.
static bool dag_enabled() { return env_int("RELAPACK_DAG", 1) != 0; }
// CTA cap of the deferred (lookahead) trailing updates: leaves SMs to the
// next panel's chain; 0 = uncapped
static int bulk_ctas() { return env_int("RELAPACK_BULK_CTAS", 132); }
static double bulk_min_flops() { return 1e9 * env_int("RELAPACK_BULK_MIN_GF", 16); }
// CTA cap of the non-deferred updates (0 = uncapped)
static int upd_ctas() { return env_int("RELAPACK_UPD_CTAS", 0); }
// deferred (lookahead) updates at low graph-node priority (RELAPACK_DEFER_LOW=0: equal)
static bool defer_low_priority() { return env_int("RELAPACK_DEFER_LOW", 1) != 0; }

static bool splitk_enabled() { return env_int("RELAPACK_SPLITK", 1) != 0; }
// programmatic dependent launch on the plan DAG's kernel-to-kernel edges
// (1: every edge between plan kernels, 2: edges into base cases and TRSMs,
// 3 (default): 2 + edges into the non-deferred SYRKs of the chain; 0: off;
// n = 4096 2.186 -> 2.130 ms, n = 16384 47.26 -> 47.01 ms, exp_pdl.sh)
static int pdl_mode() { return env_int("RELAPACK_PDL", 3); }

// RELAPACK_TRACE=1: every kernel of the plan records its first-CTA start and
// last-CTA end (tools/trace_timeline.py reads them with relapack_trace_read).
static bool trace_enabled() { return env_int("RELAPACK_TRACE", 0) != 0; }
static std::mutex g_trace_mu;
static const void* g_trace_plan = nullptr;  // the Plan whose trace relapack_trace_read returns (cleared when it dies)

static bool graphs_enabled() {
  int g = g_graphs.load();
  if (g < 0) g = env_int("RELAPACK_GRAPH", 1);
  return g != 0;
}

// ------------------------------------------------------------------ per-device state
struct Plan {
  std::vector<PlanOp> ops;
  const double* host = nullptr;  // host-matrix path: the caller's pinned matrix (OP_H2D / OP_D2H ops)
  int64_t hld = 0;
  // split copies: the graph holds an external event wait (H2D) / record (D2H)
  // node per copy block; the copies themselves run on two library streams, one
  // per link direction (memcpy nodes inside one graph were serialised: 38 ms
  // for n = 16384 against 21.6 ms for both directions on two streams)
  bool split_copies = false;
  std::vector<cudaEvent_t> ev;  // per op (copy ops only)
  // copy ops in issue order: H2D by first use, D2H by last write (no block
  // waits behind one that is needed later / ready later on its stream)
  std::vector<int> h2d_order, d2h_order;
  std::vector<UpdateOp> upd;  // parallel to ops (only GEMM/SYRK entries used)
  cudaGraphExec_t exec = nullptr;
  TraceRec* d_trace = nullptr;  // RELAPACK_TRACE=1: per-op kernel start/end (globaltimer)
  double* splitk_ws = nullptr;  // split-K partial tiles, one slot per concurrently runnable update
  int* splitk_cnt = nullptr;    // per-tile arrival counters (self-resetting; zeroed at every run start)
  size_t cnt_bytes = 0;
  // Pointer-independent graph (RELAPACK_REBASE, default on): the kernels get
  // byte offsets from the matrix base and a d_info tagged to d_state; the
  // graph's first node (begin_node: k_plan_begin) writes the run's base into
  // d_state and rebases the TMA descriptors d_maps (tensormap.replace), its
  // last node (end_node: k_plan_end) copies the info word out.  A call with
  // another matrix / info pointer updates only these two nodes' parameters.
  bool rebased = false;
  PlanState* d_state = nullptr;
  CUtensorMap* d_maps = nullptr;
  long long* d_map_off = nullptr;  // byte offset of each descriptor's global address from the base
  int nmaps = 0;
  cudaGraph_t graph = nullptr;     // kept for cudaGraphExecKernelNodeSetParams
  cudaGraphNode_t begin_node = nullptr, end_node = nullptr;
  const double* cur_A = nullptr;   // what the begin / end nodes currently hold
  int* cur_info = nullptr;
  ~Plan() {
    {
      std::lock_guard<std::mutex> tl(g_trace_mu);
      if (g_trace_plan == this) g_trace_plan = nullptr;
    }
    if (exec) cudaGraphExecDestroy(exec);
    if (d_trace) cudaFree(d_trace);
    for (cudaEvent_t e : ev)
      if (e) cudaEventDestroy(e);
    if (splitk_ws) cudaFree(splitk_ws);
    if (splitk_cnt) cudaFree(splitk_cnt);
    if (graph) cudaGraphDestroy(graph);
    if (d_state) cudaFree(d_state);
    if (d_maps) cudaFree(d_maps);
    if (d_map_off) cudaFree(d_map_off);
  }
};

__global__ void k_plan_begin(PlanState* ps, unsigned long long base, CUtensorMap* maps, const long long* off,
                             int nmaps) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) {
    ps->info = 0;
    ps->base = base;
  }
  if (i < nmaps)
    asm volatile("tensormap.replace.tile.global_address.global.b1024.b64 [%0], %1;" ::"l"(maps + i),
                 "l"(base + (unsigned long long)off[i])
                 : "memory");
  asm volatile("fence.proxy.tensormap::generic.release.gpu;" ::: "memory");
}

__global__ void k_plan_end(const PlanState* ps, int* info) { *info = ps->info; }

static int begin_grid(int nmaps) { return (nmaps + 255) / 256 > 0 ? (nmaps + 255) / 256 : 1; }

static cudaError_t launch_plan_begin(const Plan& pl, const double* A, cudaStream_t st) {
  k_plan_begin<<<begin_grid(pl.nmaps), 256, 0, st>>>(pl.d_state, (unsigned long long)reinterpret_cast<uintptr_t>(A),
                                                     pl.d_maps, pl.d_map_off, pl.nmaps);
  return cudaGetLastError();
}

// Point the instantiated graph at another matrix / info word (two nodes).
static cudaError_t retarget(Plan& pl, const double* A, int* d_info) {
  cudaError_t e;
  if (A != pl.cur_A) {
    PlanState* ps = pl.d_state;
    unsigned long long base = (unsigned long long)reinterpret_cast<uintptr_t>(A);
    CUtensorMap* maps = pl.d_maps;
    const long long* off = pl.d_map_off;
    int nm = pl.nmaps;
    void* args[] = {&ps, &base, &maps, &off, &nm};
    cudaKernelNodeParams kp{};
    kp.func = reinterpret_cast<void*>(k_plan_begin);
    kp.gridDim = dim3(begin_grid(pl.nmaps));
    kp.blockDim = dim3(256);
    kp.kernelParams = args;
    if ((e = cudaGraphExecKernelNodeSetParams(pl.exec, pl.begin_node, &kp)) != cudaSuccess) return e;
    pl.cur_A = A;
  }
  if (d_info != pl.cur_info) {
    const PlanState* ps = pl.d_state;
    int* info = d_info;
    void* args[] = {&ps, &info};
    cudaKernelNodeParams kp{};
    kp.func = reinterpret_cast<void*>(k_plan_end);
    kp.gridDim = dim3(1);
    kp.blockDim = dim3(1);
    kp.kernelParams = args;
    if ((e = cudaGraphExecKernelNodeSetParams(pl.exec, pl.end_node, &kp)) != cudaSuccess) return e;
    pl.cur_info = d_info;
  }
  return cudaSuccess;
}

// (A, n, ld, layout, d_info, host, hld, knob signature): every knob that shapes
// the plan, its launches or the capture is part of the key (knob_signature)
using PlanKey = std::tuple<uintptr_t, int, int64_t, int, uintptr_t, uintptr_t, int64_t, std::string>;

struct DeviceState {
  std::mutex mu;          // guards the plan cache
  std::mutex sync_mu;     // serialises the synchronous entry point (shared info / staging)
  bool configured = false;
  cudaStream_t capture = nullptr;
  int* d_info = nullptr;  // library-owned info scalar for the synchronous API
  int* h_info = nullptr;  // pinned
  double* stage = nullptr;  // staging buffer for host matrices
  double* bounce = nullptr;  // pinned 256 x 256 bounce for the pageable path's diagonal blocks
  size_t stage_elems = 0;
  cudaStream_t h2d = nullptr, d2h = nullptr;  // split-copy streams (one per link direction)
  cudaEvent_t ev_start = nullptr, ev_done = nullptr;
  std::list<std::pair<PlanKey, std::unique_ptr<Plan>>> lru;
  std::map<PlanKey, std::list<std::pair<PlanKey, std::unique_ptr<Plan>>>::iterator> index;
};

static std::mutex g_dev_mu;
static DeviceState* g_dev[kMaxDevices] = {};

DeviceState* device_state(int dev) {
  std::lock_guard<std::mutex> lk(g_dev_mu);
  if (!g_dev[dev]) g_dev[dev] = new DeviceState();
  return g_dev[dev];
}

static cudaError_t ensure_device(DeviceState* ds) {
  if (ds->configured) return cudaSuccess;
  cudaError_t e;
  if ((e = cudaStreamCreateWithFlags(&ds->capture, cudaStreamNonBlocking)) != cudaSuccess) return e;
  if ((e = cudaMalloc(&ds->d_info, sizeof(int))) != cudaSuccess) return e;
  if ((e = cudaHostAlloc(&ds->h_info, sizeof(int), cudaHostAllocDefault)) != cudaSuccess) return e;
  if ((e = configure_kernels()) != cudaSuccess) return e;
  if ((e = cudaStreamCreateWithFlags(&ds->h2d, cudaStreamNonBlocking)) != cudaSuccess) return e;
  if ((e = cudaStreamCreateWithFlags(&ds->d2h, cudaStreamNonBlocking)) != cudaSuccess) return e;
  if ((e = cudaEventCreateWithFlags(&ds->ev_start, cudaEventDisableTiming)) != cudaSuccess) return e;
  if ((e = cudaEventCreateWithFlags(&ds->ev_done, cudaEventDisableTiming)) != cudaSuccess) return e;
  ds->configured = true;
  return cudaSuccess;
}

// ------------------------------------------------------------------ executor
__global__ void k_set_int(int* p, int v) { *p = v; }

cudaError_t launch_set_int(int* p, int v, cudaStream_t st) {
  k_set_int<<<1, 1, 0, st>>>(p, v);
  return cudaGetLastError();
}

static void fill_update(UpdateOp& u, const PlanOp& op, double* A, int64_t ld, int layout, const int* d_info) {
  const bool syrk = op.kind == OP_SYRK;
  init_update(u, A + lv_off(layout, op.c_i, op.c_j, ld), ld, layout, A + lv_off(layout, op.a_i, op.a_j, ld), ld, layout,
              A + lv_off(layout, op.b_i, op.b_j, ld), ld, layout, syrk ? op.n : op.m, op.n, op.k, -1.0, syrk ? 1 : 0);
  u.args.d_info = d_info;
}

// Enable split-K on the plan's small-grid / long-K updates and give each a
// workspace slot.  Two split-K updates share a slot only if one is an
// ancestor of the other in the dependency DAG (`anc`, or the serial order
// when anc is null), so concurrently runnable updates never share partials.
cudaError_t setup_splitk_ops(const std::vector<PlanOp>& ops, std::vector<UpdateOp>& upd,
                             const std::vector<uint64_t>* anc, double** ws_out, int** cnt_out, size_t* cnt_bytes) {
  const size_t nops = ops.size(), words = (nops + 63) / 64;
  int64_t ws = 0;
  int cnt = 0;
  std::vector<int> slot_last;  // last op assigned to each slot
  std::vector<int> slot_of(nops, -1);
  for (size_t i = 0; i < nops; ++i) {
    if (ops[i].kind != OP_GEMM && ops[i].kind != OP_SYRK) continue;
    UpdateArgs& a = upd[i].args;
    int ks = update_ksplit_for(a.M, a.N, a.K, a.tri, upd[i].tile, ops[i].kind == OP_SYRK && !ops[i].deferred);
    int full = 0;
    if (ks <= 1) ks = update_tail_split(a.ntiles, a.K, upd[i].tile, upd[i].max_ctas, &full);
    if (ks <= 1) continue;
    a.ksplit = ks;
    a.full_items = full;
    const int64_t e = update_ws_elems(a.M, a.N, a.tri, upd[i].tile, ks, full);
    ws = e > ws ? e : ws;
    cnt = a.ntiles > cnt ? a.ntiles : cnt;
    int s = -1;
    for (size_t q = 0; q < slot_last.size() && s < 0; ++q) {
      const int l = slot_last[q];
      if (!anc || ((*anc)[i * words + l / 64] >> (l % 64) & 1)) s = (int)q;
    }
    if (s < 0) {
      s = (int)slot_last.size();
      slot_last.push_back(0);
    }
    slot_last[s] = (int)i;
    slot_of[i] = s;
  }
  *ws_out = nullptr;
  *cnt_out = nullptr;
  *cnt_bytes = 0;
  if (ws == 0) return cudaSuccess;
  const size_t nslots = slot_last.size();
  cudaError_t e;
  if ((e = cudaMalloc(ws_out, nslots * ws * sizeof(double))) != cudaSuccess) return e;
  *cnt_bytes = nslots * cnt * sizeof(int);
  if ((e = cudaMalloc(cnt_out, *cnt_bytes)) != cudaSuccess) return e;
  if ((e = cudaMemset(*cnt_out, 0, *cnt_bytes)) != cudaSuccess) return e;
  for (size_t i = 0; i < nops; ++i) {
    if (slot_of[i] < 0) continue;
    upd[i].args.ws = *ws_out + (size_t)slot_of[i] * ws;
    upd[i].args.counters = *cnt_out + (size_t)slot_of[i] * cnt;
  }
  return cudaSuccess;
}

static cudaError_t setup_splitk(Plan& p, const std::vector<uint64_t>* anc) {
  return setup_splitk_ops(p.ops, p.upd, anc, &p.splitk_ws, &p.splitk_cnt, &p.cnt_bytes);
}

// ------------------------------------------------------------------ profiling
struct ProfRecord {
  cudaEvent_t start, stop;
  int kind;
  double flops;
  int m, n, k, level;
};
static std::mutex g_prof_mu;
static std::atomic<int> g_prof_on{0};
static std::vector<ProfRecord> g_prof;
static std::vector<cudaEvent_t> g_prof_pool;

static cudaEvent_t prof_event() {
  if (!g_prof_pool.empty()) {
    cudaEvent_t e = g_prof_pool.back();
    g_prof_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

__global__ void k_noop() {}

// 2-D copy dst[c * dld + r] = src[c * sld + r], r < w (contiguous), c < h; one
// of the two is pinned host memory addressed through UVA.  16-byte accesses
// when both sides allow them, many loads in flight per thread.
// tri (scalar path only): 0 every element, 1 only r >= c, 2 only r <= c (r < w
// the contiguous index, c < h the strided one): the uplo triangle of a
// diagonal block, so nothing outside it is written.
__global__ void __launch_bounds__(256) k_copy2d(double* __restrict__ dst, int64_t dld,
                                                const double* __restrict__ src, int64_t sld, int64_t w, int64_t h,
                                                int vec, int tri) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (vec) {
    const int64_t w2 = w / 2, tot = w2 * h;
    for (int64_t e0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e0 < tot; e0 += 4 * stride) {
      double2 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t e = e0 + u * stride;
        if (e < tot) v[u] = reinterpret_cast<const double2*>(src + (e / w2) * sld)[e % w2];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t e = e0 + u * stride;
        if (e < tot) reinterpret_cast<double2*>(dst + (e / w2) * dld)[e % w2] = v[u];
      }
    }
  } else {
    const int64_t tot = w * h;
    for (int64_t e0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e0 < tot; e0 += 4 * stride) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t e = e0 + u * stride;
        if (e < tot) v[u] = src[(e / w) * sld + e % w];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t e = e0 + u * stride;
        const int64_t r = e % w, c = e / w;
        if (e < tot && (tri == 0 || (tri == 1 ? r >= c : r <= c))) dst[c * dld + r] = v[u];
      }
    }
  }
}

static cudaError_t launch_copy2d(double* dst, int64_t dld, const double* src, int64_t sld, int64_t w, int64_t h,
                                 cudaStream_t st, int tri = 0) {
  const bool vec = tri == 0 && (w % 2 == 0) && (dld % 2 == 0) && (sld % 2 == 0) &&
                   ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0;
  const int64_t items = vec ? (w / 2) * h : w * h;
  int grid = (int)((items + 256 * 4 - 1) / (256 * 4));
  grid = grid < 8 ? (grid < 1 ? 1 : grid) : 8;  // 8 CTAs keep ~32 KB of PCIe requests in flight
  k_copy2d<<<grid, 256, 0, st>>>(dst, dld, src, sld, w, h, vec ? 1 : 0, tri);
  return cudaGetLastError();
}

// Host-matrix path: copies on two copy streams synchronised with the graph by
// events (default) or as memcpy nodes inside the graph (RELAPACK_SPLIT_COPIES=0)
static bool split_copies_enabled() {
  static const bool on = env_int("RELAPACK_SPLIT_COPIES", 1) != 0;
  return on;
}

// Host-matrix copies as cudaMemcpy2DAsync nodes (default) or SM kernels
// (RELAPACK_COPY_KERNEL=1; measured slower: n = 16384 e2e 78.8 vs 65.4 ms,
// tools/exp15.sh).
static bool copy_kernels() {
  static const bool on = env_int("RELAPACK_COPY_KERNEL", 0) != 0;
  return on;
}

// Timing experiments only (tools/): RELAPACK_DEBUG_SKIP = bit mask of op kinds
// (1 potf2, 2 trsm, 4 gemm, 8 syrk) replaced by an empty kernel.  The result
// is then not a factorization.
static int debug_skip_mask() {
  static const int m = env_int("RELAPACK_DEBUG_SKIP", 0);
  return m;
}

// The copy of host-path op i (OP_H2D / OP_D2H): L-view block rows [c_i,
// c_i+m) x cols [c_j, c_j+k) as one 2-D copy on stream st.
static cudaError_t copy_block(const Plan& pl, size_t i, double* A, int64_t ld, int layout, cudaStream_t st) {
  const PlanOp& op = pl.ops[i];
  const size_t width = sizeof(double) * (layout == kLayoutN ? op.m : op.k);
  const size_t height = layout == kLayoutN ? op.k : op.m;
  double* dev = A + lv_off(layout, op.c_i, op.c_j, ld);
  double* host = const_cast<double*>(pl.host) + lv_off(layout, op.c_i, op.c_j, pl.hld);
  if (copy_kernels()) {
    const int64_t w = (int64_t)(width / sizeof(double)), h = (int64_t)height;
    return op.kind == OP_H2D ? launch_copy2d(dev, ld, host, pl.hld, w, h, st)
                             : launch_copy2d(host, pl.hld, dev, ld, w, h, st);
  }
  return op.kind == OP_H2D ? cudaMemcpy2DAsync(dev, ld * sizeof(double), host, pl.hld * sizeof(double), width, height,
                                               cudaMemcpyHostToDevice, st)
                           : cudaMemcpy2DAsync(host, pl.hld * sizeof(double), dev, ld * sizeof(double), width, height,
                                               cudaMemcpyDeviceToHost, st);
}

static cudaError_t launch_op_impl(const Plan& pl, size_t i, double* A, int64_t ld, int layout, int* d_info,
                                  cudaStream_t st);

// Kernel pointer argument of element offset `off`: absolute, or (rebased
// plan) the byte offset from the matrix base the kernel adds at run time.
static double* at_off(const Plan& pl, double* A, int64_t off) {
  return pl.rebased ? reinterpret_cast<double*>(static_cast<uintptr_t>(off) * sizeof(double)) : A + off;
}
// The info pointer plan kernels get: the tagged PlanState of a rebased plan.
static int* op_info(const Plan& pl, int* d_info) {
  return pl.rebased ? reinterpret_cast<int*>(reinterpret_cast<uintptr_t>(pl.d_state) | 1) : d_info;
}

static cudaError_t launch_op(const Plan& pl, size_t i, double* A, int64_t ld, int layout, int* d_info,
                             cudaStream_t st) {
  g_launch_trace = pl.d_trace ? pl.d_trace + i : nullptr;
  const cudaError_t e = launch_op_impl(pl, i, A, ld, layout, d_info, st);
  g_launch_trace = nullptr;
  return e;
}

static cudaError_t launch_op_impl(const Plan& pl, size_t i, double* A, int64_t ld, int layout, int* d_info,
                                  cudaStream_t st) {
  const PlanOp& op = pl.ops[i];
  if (debug_skip_mask() & (1 << (int)op.kind)) {
    k_noop<<<1, 32, 0, st>>>();
    return cudaGetLastError();
  }
  switch (op.kind) {
    case OP_H2D:
    case OP_D2H: {
      if (pl.split_copies)  // graph-side half of a split copy (the copy runs on a copy stream)
        return op.kind == OP_H2D ? cudaStreamWaitEvent(st, pl.ev[i], cudaEventWaitExternal)
                                 : cudaEventRecordWithFlags(pl.ev[i], st, cudaEventRecordExternal);
      return copy_block(pl, i, A, ld, layout, st);
    }
    case OP_POTF2:
      return launch_potf2(at_off(pl, A, lv_off(layout, op.c_i, op.c_j, ld)), ld, layout, op.n, op_info(pl, d_info),
                          op.info_base, st);
    case OP_TRSM:
      return launch_trsm_any(at_off(pl, A, lv_off(layout, op.a_i, op.a_j, ld)), ld,
                             at_off(pl, A, lv_off(layout, op.c_i, op.c_j, ld)), ld, layout, op.m, op.k,
                             op_info(pl, d_info), st);
    case OP_GEMM:
    case OP_SYRK:
      return launch_update(pl.upd[i], st);
    default:
      return cudaErrorInvalidValue;
  }
}

// Run-start nodes: reset info and (robustness after an early exit) the
// split-K arrival counters.
__global__ void k_trace_reset(TraceRec* tr, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    tr[i].t0 = ~0ull;
    tr[i].t1 = 0;
  }
}

// the prologue's nodes after the info reset (set_info false: the caller did it)
static cudaError_t run_prologue_rest(const Plan& pl, int* d_info, cudaStream_t st, bool set_info) {
  cudaError_t e = set_info ? launch_set_int(d_info, 0, st) : cudaSuccess;
  if (e == cudaSuccess && pl.d_trace) {
    const int n = (int)pl.ops.size();
    k_trace_reset<<<(n + 255) / 256, 256, 0, st>>>(pl.d_trace, n);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess && pl.splitk_cnt) e = cudaMemsetAsync(pl.splitk_cnt, 0, pl.cnt_bytes, st);
  return e;
}

// Serial execution in plan order (eager mode and the profiler).
static cudaError_t run_ops(const Plan& pl, double* A, int64_t ld, int layout, int* d_info, cudaStream_t st,
                           bool profile) {
  cudaError_t e = run_prologue_rest(pl, d_info, st, true);
  if (e != cudaSuccess) return e;
  std::unique_lock<std::mutex> plk(g_prof_mu, std::defer_lock);
  if (profile) plk.lock();
  for (size_t i = 0; i < pl.ops.size(); ++i) {
    const PlanOp& op = pl.ops[i];
    ProfRecord rec{};
    const bool rec_this = profile && op.kind < OP_H2D;
    if (rec_this) {
      rec.start = prof_event();
      rec.stop = prof_event();
      rec.kind = (int)op.kind;
      rec.flops = op.flops;
      rec.m = op.m;
      rec.n = op.n;
      rec.k = op.k;
      rec.level = op.level;
      cudaEventRecord(rec.start, st);
    }
    if ((e = launch_op(pl, i, A, ld, layout, d_info, st)) != cudaSuccess) return e;
    if (rec_this) {
      cudaEventRecord(rec.stop, st);
      g_prof.push_back(rec);
    }
  }
  return cudaSuccess;
}

// Capture the plan as a DAG on one stream: before each op the capture
// dependencies are set to the graph nodes of the op's footprint
// dependencies, so independent ops (the lookahead trailing updates and the
// next panel's chain) become parallel branches of the graph.  `launch(i, st)`
// issues op i; cls receives each op's priority class (set_node_priorities).
// Used by the single-GPU executor and by the multi-GPU one (dist.cu, whose
// collectives are captured nodes too).
cudaError_t capture_plan_dag(const std::vector<PlanOp>& ops, const std::vector<std::vector<int>>& deps,
                             cudaStream_t st, const std::function<cudaError_t(size_t, cudaStream_t)>& launch,
                             std::vector<cudaGraphNode_t>& nodes, std::vector<char>& deferred_node) {
  cudaError_t e;
  cudaStreamCaptureStatus cs;
  const cudaGraphNode_t* cur = nullptr;
  size_t ncur = 0;
  if ((e = cudaStreamGetCaptureInfo(st, &cs, nullptr, nullptr, &cur, &ncur)) != cudaSuccess) return e;
  if (ncur != 1) return cudaErrorStreamCaptureInvalidated;
  const cudaGraphNode_t root = cur[0];
  nodes.assign(ops.size(), nullptr);
  std::vector<cudaGraphNode_t> want;
  std::vector<cudaGraphEdgeData> edge;
  auto kernel_op = [&](int j) { return ops[j].kind <= OP_SYRK && !(debug_skip_mask() >> ops[j].kind & 1); };
  for (size_t i = 0; i < ops.size(); ++i) {
    want.clear();
    edge.clear();
    for (int d : deps[i]) {
      want.push_back(nodes[d]);
      // programmatic edge between two plan kernels (the downstream grid may
      // launch once every CTA of the upstream one passed pdl_trigger; it
      // still waits for its completion in ld_info) — not out of the
      // deferred, SM-capped updates, whose early trigger would park the
      // dependents' CTAs on the SMs the chain needs
      cudaGraphEdgeData x{};
      const int pm = pdl_mode();
      const OpKind dk = ops[i].kind;
      const bool into = pm == 1 || dk == OP_POTF2 || dk == OP_TRSM || (pm == 3 && dk == OP_SYRK && !ops[i].deferred);
      if (pm > 0 && into && kernel_op((int)i) && kernel_op(d) && !ops[d].deferred) {
        x.from_port = cudaGraphKernelNodePortProgrammatic;
        x.type = cudaGraphDependencyTypeProgrammatic;
      }
      edge.push_back(x);
    }
    if (want.empty()) {
      want.push_back(root);
      edge.push_back(cudaGraphEdgeData{});
    }
    if ((e = cudaStreamUpdateCaptureDependencies_v2(st, want.data(), edge.data(), want.size(),
                                                    cudaStreamSetCaptureDependencies)) != cudaSuccess)
      return e;
    if ((e = launch(i, st)) != cudaSuccess) return e;
    if ((e = cudaStreamGetCaptureInfo(st, &cs, nullptr, nullptr, &cur, &ncur)) != cudaSuccess) return e;
    if (ncur != 1) return cudaErrorStreamCaptureInvalidated;
    nodes[i] = cur[0];
    // priority class: 2 deferred update, 1 other GEMM (the TRSM's updates),
    // 0 the chain (base cases, TRSM bases, the non-deferred SYRKs)
    const PlanOp& o = ops[i];
    deferred_node.push_back((char)(o.deferred ? (o.flops >= bulk_min_flops() ? 3 : 2) : o.kind == OP_GEMM ? 1 : 0));
  }
  // join every sink so the capture ends on one node
  std::vector<char> has_succ(ops.size(), 0);
  for (size_t i = 0; i < ops.size(); ++i)
    for (int d : deps[i]) has_succ[d] = 1;
  want.clear();
  for (size_t i = 0; i < ops.size(); ++i)
    if (!has_succ[i]) want.push_back(nodes[i]);
  if (want.empty()) want.push_back(root);
  return cudaStreamUpdateCaptureDependencies(st, want.data(), want.size(), cudaStreamSetCaptureDependencies);
}

static cudaError_t capture_node(cudaStream_t st, cudaGraphNode_t* node) {
  cudaStreamCaptureStatus cs;
  const cudaGraphNode_t* cur = nullptr;
  size_t ncur = 0;
  cudaError_t e = cudaStreamGetCaptureInfo(st, &cs, nullptr, nullptr, &cur, &ncur);
  if (e == cudaSuccess && ncur != 1) e = cudaErrorStreamCaptureInvalidated;
  if (e == cudaSuccess) *node = cur[0];
  return e;
}

static cudaError_t capture_dag(Plan& pl, const std::vector<std::vector<int>>& deps, double* A, int64_t ld,
                               int layout, int* d_info, cudaStream_t st, std::vector<cudaGraphNode_t>& nodes,
                               std::vector<char>& deferred_node) {
  cudaError_t e;
  if (pl.rebased) {
    if ((e = launch_plan_begin(pl, A, st)) != cudaSuccess) return e;
    if ((e = capture_node(st, &pl.begin_node)) != cudaSuccess) return e;
    pl.cur_A = A;
  }
  if ((e = run_prologue_rest(pl, d_info, st, !pl.rebased)) != cudaSuccess) return e;
  e = capture_plan_dag(
      pl.ops, deps, st, [&](size_t i, cudaStream_t s) { return launch_op(pl, i, A, ld, layout, d_info, s); }, nodes,
      deferred_node);
  if (e == cudaSuccess && pl.rebased) {
    k_plan_end<<<1, 1, 0, st>>>(pl.d_state, d_info);
    if ((e = cudaGetLastError()) == cudaSuccess) e = capture_node(st, &pl.end_node);
    pl.cur_info = d_info;
  }
  return e;
}

cudaError_t set_node_priorities(const std::vector<cudaGraphNode_t>& nodes, const std::vector<char>& deferred) {
  int least = 0, greatest = 0;
  cudaError_t e = cudaDeviceGetStreamPriorityRange(&least, &greatest);
  if (e != cudaSuccess) return e;
  for (size_t i = 0; i < nodes.size(); ++i) {
    cudaGraphNodeType t;
    if ((e = cudaGraphNodeGetType(nodes[i], &t)) != cudaSuccess) return e;
    if (t != cudaGraphNodeTypeKernel) continue;
    cudaKernelNodeAttrValue v{};
    const int cls = deferred[i];
    const int mode = env_int("RELAPACK_PRIO_MODE", 1);
    // mode 0: deferred lowest, the rest highest; 1: chain > TRSM GEMMs >
    // deferred; 2: TRSM GEMMs > chain > deferred; 3: as 1 with the small
    // (uncapped) deferred updates one level above the large ones
    const int step = greatest < least ? 1 : -1;  // towards lower priority
    if (cls >= 2)
      v.priority = !defer_low_priority() ? greatest
                   : (mode == 3 && cls == 2 && least != greatest + 2 * step) ? least - step
                                                                             : least;
    else if (mode == 1 || mode == 3)
      v.priority = cls == 0 ? greatest : greatest + step;
    else if (mode == 2)
      v.priority = cls == 1 ? greatest : greatest + step;
    else
      v.priority = greatest;
    if ((e = cudaGraphKernelNodeSetAttribute(nodes[i], cudaLaunchAttributePriority, &v)) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// Host-matrix copy blocks: column panels x row chunks of the lower L-view
// (RELAPACK_COPY_PANEL / RELAPACK_COPY_ROWS; the panel must divide the rows).
static int copy_panel() { return env_int("RELAPACK_COPY_PANEL", 512); }
// host-path copy block height: n / 8 clamped to [512, 2048] (n = 4096: 512
// rows, the first base cases start sooner: e2e 2.88 -> 2.77 ms; n >= 16384:
// 2048), RELAPACK_COPY_ROWS overrides
static int copy_rows(int n) {
  const int r = env_int("RELAPACK_COPY_ROWS", 0);
  if (r > 0) return r;
  return n / 8 < 512 ? 512 : (n / 8 > 2048 ? 2048 : n / 8);
}

// Every knob the executor reads while building, launching or capturing a plan,
// as one string (part of the plan-cache key, so changing any of them inside a
// process never replays a stale graph).  The update kernel's tile / split-K
// environment knobs are read once per process (update.cu) and are not here.
static std::string knob_signature(const PlanParams& pp, bool use_graph, bool use_dag) {
  char b[512];
  snprintf(b, sizeof(b),
           "c%d T%d tb%d la%d tr%d ld%d db%d bc%d hg%d g%d d%d bulk%d bmin%g upd%d dl%d sk%d pdl%d tr%d pm%d sc%d ck%d "
           "cp%d cr%d skip%d nb%d",
           pp.crossover, pp.split_tile, pp.trsm_base, (int)pp.lookahead, pp.trsm_rows, pp.lookahead_depth,
           (int)pp.defer_b21, pp.b21_chunks, pp.host_gemm_cols, (int)use_graph, (int)use_dag, bulk_ctas(),
           bulk_min_flops(), upd_ctas(), (int)defer_low_priority(), (int)splitk_enabled(), pdl_mode(),
           (int)trace_enabled(), env_int("RELAPACK_PRIO_MODE", 1), (int)split_copies_enabled(), (int)copy_kernels(),
           copy_panel(), env_int("RELAPACK_COPY_ROWS", 0), debug_skip_mask(), pp.blocked_nb);
  return b;
}

// Enqueue the factorization of the device matrix A (already validated).
int enqueue_potrf(int dev, double* A, int n, int64_t ld, int layout, int* d_info, cudaStream_t st, const double* host,
                  int64_t hld, int blocked_nb) {
  DeviceState* ds = device_state(dev);
  cudaError_t e;
  PlanParams pp = current_params();
  pp.blocked_nb = blocked_nb;
  if (host) {
    // host-matrix path: the TRSM GEMMs go in copy-panel-wide column chunks,
    // each waiting only for its own host blocks (n = 16384 e2e 57.0 -> 52.7 ms,
    // tools/experiments/exp_e2e2.sh; no effect on the device-only path)
    pp.host_gemm_cols = env_int("RELAPACK_HOST_GEMM_COLS", copy_panel());
    pp.b21_chunks = env_int("RELAPACK_HOST_B21_CHUNKS", pp.b21_chunks);
  }
  const bool profile = g_prof_on.load() != 0;
  const bool use_graph = graphs_enabled() && !profile;
  std::lock_guard<std::mutex> lk(ds->mu);
  if ((e = ensure_device(ds)) != cudaSuccess) return cuda_fail(e, "device setup");
  const bool use_dag = use_graph && dag_enabled();
  const int bulk = bulk_ctas();
  const int upd_cap = upd_ctas();
  (void)bulk;
  // a pointer-independent graph serves every matrix of this shape (its key
  // holds only whether A allows TMA: 16-byte aligned base, even ld) and every
  // info pointer; the host matrix of the pinned path only enters the graph
  // when its copies are graph nodes (split copies off)
  const bool rebased = use_dag && env_int("RELAPACK_REBASE", 1) != 0;
  const uintptr_t a_key = rebased ? 1 + (((reinterpret_cast<uintptr_t>(A) & 15) == 0 && ld % 2 == 0) ? 1 : 0)
                                  : reinterpret_cast<uintptr_t>(A);
  const uintptr_t h_key = rebased && split_copies_enabled() ? (host ? 1 : 0) : reinterpret_cast<uintptr_t>(host);
  PlanKey key{a_key, n, ld, layout, rebased ? 0 : reinterpret_cast<uintptr_t>(d_info), h_key, hld,
              knob_signature(pp, use_graph, use_dag) + (rebased ? " rebased" : "")};
  Plan* plan = nullptr;
  auto it = ds->index.find(key);
  if (it != ds->index.end()) {
    ds->lru.splice(ds->lru.begin(), ds->lru, it->second);
    plan = it->second->second.get();
  } else {
    auto p = std::make_unique<Plan>();
    build_potrf_plan(n, pp, p->ops);
    if (host) {
      // host-matrix path: H2D blocks first, D2H blocks last; the footprint
      // DAG lets the first leaves start on the first blocks and each block go
      // back as soon as its last writer is done
      std::vector<PlanOp> all;
      append_copies(n, copy_panel(), copy_rows(n), OP_H2D, all);
      all.insert(all.end(), p->ops.begin(), p->ops.end());
      append_copies(n, copy_panel(), copy_rows(n), OP_D2H, all);
      p->ops.swap(all);
      p->host = host;
      p->hld = hld;
      p->split_copies = use_graph && split_copies_enabled();
      if (p->split_copies) {
        // first use / last write of every copy block (footprint overlap)
        std::vector<Rect> W(p->ops.size()), R1(p->ops.size()), R2(p->ops.size());
        for (size_t i = 0; i < p->ops.size(); ++i) op_regions(p->ops[i], &W[i], &R1[i], &R2[i]);
        auto hit = [](const Rect& a, const Rect& b) {
          return a.buf >= 0 && a.buf == b.buf && a.r0 < b.r1 && b.r0 < a.r1 && a.c0 < b.c1 && b.c0 < a.c1;
        };
        std::vector<std::pair<size_t, int>> hk, dk;
        for (size_t i = 0; i < p->ops.size(); ++i) {
          const OpKind kd = p->ops[i].kind;
          if (kd != OP_H2D && kd != OP_D2H) continue;
          const Rect blk = kd == OP_H2D ? W[i] : R1[i];
          size_t key = kd == OP_H2D ? p->ops.size() : 0;
          for (size_t j = 0; j < p->ops.size(); ++j) {
            const OpKind kj = p->ops[j].kind;
            if (kj == OP_H2D || kj == OP_D2H) continue;
            if (kd == OP_H2D && (hit(blk, W[j]) || hit(blk, R1[j]) || hit(blk, R2[j]))) {
              key = j;
              break;
            }
            if (kd == OP_D2H && hit(blk, W[j])) key = j;
          }
          (kd == OP_H2D ? hk : dk).push_back({key, (int)i});
        }
        std::stable_sort(hk.begin(), hk.end());
        std::stable_sort(dk.begin(), dk.end());
        for (auto& q : hk) p->h2d_order.push_back(q.second);
        for (auto& q : dk) p->d2h_order.push_back(q.second);
        p->ev.assign(p->ops.size(), nullptr);
        for (size_t i = 0; i < p->ops.size(); ++i)
          if (p->ops[i].kind == OP_H2D || p->ops[i].kind == OP_D2H)
            if ((e = cudaEventCreateWithFlags(&p->ev[i], cudaEventDisableTiming)) != cudaSuccess)
              return cuda_fail(e, "copy event");
      }
    }
    p->upd.resize(p->ops.size());
    if (trace_enabled() && (e = cudaMalloc(&p->d_trace, p->ops.size() * sizeof(TraceRec))) != cudaSuccess)
      return cuda_fail(e, "trace buffer");
    p->rebased = rebased;
    std::vector<CUtensorMap> hmaps;
    std::vector<long long> hoff;
    if (rebased && (e = cudaMalloc(&p->d_state, sizeof(PlanState))) != cudaSuccess) return cuda_fail(e, "plan state");
    for (size_t i = 0; i < p->ops.size(); ++i)
      if (p->ops[i].kind == OP_GEMM || p->ops[i].kind == OP_SYRK) {
        fill_update(p->upd[i], p->ops[i], A, ld, layout, d_info);
        if (rebased) {
          // descriptors encoded for this call's A, rebased by every run's first
          // node; pointer arguments become byte offsets from the matrix base
          UpdateArgs& a = p->upd[i].args;
          auto boff = [&](const double* x) {
            return (long long)(reinterpret_cast<uintptr_t>(x) - reinterpret_cast<uintptr_t>(A));
          };
          if (p->upd[i].use_tma) {
            a.gmap = reinterpret_cast<const CUtensorMap*>(hmaps.size());  // slot index, patched below
            hmaps.push_back(p->upd[i].tmA);
            hmaps.push_back(p->upd[i].tmB);
            hoff.push_back(boff(a.A));
            hoff.push_back(boff(a.B));
          }
          a.C = reinterpret_cast<double*>(static_cast<uintptr_t>(boff(a.C)));
          a.A = reinterpret_cast<const double*>(static_cast<uintptr_t>(boff(a.A)));
          a.B = reinterpret_cast<const double*>(static_cast<uintptr_t>(boff(a.B)));
          a.d_info = op_info(*p, d_info);
        }
        // deferred (lookahead) updates big enough to hold SMs for long run
        // persistent on `bulk` CTAs, leaving SMs to the chain; small ones
        // (below RELAPACK_BULK_MIN_GF GFLOP) run uncapped at low priority —
        // capped, a small 64-tile GEMM runs one 4-warp CTA per SM at half the
        // SM's rate and ends up on the critical path (n = 4096 trace)
        if (use_dag && p->ops[i].deferred && p->ops[i].flops >= bulk_min_flops()) p->upd[i].max_ctas = bulk;
        // every other big update also leaves a few SMs free, so a base case
        // or TRSM that becomes ready does not wait for a long tile to drain
        // (tools/trace_timeline.py: otherwise the chain waits ~24 ms at n = 16384)
        else if (use_dag && upd_cap > 0) p->upd[i].max_ctas = upd_cap;
      }
    if (rebased) {
      p->nmaps = (int)hmaps.size();
      if (p->nmaps > 0) {
        if ((e = cudaMalloc(&p->d_maps, hmaps.size() * sizeof(CUtensorMap))) != cudaSuccess ||
            (e = cudaMemcpy(p->d_maps, hmaps.data(), hmaps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice)) !=
                cudaSuccess ||
            (e = cudaMalloc(&p->d_map_off, hoff.size() * sizeof(long long))) != cudaSuccess ||
            (e = cudaMemcpy(p->d_map_off, hoff.data(), hoff.size() * sizeof(long long), cudaMemcpyHostToDevice)) !=
                cudaSuccess)
          return cuda_fail(e, "plan descriptors");
      }
      for (size_t i = 0; i < p->ops.size(); ++i)
        if ((p->ops[i].kind == OP_GEMM || p->ops[i].kind == OP_SYRK) && p->upd[i].use_tma)
          p->upd[i].args.gmap = p->d_maps + reinterpret_cast<uintptr_t>(p->upd[i].args.gmap);
    }
    std::vector<std::vector<int>> deps;
    std::vector<uint64_t> anc;
    if (use_dag) compute_deps(p->ops, deps, &anc);
    if (splitk_enabled() && (e = setup_splitk(*p, use_dag ? &anc : nullptr)) != cudaSuccess)
      return cuda_fail(e, "split-K workspace");
    if (use_graph) {
      cudaGraph_t g = nullptr;
      std::vector<cudaGraphNode_t> nodes;
      std::vector<char> deferred;
      if ((e = cudaStreamBeginCapture(ds->capture, cudaStreamCaptureModeThreadLocal)) != cudaSuccess)
        return cuda_fail(e, "begin capture");
      cudaError_t er = use_dag ? capture_dag(*p, deps, A, ld, layout, d_info, ds->capture, nodes, deferred)
                               : run_ops(*p, A, ld, layout, d_info, ds->capture, false);
      e = cudaStreamEndCapture(ds->capture, &g);
      if (er != cudaSuccess) {
        if (g) cudaGraphDestroy(g);
        return cuda_fail(er, "launch during capture");
      }
      if (e != cudaSuccess) return cuda_fail(e, "end capture");
      if (use_dag && (e = set_node_priorities(nodes, deferred)) != cudaSuccess) {
        cudaGraphDestroy(g);
        return cuda_fail(e, "graph node priority");
      }
      e = cudaGraphInstantiateWithFlags(&p->exec, g, use_dag ? cudaGraphInstantiateFlagUseNodePriority : 0);
      if (rebased)
        p->graph = g;  // its begin / end node handles retarget the exec per call
      else
        cudaGraphDestroy(g);
      if (e != cudaSuccess) return cuda_fail(e, "graph instantiate");
    }
    ds->lru.emplace_front(key, std::move(p));
    ds->index[key] = ds->lru.begin();
    plan = ds->lru.front().second.get();
    while (ds->lru.size() > 32) {
      ds->index.erase(ds->lru.back().first);
      ds->lru.pop_back();
    }
  }
  if (plan->rebased) {
    if ((e = retarget(*plan, A, d_info)) != cudaSuccess) return cuda_fail(e, "graph retarget");
    if (host) plan->host = host;  // the split copies run outside the graph
  }
  if (use_graph && plan->split_copies) {
    // H2D blocks on one copy stream (each followed by its event), the graph
    // (waiting on those events per block), the D2H blocks on the other copy
    // stream (each after the graph's record of its event); `st` ends after all
    const Plan& pl = *plan;
    e = cudaEventRecord(ds->ev_start, st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(ds->h2d, ds->ev_start, 0);
    for (size_t q = 0; q < pl.h2d_order.size() && e == cudaSuccess; ++q) {
      const int i = pl.h2d_order[q];
      e = copy_block(pl, i, A, ld, layout, ds->h2d);
      if (e == cudaSuccess) e = cudaEventRecord(pl.ev[i], ds->h2d);
    }
    if (e == cudaSuccess) e = cudaGraphLaunch(pl.exec, st);
    for (size_t q = 0; q < pl.d2h_order.size() && e == cudaSuccess; ++q) {
      const int i = pl.d2h_order[q];
      e = cudaStreamWaitEvent(ds->d2h, pl.ev[i], 0);
      if (e == cudaSuccess) e = copy_block(pl, i, A, ld, layout, ds->d2h);
    }
    if (e == cudaSuccess) e = cudaEventRecord(ds->ev_done, ds->d2h);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ds->ev_done, 0);
  } else if (use_graph) {
    e = cudaGraphLaunch(plan->exec, st);
  } else {
    e = run_ops(*plan, A, ld, layout, d_info, st, profile);
  }
  if (e != cudaSuccess) return cuda_fail(e, "launch");
  if (plan->d_trace) {
    std::lock_guard<std::mutex> tl(g_trace_mu);
    g_trace_plan = plan;
  }
  return 0;
}

// Copy the last traced plan's records: 7 doubles per op (kind, m, n, k, flops,
// start_us, end_us; times relative to the earliest start).  Synchronizes.
int trace_read(int max, double* out) {
  std::lock_guard<std::mutex> tl(g_trace_mu);
  const Plan* pl = static_cast<const Plan*>(g_trace_plan);
  if (!pl || !pl->d_trace) return 0;
  const size_t nops = pl->ops.size();
  std::vector<TraceRec> h(nops);
  if (cudaDeviceSynchronize() != cudaSuccess ||
      cudaMemcpy(h.data(), pl->d_trace, nops * sizeof(TraceRec), cudaMemcpyDeviceToHost) != cudaSuccess)
    return -1;
  unsigned long long t00 = ~0ull;
  for (const TraceRec& r : h)
    if (r.t1 && r.t0 < t00) t00 = r.t0;
  int cnt = 0;
  for (size_t i = 0; i < nops && cnt < max; ++i, ++cnt) {
    const PlanOp& op = pl->ops[i];
    double* o = out + 7 * cnt;
    o[0] = op.kind; o[1] = op.m; o[2] = op.n; o[3] = op.k; o[4] = op.flops;
    o[5] = h[i].t1 ? (double)(h[i].t0 - t00) * 1e-3 : -1.0;
    o[6] = h[i].t1 ? (double)(h[i].t1 - t00) * 1e-3 : -1.0;
  }
  return cnt;
}

static int check_args(char uplo, int n, const void* A, int lda, int* layout) {
  if (uplo == 'L' || uplo == 'l')
    *layout = kLayoutN;
  else if (uplo == 'U' || uplo == 'u')
    *layout = kLayoutT;
  else
    return -1;
  if (n < 0) return -2;
  if (n > 0 && A == nullptr) return -3;
  if (lda < (n > 1 ? n : 1)) return -4;
  return 0;
}

static bool is_device_pointer(const void* p, int* dev) {
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) {
    *dev = at.device;
    return true;
  }
  return false;
}

static bool is_pinned_host(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// Copy the uplo triangle between a pageable host matrix and a device matrix in
// column panels of w columns.  Host -> device: each panel's rows from its
// diagonal block on (the diagonal block whole; the other-triangle values it
// carries into the staging buffer are never used).  Device -> host: the part
// of the panel outside its diagonal block as one 2-D copy, the diagonal block
// through a pinned bounce buffer and per-column host copies of its uplo part
// only, so nothing outside the triangle is written in the caller's matrix.
static cudaError_t copy_triangle(double* dst, int64_t ld_dst, const double* src, int64_t ld_src, int n, int layout,
                                 cudaMemcpyKind kind, cudaStream_t st, double* bounce = nullptr) {
  const int w = 256;
  for (int j0 = 0; j0 < n; j0 += w) {
    const int jw = (n - j0 < w) ? n - j0 : w;
    // memory rows of the panel's triangle part: [r0, r0 + rows)
    const int64_t r0 = layout == kLayoutN ? j0 : 0;
    const int64_t rows = layout == kLayoutN ? n - j0 : j0 + jw;
    cudaError_t e;
    if (kind == cudaMemcpyHostToDevice || !bounce) {
      e = cudaMemcpy2DAsync(dst + r0 + (int64_t)j0 * ld_dst, ld_dst * sizeof(double), src + r0 + (int64_t)j0 * ld_src,
                            ld_src * sizeof(double), rows * sizeof(double), jw, kind, st);
      if (e != cudaSuccess) return e;
      continue;
    }
    // the rectangle outside the diagonal block: below it (L) / above it (U)
    const int64_t q0 = layout == kLayoutN ? j0 + jw : 0;
    const int64_t qn = layout == kLayoutN ? n - (j0 + jw) : j0;
    if (qn > 0 && (e = cudaMemcpy2DAsync(dst + q0 + (int64_t)j0 * ld_dst, ld_dst * sizeof(double),
                                         src + q0 + (int64_t)j0 * ld_src, ld_src * sizeof(double),
                                         qn * sizeof(double), jw, kind, st)) != cudaSuccess)
      return e;
    if ((e = cudaMemcpy2DAsync(bounce, jw * sizeof(double), src + j0 + (int64_t)j0 * ld_src, ld_src * sizeof(double),
                               jw * sizeof(double), jw, kind, st)) != cudaSuccess)
      return e;
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
    for (int c = 0; c < jw; ++c) {
      const int a = layout == kLayoutN ? c : 0, b = layout == kLayoutN ? jw : c + 1;  // rows [a, b) of column c
      memcpy(dst + (j0 + a) + (int64_t)(j0 + c) * ld_dst, bounce + a + (int64_t)c * jw, (b - a) * sizeof(double));
    }
  }
  return cudaSuccess;
}

// Restores the calling thread's current device on every return path.
struct DeviceGuard {
  int saved = -1;
  DeviceGuard() { cudaGetDevice(&saved); }
  ~DeviceGuard() {
    int cur = -1;
    if (saved >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != saved) cudaSetDevice(saved);
  }
};

}  // namespace relapack

using namespace relapack;

// =================================================================== C ABI
extern "C" {

void relapack_dpotrf(const char* uplo, const int* n_, double* A, const int* lda_, int* info) {
  if (!uplo || !n_ || !lda_ || !info) {
    if (info) *info = -1;
    return;
  }
  const int n = *n_, lda = *lda_;
  int layout = 0;
  int ai = check_args(*uplo, n, A, lda, &layout);
  if (ai != 0) {
    *info = ai;
    return;
  }
  if (n == 0) {
    *info = 0;
    return;
  }
  cudaStream_t st = g_stream;
  int dev = 0;
  const bool on_device = is_device_pointer(A, &dev);
  cudaError_t e;
  DeviceGuard guard;
  const int cur = guard.saved;
  if (on_device && dev != cur) {
    if ((e = cudaSetDevice(dev)) != cudaSuccess) {
      *info = cuda_fail(e, "set device");
      return;
    }
  }
  if (!on_device) dev = cur;
  DeviceState* ds = device_state(dev);
  std::lock_guard<std::mutex> sync_lk(ds->sync_mu);
  {
    std::lock_guard<std::mutex> lk(ds->mu);
    if ((e = ensure_device(ds)) != cudaSuccess) {
      *info = cuda_fail(e, "device setup");
      return;
    }
  }
  double* dA = A;
  int64_t ld = lda;
  bool pinned = false;
  if (!on_device) {
    // stage through a library-owned device buffer (ld rounded up for TMA alignment)
    const int64_t ldd = ((int64_t)n + 31) / 32 * 32;
    const size_t need = (size_t)ldd * n;
    if (ds->stage_elems < need) {
      if (ds->stage) cudaFree(ds->stage);
      ds->stage = nullptr;
      ds->stage_elems = 0;
      if ((e = cudaMalloc(&ds->stage, need * sizeof(double))) != cudaSuccess) {
        *info = cuda_fail(e, "staging buffer");
        return;
      }
      ds->stage_elems = need;
    }
    dA = ds->stage;
    ld = ldd;
    pinned = is_pinned_host(A);
    if (!pinned && (e = copy_triangle(dA, ld, A, lda, n, layout, cudaMemcpyHostToDevice, st)) != cudaSuccess) {
      *info = cuda_fail(e, "H2D");
      return;
    }
  }
  // pinned host matrix: the copies are nodes of the captured DAG, overlapped
  // with the factorization; pageable: staged before and after
  int r = pinned ? enqueue_potrf(dev, dA, n, ld, layout, ds->d_info, st, A, lda)
                 : enqueue_potrf(dev, dA, n, ld, layout, ds->d_info, st);
  if (r != 0) {
    *info = r;
    return;
  }
  if (!on_device && !pinned) {
    if (!ds->bounce && (e = cudaHostAlloc(&ds->bounce, 256 * 256 * sizeof(double), cudaHostAllocDefault)) != cudaSuccess) {
      *info = cuda_fail(e, "bounce buffer");
      return;
    }
    if ((e = copy_triangle(A, lda, dA, ld, n, layout, cudaMemcpyDeviceToHost, st, ds->bounce)) != cudaSuccess) {
      *info = cuda_fail(e, "D2H");
      return;
    }
  }
  if ((e = cudaMemcpyAsync(ds->h_info, ds->d_info, sizeof(int), cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
      (e = cudaStreamSynchronize(st)) != cudaSuccess) {
    *info = cuda_fail(e, "sync");
    return;
  }
  *info = *ds->h_info;
}

int relapack_dpotrf_async(char uplo, int n, double* A, int lda, int* d_info, relapack_stream_t stream) {
  int layout = 0;
  int ai = check_args(uplo, n, A, lda, &layout);
  if (ai != 0) return ai;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int dev = 0;
  if (n > 0 && !is_device_pointer(A, &dev)) {
    set_error("relapack_dpotrf_async: A is not a device pointer");
    return -3;
  }
  if (d_info == nullptr) return -5;
  if (n == 0) {
    cudaError_t e = cudaMemsetAsync(d_info, 0, sizeof(int), st);
    return e == cudaSuccess ? 0 : cuda_fail(e, "memset info");
  }
  DeviceGuard guard;
  if (dev != guard.saved) cudaSetDevice(dev);
  return enqueue_potrf(dev, A, n, lda, layout, d_info, st);
}

int relapack_dpotrf_batched(char uplo, int batch, const int* d_n, double* const* d_A, const int* d_lda, int* d_info,
                            relapack_stream_t stream) {
  int layout;
  if (uplo == 'L' || uplo == 'l')
    layout = kLayoutN;
  else if (uplo == 'U' || uplo == 'u')
    layout = kLayoutT;
  else
    return -1;
  if (batch < 0) return -2;
  if (batch == 0) return 0;
  cudaError_t e = launch_potf2_batched(layout, batch, d_n, d_A, d_lda, d_info, reinterpret_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "batched launch");
}

void relapack_dpotrf_blocked(const char* uplo, const int* n_, double* A, const int* lda_, int nb, int* info) {
  if (!info) return;
  if (!uplo || !n_ || !lda_) {
    *info = -1;
    return;
  }
  int layout = 0;
  const int n = *n_, lda = *lda_;
  int ai = check_args(*uplo, n, A, lda, &layout);
  if (ai != 0) {
    *info = ai;
    return;
  }
  if (n == 0) {
    *info = 0;
    return;
  }
  int dev = 0;
  if (!is_device_pointer(A, &dev)) {
    *info = -3;
    return;
  }
  if (nb < 16) {
    *info = -5;
    return;
  }
  DeviceGuard guard;
  if (dev != guard.saved) cudaSetDevice(dev);
  DeviceState* ds = device_state(dev);
  std::lock_guard<std::mutex> sync_lk(ds->sync_mu);
  cudaError_t e;
  {
    std::lock_guard<std::mutex> lk(ds->mu);
    if ((e = ensure_device(ds)) != cudaSuccess) {
      *info = cuda_fail(e, "device setup");
      return;
    }
  }
  cudaStream_t st = g_stream;
  const int r = enqueue_potrf(dev, A, n, lda, layout, ds->d_info, st, nullptr, 0, nb < n ? nb : n);
  if (r != 0) {
    *info = r;
    return;
  }
  if ((e = cudaMemcpyAsync(ds->h_info, ds->d_info, sizeof(int), cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
      (e = cudaStreamSynchronize(st)) != cudaSuccess) {
    *info = cuda_fail(e, "sync");
    return;
  }
  *info = *ds->h_info;
}

int relapack_batch_split(int batch, const int* n, int nranks, int* bounds) {
  if (batch < 0 || nranks < 1 || !bounds || (batch > 0 && !n)) return -1;
  // contiguous ranges balanced by the leading-term work sum n_b^3 / 3 (SURVEY
  // §8e: the batch is split across GPUs, no collective in the data path)
  std::vector<double> pre((size_t)batch + 1, 0.0);
  for (int b = 0; b < batch; ++b) {
    const double nb = n[b] > 0 ? (double)n[b] : 0.0;
    pre[b + 1] = pre[b] + nb * nb * nb;
  }
  bounds[0] = 0;
  int cur = 0;
  for (int r = 1; r < nranks; ++r) {
    const double target = pre[batch] * r / nranks;
    while (cur < batch && pre[cur + 1] <= target) ++cur;
    // the boundary closer to the target (ties: the earlier one)
    if (cur < batch && pre[cur + 1] - target < target - pre[cur]) ++cur;
    bounds[r] = cur > bounds[r - 1] ? cur : bounds[r - 1];
  }
  bounds[nranks] = batch;
  return 0;
}

void relapack_set_stream(relapack_stream_t stream) {
  g_stream = reinterpret_cast<cudaStream_t>(stream);
  g_stream_set = 1;
}

const char* relapack_last_error(void) {
  if (!g_last_error.empty()) return g_last_error.c_str();
  std::lock_guard<std::mutex> lk(g_err_mu);
  static thread_local std::string copy;
  copy = g_last_error_global;
  return copy.c_str();
}

void relapack_finalize(void) {
  std::lock_guard<std::mutex> lk(g_dev_mu);
  int cur = 0;
  cudaGetDevice(&cur);
  for (int d = 0; d < kMaxDevices; ++d) {
    DeviceState* ds = g_dev[d];
    if (!ds) continue;
    cudaSetDevice(d);
    {
      std::lock_guard<std::mutex> l2(ds->mu);
      ds->index.clear();
      ds->lru.clear();
      if (ds->stage) cudaFree(ds->stage);
      if (ds->d_info) cudaFree(ds->d_info);
      if (ds->h_info) cudaFreeHost(ds->h_info);
      if (ds->bounce) cudaFreeHost(ds->bounce);
      if (ds->capture) cudaStreamDestroy(ds->capture);
      if (ds->h2d) cudaStreamDestroy(ds->h2d);
      if (ds->d2h) cudaStreamDestroy(ds->d2h);
      if (ds->ev_start) cudaEventDestroy(ds->ev_start);
      if (ds->ev_done) cudaEventDestroy(ds->ev_done);
    }
    delete ds;
    g_dev[d] = nullptr;
  }
  cudaSetDevice(cur);
  release_batched_workspace();
}

int relapack_set_crossover(int c) {
  if (c < 16 || c > kPotf2Max) return -1;  // base case held in one SM's shared memory
  g_crossover.store(c);
  return 0;
}

int relapack_set_split_tile(int t) {
  if (t != 8 && t != 16 && t != 32 && t != 64 && t != 128) return -1;
  g_split_tile.store(t);
  return 0;
}

int relapack_set_graphs(int enabled) {
  g_graphs.store(enabled ? 1 : 0);
  return 0;
}

int relapack_get_crossover(void) { return current_params().crossover; }

int relapack_split_point(int n, int align) { return split_point(n, align); }

int relapack_plan_ledger(int n, int c, int T, int levels, double* flops_by_level, int* count) {
  if (n < 0 || c < 1 || T < 1 || levels < 0 || (levels > 0 && !flops_by_level)) return -1;
  PlanParams p;
  p.crossover = c;
  p.split_tile = T;
  p.trsm_base = trsm_base_cols();
  std::vector<PlanOp> ops;
  build_potrf_plan(n, p, ops);
  if (flops_by_level)
    for (int l = 0; l <= levels; ++l) flops_by_level[l] = 0.0;
  for (const PlanOp& op : ops) {
    if (!flops_by_level) break;
    if (op.kind == OP_POTF2)
      flops_by_level[levels] += op.flops;
    else if (op.level >= 1 && op.level <= levels)
      flops_by_level[op.level - 1] += op.flops;
  }
  if (count) *count = (int)ops.size();
  return plan_depth(n, p);
}

int relapack_plan_schedule(int n, int c, int T, int lookahead, int64_t* out, int max_ops, int* dep_off,
                           int* dep_idx, int max_deps) {
  if (n < 0 || c < 1 || T < 1 || max_ops < 0 || max_deps < 0) return -1;
  PlanParams p;
  p.crossover = c;
  p.split_tile = T;
  p.trsm_base = trsm_base_cols();
  p.lookahead = lookahead != 0;
  p.trsm_rows = current_params().trsm_rows;
  p.lookahead_depth = current_params().lookahead_depth;
  p.defer_b21 = current_params().defer_b21;
  p.b21_chunks = current_params().b21_chunks;
  std::vector<PlanOp> ops;
  build_potrf_plan(n, p, ops);
  const int cnt = (int)ops.size();
  if (out && cnt <= max_ops)
    for (int i = 0; i < cnt; ++i) {
      const PlanOp& o = ops[i];
      int64_t* w = out + 16 * i;
      w[0] = o.kind; w[1] = o.level; w[2] = o.c_i; w[3] = o.c_j; w[4] = o.a_i; w[5] = o.a_j; w[6] = o.b_i;
      w[7] = o.b_j; w[8] = o.m; w[9] = o.n; w[10] = o.k; w[11] = o.info_base; w[12] = o.c_buf; w[13] = o.a_buf;
      w[14] = o.b_buf; w[15] = o.deferred;
    }
  if (dep_off && cnt <= max_ops) {
    std::vector<std::vector<int>> deps;
    compute_deps(ops, deps);
    int tot = 0;
    for (int i = 0; i < cnt; ++i) {
      dep_off[i] = tot;
      for (int d : deps[i]) {
        if (dep_idx && tot < max_deps) dep_idx[tot] = d;
        ++tot;
      }
    }
    dep_off[cnt] = tot;
  }
  return cnt;
}

int relapack_profile_enable(int on) {
  g_prof_on.store(on ? 1 : 0);
  return 0;
}

int relapack_profile_read(int kind, double* ms_total, double* flops_total, int* launches) {
  if (kind < 0 || kind > 3) return -1;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  double ms = 0.0, fl = 0.0;
  int cnt = 0;
  for (const ProfRecord& r : g_prof) {
    if (r.kind != kind) continue;
    cudaEventSynchronize(r.stop);
    float t = 0.f;
    cudaEventElapsedTime(&t, r.start, r.stop);
    ms += t;
    fl += r.flops;
    ++cnt;
  }
  if (ms_total) *ms_total = ms;
  if (flops_total) *flops_total = fl;
  if (launches) *launches = cnt;
  return 0;
}

int relapack_trace_read(int max, double* out) { return max < 0 || !out ? -1 : trace_read(max, out); }

int relapack_profile_records(int max, double* out) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  int cnt = 0;
  for (const ProfRecord& r : g_prof) {
    if (cnt >= max) break;
    cudaEventSynchronize(r.stop);
    float t = 0.f;
    cudaEventElapsedTime(&t, r.start, r.stop);
    double* o = out + 7 * cnt;
    o[0] = r.kind; o[1] = r.m; o[2] = r.n; o[3] = r.k; o[4] = r.level; o[5] = r.flops; o[6] = t;
    ++cnt;
  }
  return cnt;
}

void relapack_profile_reset(void) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (ProfRecord& r : g_prof) {
    cudaEventSynchronize(r.stop);
    g_prof_pool.push_back(r.start);
    g_prof_pool.push_back(r.stop);
  }
  g_prof.clear();
}

const char* relapack_version(void) { return "relapack-b200 0.1 (sm_100a, DMMA FP64)"; }

}  // extern "C"
