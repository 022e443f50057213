// xdriver.cu — executor and C-ABI entry points of the other recursive
// operations (N1 dtrtri / blocked dtrtri, N3 dlauum / dpotri /
// dpotrs, N4 dgetrf).  A plan (xplan.cpp) is turned into kernel launches —
// the mixed-layout update kernel (update.cu) for every BLAS-3 step, the base
// kernels of xkernels.cu / potf2.cu for the leaves — captured once per
// (operation, shape, operands) into a CUDA graph whose edges are the plan's
// footprint dependencies, and replayed.  No CPU fallback.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <list>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/relapack.h"
#include "common.cuh"
#include "driver_internal.h"
#include "kernels.h"
#include "xkernels.h"
#include "xplan.h"

namespace relapack {

namespace {

constexpr int kIntMax = 0x7fffffff;

struct XBuffers {
  double* base[2] = {nullptr, nullptr};  // buffer 0 (matrix), buffer 1 (right-hand sides)
  int64_t ld[2] = {1, 1};
  int layout[2] = {kLayoutN, kLayoutN};  // logical -> memory layout of each buffer
  int* ipiv = nullptr;                   // buffer 2 (1-based pivots, indexed by row / column)
  int total_rows = 0, total_cols = 0;
  int cl_size = 0;  // getrf: CTAs per cluster of the panel-only leaves (0: cooperative leaves)
};

struct XOperand {
  double* p;
  int64_t ld;
  int layout;
};

XOperand resolve(const XBuffers& b, const XView& v) {
  const int bl = b.layout[v.buf];
  return XOperand{b.base[v.buf] + lv_off(bl, v.r0, v.c0, b.ld[v.buf]), b.ld[v.buf], bl ^ v.trans};
}

struct XExec {
  std::vector<XOp> ops;
  std::vector<UpdateOp> upd;
  std::vector<int> slot;  // getf2 workspace slot per op (-1 none)
  XBuffers bufs;
  int* d_info = nullptr;  // [0] stop flag / info, [1] getrf zero-pivot info (min), [2] pad
  double* splitk_ws = nullptr;
  int* splitk_cnt = nullptr;
  size_t cnt_bytes = 0;
  unsigned* bars = nullptr;
  size_t nbars = 0;
  double* cand = nullptr;  // per getf2 slot: 2G vals, 2G*kGetf2Max rows, 2*kGetf2Max diag rows
  int* cand_idx = nullptr;
  void* poll_ws = nullptr;  // epoch-stamped exchange records (shared by the panels)
  int sms = 148;
  int cl_size = 0;  // getrf cluster panels: CTAs per cluster
  int defer_ctas = 0;  // getrf lookahead: CTA cap of the deferred updates
  bool is_getrf = false, has_check = false;
  cudaGraphExec_t exec = nullptr;
  ~XExec() {
    if (exec) cudaGraphExecDestroy(exec);
    for (void* p : {(void*)d_info, (void*)splitk_ws, (void*)splitk_cnt, (void*)bars, (void*)cand, (void*)cand_idx,
                    poll_ws})
      if (p) cudaFree(p);
  }
};

constexpr size_t kCandDoubles = 2 * 160 + 2 * 160 * kGetf2Max + 2 * kGetf2Max;

// CTAs of a getrf panel: one per RELAPACK_GETF2_ROWS rows (default 32), at
// most one per SM — measured at n = 16384 (tools/experiments r2j / r2o): 256
// rows per CTA 277 ms, 128 231 ms, 64 (= one CTA per SM at the top) 215 ms:
// the per-CTA row work outweighs the cheaper barrier of fewer CTAs.
int getf2_grid(int m, int sms) {
  static const int rows = [] {
    const char* v = getenv("RELAPACK_GETF2_ROWS");
    const int r = v ? atoi(v) : 32;
    return r < 16 ? 16 : r;
  }();
  int g = (m + rows - 1) / rows;
  // shared memory holds the CTA's rows: at most ~700 rows of 32 columns
  g = std::max(g, (m + 699) / 700);
  return std::max(1, std::min(g, sms));
}

// Epoch-stamped panel exchange (RELAPACK_GETF2_POLL=1, opt-in): no grid
// barrier, every CTA polls the others' 16-byte records.  Measured alone
// (tools/experiments r4d): faster with few CTAs (G = 2: 104 vs 122 us per
// 32-column panel) but the G x G polling contends at G >= 128 (205 vs 149 us);
// getrf n = 16384 225 vs 195 ms.
bool getf2_poll() {
  static const bool v = [] {
    const char* e = getenv("RELAPACK_GETF2_POLL");
    return e && e[0] == '1';
  }();
  return v;
}
// one workspace for all panels of a plan (they run one after another):
// records for up to 160 CTAs
constexpr size_t kPollRecBytes = 2 * 160 * 16, kPollRowBytes = 2 * 160 * kGetf2Max * 16,
                 kPollDiagBytes = 2 * kGetf2Max * 16;

__global__ void k_xprologue(int* d_info, int check) {
  if (!check) d_info[0] = 0;
  d_info[1] = kIntMax;
  d_info[2] += 1;  // replay counter: the panels' exchange epochs are unique per replay
}

__global__ void k_xepilogue(int* d_info) {
  if (d_info[0] == 0 && d_info[1] != kIntMax) d_info[0] = d_info[1];
}

__global__ void k_xnop() {}

cudaError_t launch_xop(const XExec& x, size_t i, cudaStream_t st) {
  const XOp& o = x.ops[i];
  const XBuffers& b = x.bufs;
  // measurement only (wrong results): RELAPACK_GETRF_SKIP_DEFER=1 replaces the
  // deferred lookahead pieces by empty kernels — the time of the chain alone
  static const int skip_defer = getenv("RELAPACK_GETRF_SKIP_DEFER") ? atoi(getenv("RELAPACK_GETRF_SKIP_DEFER")) : 0;
  if (o.defer && skip_defer) {
    k_xnop<<<1, 32, 0, st>>>();
    return cudaGetLastError();
  }
  switch (o.kind) {
    case XK_GEMM:
      return launch_update(x.upd[i], st);
    case XK_TRI: {
      const XOperand T = resolve(b, o.a), B = resolve(b, o.c);
      XTriArgs a{T.p, T.ld, T.layout, B.p, B.ld, B.layout, o.m, o.k, o.mode, o.unit, o.alpha, x.d_info};
      return launch_tri_rows(a, st);
    }
    case XK_TRTI2:
    case XK_LAUU2: {
      const XOperand A = resolve(b, o.c);
      XBlockArgs a{A.p, A.ld, A.layout, o.n, o.unit, x.d_info};
      return o.kind == XK_TRTI2 ? launch_trti2(a, st) : launch_lauu2(a, st);
    }
    case XK_POTF2: {
      const XOperand A = resolve(b, o.c);
      return launch_potf2(A.p, A.ld, A.layout, o.n, x.d_info, o.info_base, st);
    }
    case XK_GETF2: {
      const XOperand P = resolve(b, o.c);
      if (o.mode == 1) {
        XGetf2ClArgs a{};
        a.P = P.p;
        a.ld = P.ld;
        a.m = o.m;
        a.w = o.n;
        a.rows_per_cta = (o.m + x.cl_size - 1) / x.cl_size;
        a.ipiv = b.ipiv + o.c.c0;
        a.pivot_base = o.c.r0 + 1;
        a.getrf_info = x.d_info + 1;
        a.info_base = o.info_base;
        a.d_info = x.d_info;
        return launch_getf2_cl(a, x.cl_size, st);
      }
      const int G = getf2_grid(o.m, x.sms);
      double* c = x.cand + (size_t)x.slot[i] * kCandDoubles;
      XGetf2Args a{};
      a.P = P.p;
      a.ld = P.ld;
      a.m = o.m;
      a.w = o.n;
      a.rows_per_cta = (o.m + G - 1) / G;
      a.ipiv = b.ipiv + o.c.c0;
      a.pivot_base = o.c.r0 + 1;
      a.getrf_info = x.d_info + 1;
      a.info_base = o.info_base;
      a.bar = x.bars + x.slot[i];
      a.cand_val = c;
      a.cand_rows = c + 2 * 160;
      a.diag_row = c + 2 * 160 + 2 * 160 * kGetf2Max;
      a.cand_idx = x.cand_idx + (size_t)x.slot[i] * 2 * 160;
      a.A0 = resolve(b, XView{o.c.buf, o.c.r0, 0, 0}).p;
      a.ncols = b.total_cols;
      a.c0 = o.c.c0;
      a.d_info = x.d_info;
      if (getf2_poll()) {
        a.poll = 1;
        a.epoch_base = (unsigned)(x.slot[i] & 1023) << 6;
        a.replay = reinterpret_cast<const unsigned*>(x.d_info + 2);
        a.prec = x.poll_ws;
        a.prow = static_cast<char*>(x.poll_ws) + kPollRecBytes;
        a.pdiag = static_cast<char*>(x.poll_ws) + kPollRecBytes + kPollRowBytes;
      }
      return launch_getf2(a, G, st);
    }
    case XK_PERM: {
      const XOperand A = resolve(b, o.c);
      XPermArgs a{A.p, A.ld, o.n, b.ipiv, o.k, o.m, o.c.r0 + 1, x.d_info};
      return launch_permute(a, st);
    }
    case XK_LASWP: {
      const XOperand A = resolve(b, XView{o.c.buf, 0, o.c.c0, 0});
      XLaswpArgs a{A.p, A.ld, o.n, b.ipiv, o.m, o.k, 1, x.d_info};
      return launch_laswp(a, st);
    }
    case XK_CHECK: {
      const XOperand A = resolve(b, XView{0, 0, 0, 0});
      return launch_diag_check(A.p, A.ld, A.layout, o.n, x.d_info, st);
    }
  }
  return cudaErrorInvalidValue;
}

int env_int_x(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

// getrf lookahead: the deferred updates (each a persistent grid capped below
// the SM count) one at a time, in the order the chain first needs them, so
// the SMs they leave free stay free for the windows.  An edge is only added
// forwards in plan order (the capture creates nodes in that order).
void serialize_deferred(const std::vector<XOp>& ops, std::vector<std::vector<int>>& deps) {
  const size_t n = ops.size();
  std::vector<int> first_use(n, kIntMax);
  for (size_t j = 0; j < n; ++j)
    for (int d : deps[j]) first_use[d] = std::min(first_use[d], (int)j);
  std::vector<int> dg;
  for (size_t i = 0; i < n; ++i)
    if (ops[i].defer && ops[i].kind == XK_GEMM) dg.push_back((int)i);
  std::stable_sort(dg.begin(), dg.end(), [&](int a, int b) { return first_use[a] < first_use[b]; });
  if (env_int_x("RELAPACK_GETRF_SERIAL", 1) == 0) return;
  for (size_t q = 1; q < dg.size(); ++q)
    if (dg[q - 1] < dg[q]) deps[dg[q]].push_back(dg[q - 1]);
}

// Update descriptors, split-K slots (as the factorization's: two split-K
// updates share a slot only if one is an ancestor of the other) and the
// getf2 workspaces.
cudaError_t setup_exec(XExec& x, const std::vector<uint64_t>& anc) {
  const size_t n = x.ops.size(), words = (n + 63) / 64;
  x.upd.assign(n, UpdateOp{});
  x.slot.assign(n, -1);
  int64_t ws = 0;
  int cnt = 0;
  std::vector<int> slot_last, slot_of(n, -1);
  int nget = 0;
  cudaError_t e;
  if ((e = cudaMalloc(&x.d_info, 4 * sizeof(int))) != cudaSuccess) return e;  // before the descriptors use it
  if ((e = cudaMemset(x.d_info, 0, 4 * sizeof(int))) != cudaSuccess) return e;   // [2]: the replay counter
  for (size_t i = 0; i < n; ++i) {
    const XOp& o = x.ops[i];
    if (o.kind == XK_GETF2 && o.mode == 0) x.slot[i] = nget++;
    if (o.kind != XK_GEMM) continue;
    const XOperand C = resolve(x.bufs, o.c), A = resolve(x.bufs, o.a), B = resolve(x.bufs, o.b);
    UpdateOp& u = x.upd[i];
    init_update(u, C.p, C.ld, C.layout, A.p, A.ld, A.layout, B.p, B.ld, B.layout, o.m, o.n, o.k, o.alpha, o.tri);
    u.args.d_info = x.d_info;
    if (o.defer) u.max_ctas = x.defer_ctas;  // persistent, leaves the window's SMs free
    const int ks = o.defer ? 1 : update_ksplit_for(u.args.M, u.args.N, u.args.K, u.args.tri != 0, u.tile);
    if (ks <= 1) continue;
    u.args.ksplit = ks;
    ws = std::max(ws, update_ws_elems(u.args.M, u.args.N, u.args.tri != 0, u.tile, ks));
    cnt = std::max(cnt, u.args.ntiles);
    int s = -1;
    for (size_t q = 0; q < slot_last.size() && s < 0; ++q) {
      const int l = slot_last[q];
      if (anc[i * words + l / 64] >> (l % 64) & 1) s = (int)q;
    }
    if (s < 0) {
      s = (int)slot_last.size();
      slot_last.push_back(0);
    }
    slot_last[s] = (int)i;
    slot_of[i] = s;
  }
  if (ws > 0) {
    const size_t nslots = slot_last.size();
    if ((e = cudaMalloc(&x.splitk_ws, nslots * ws * sizeof(double))) != cudaSuccess) return e;
    x.cnt_bytes = nslots * cnt * sizeof(int);
    if ((e = cudaMalloc(&x.splitk_cnt, x.cnt_bytes)) != cudaSuccess) return e;
    if ((e = cudaMemset(x.splitk_cnt, 0, x.cnt_bytes)) != cudaSuccess) return e;
    for (size_t i = 0; i < n; ++i) {
      if (slot_of[i] < 0) continue;
      x.upd[i].args.ws = x.splitk_ws + (size_t)slot_of[i] * ws;
      x.upd[i].args.counters = x.splitk_cnt + (size_t)slot_of[i] * cnt;
    }
  }
  if (nget > 0) {
    x.nbars = nget;
    if ((e = cudaMalloc(&x.bars, nget * sizeof(unsigned))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&x.cand, nget * kCandDoubles * sizeof(double))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&x.cand_idx, nget * 2 * 160 * sizeof(int))) != cudaSuccess) return e;
    const size_t pb = kPollRecBytes + kPollRowBytes + kPollDiagBytes;
    if ((e = cudaMalloc(&x.poll_ws, pb)) != cudaSuccess) return e;
    if ((e = cudaMemset(x.poll_ws, 0, pb)) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t run_prologue(const XExec& x, cudaStream_t st) {
  k_xprologue<<<1, 1, 0, st>>>(x.d_info, x.has_check ? 1 : 0);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && x.splitk_cnt) e = cudaMemsetAsync(x.splitk_cnt, 0, x.cnt_bytes, st);
  if (e == cudaSuccess && x.bars) e = cudaMemsetAsync(x.bars, 0, x.nbars * sizeof(unsigned), st);
  return e;
}

cudaError_t capture(const XExec& x, const std::vector<std::vector<int>>& deps, cudaStream_t st) {
  cudaError_t e = run_prologue(x, st);
  if (e != cudaSuccess) return e;
  cudaStreamCaptureStatus cs;
  const cudaGraphNode_t* cur = nullptr;
  size_t ncur = 0;
  if ((e = cudaStreamGetCaptureInfo(st, &cs, nullptr, nullptr, &cur, &ncur)) != cudaSuccess) return e;
  if (ncur != 1) return cudaErrorStreamCaptureInvalidated;
  const cudaGraphNode_t root = cur[0];
  std::vector<cudaGraphNode_t> nodes(x.ops.size(), nullptr), want;
  std::vector<char> has_succ(x.ops.size(), 0);
  for (size_t i = 0; i < x.ops.size(); ++i) {
    want.clear();
    for (int d : deps[i]) {
      want.push_back(nodes[d]);
      has_succ[d] = 1;
    }
    if (want.empty()) want.push_back(root);
    if ((e = cudaStreamUpdateCaptureDependencies(st, want.data(), want.size(), cudaStreamSetCaptureDependencies)) !=
        cudaSuccess)
      return e;
    if ((e = launch_xop(x, i, st)) != cudaSuccess) return e;
    if ((e = cudaStreamGetCaptureInfo(st, &cs, nullptr, nullptr, &cur, &ncur)) != cudaSuccess) return e;
    if (ncur != 1) return cudaErrorStreamCaptureInvalidated;
    nodes[i] = cur[0];
  }
  bool any_defer = false;
  for (const XOp& o : x.ops) any_defer |= o.defer != 0;
  if (any_defer) {  // deferred pieces lowest, everything else (the windows' chain) highest
    std::vector<char> cls(x.ops.size(), 0);
    for (size_t i = 0; i < x.ops.size(); ++i) cls[i] = x.ops[i].defer ? 2 : 0;
    if ((e = set_node_priorities(nodes, cls)) != cudaSuccess) return e;
  }
  want.clear();
  for (size_t i = 0; i < x.ops.size(); ++i)
    if (!has_succ[i]) want.push_back(nodes[i]);
  if (want.empty()) want.push_back(root);
  if ((e = cudaStreamUpdateCaptureDependencies(st, want.data(), want.size(), cudaStreamSetCaptureDependencies)) !=
      cudaSuccess)
    return e;
  k_xepilogue<<<1, 1, 0, st>>>(x.d_info);
  return cudaGetLastError();
}

// Profiling (bench.py's per-kernel-class breakdown of these plans): with
// relapack_xprofile_enable(1) plans run serially in plan order with CUDA
// events around every launch, accumulated per op kind.
struct XProfRec {
  cudaEvent_t a, b;
  int kind, level;
  double flops;
};
std::mutex g_xprof_mu;
std::vector<XProfRec> g_xprof;
int g_xprof_on = 0;

cudaError_t run_serial(const XExec& x, cudaStream_t st) {
  cudaError_t e = run_prologue(x, st);
  for (size_t i = 0; i < x.ops.size() && e == cudaSuccess; ++i) {
    XProfRec r{nullptr, nullptr, (int)x.ops[i].kind, x.ops[i].level, x.ops[i].flops};
    if (g_xprof_on) {
      cudaEventCreate(&r.a);
      cudaEventCreate(&r.b);
      cudaEventRecord(r.a, st);
    }
    e = launch_xop(x, i, st);
    if (g_xprof_on) {
      cudaEventRecord(r.b, st);
      std::lock_guard<std::mutex> lk(g_xprof_mu);
      g_xprof.push_back(r);
    }
  }
  if (e == cudaSuccess) {
    k_xepilogue<<<1, 1, 0, st>>>(x.d_info);
    e = cudaGetLastError();
  }
  return e;
}

// ---------------------------------------------------------------- plan cache
struct XCache {
  std::mutex mu;
  std::list<std::pair<std::string, std::unique_ptr<XExec>>> lru;
  cudaStream_t capture = nullptr;
  bool configured = false;
};
XCache g_xcache[kMaxDevices];

bool x_graphs() {
  const char* v = getenv("RELAPACK_GRAPH");
  return !(v && v[0] == '0');
}


// Build (or fetch) and launch the plan; returns 0 or an error code.
int x_run(const std::string& key, const std::vector<XOp>& ops_in, const XBuffers& bufs, bool is_getrf,
          bool has_check, cudaStream_t st, int* info_out) {
  int dev = 0;
  cudaGetDevice(&dev);
  XCache& c = g_xcache[dev];
  std::lock_guard<std::mutex> lk(c.mu);
  cudaError_t e;
  if (!c.configured) {
    if ((e = configure_kernels()) != cudaSuccess) return cuda_fail(e, "configure");
    if ((e = configure_xkernels()) != cudaSuccess) return cuda_fail(e, "configure x");
    if ((e = cudaStreamCreateWithFlags(&c.capture, cudaStreamNonBlocking)) != cudaSuccess)
      return cuda_fail(e, "capture stream");
    c.configured = true;
  }
  const bool graphs = x_graphs() && !g_xprof_on;
  const std::string full = key + (graphs ? " g1" : " g0");
  XExec* x = nullptr;
  for (auto it = c.lru.begin(); it != c.lru.end(); ++it)
    if (it->first == full) {
      c.lru.splice(c.lru.begin(), c.lru, it);
      x = c.lru.front().second.get();
      break;
    }
  if (!x) {
    auto p = std::make_unique<XExec>();
    p->ops = ops_in;
    p->bufs = bufs;
    p->is_getrf = is_getrf;
    p->has_check = has_check;
    p->cl_size = is_getrf ? bufs.cl_size : 0;
    cudaDeviceGetAttribute(&p->sms, cudaDevAttrMultiProcessorCount, dev);
    std::vector<std::vector<int>> deps;
    std::vector<uint64_t> anc;
    xplan_deps(p->ops, bufs.total_rows, deps, &anc);
    {  // RELAPACK_GETRF_RESERVE < 0: deferred updates one tile per CTA (no cap; yield SMs tile by tile)
      const int rs = env_int_x("RELAPACK_GETRF_RESERVE", 16);
      p->defer_ctas = rs < 0 ? 0 : std::max(1, p->sms - std::max(p->cl_size, rs));
    }
    for (size_t i = 0; i < p->ops.size(); ++i)
      if (p->ops[i].after >= 0 && p->ops[i].after < (int)i) deps[i].push_back(p->ops[i].after);
    serialize_deferred(p->ops, deps);
    if ((e = setup_exec(*p, anc)) != cudaSuccess) return cuda_fail(e, "x workspace");
    if (graphs) {
      cudaGraph_t g = nullptr;
      if ((e = cudaStreamBeginCapture(c.capture, cudaStreamCaptureModeThreadLocal)) != cudaSuccess)
        return cuda_fail(e, "begin capture");
      const cudaError_t er = capture(*p, deps, c.capture);
      e = cudaStreamEndCapture(c.capture, &g);
      if (er != cudaSuccess) {
        if (g) cudaGraphDestroy(g);
        return cuda_fail(er, "x capture");
      }
      if (e != cudaSuccess) return cuda_fail(e, "end capture");
      e = cudaGraphInstantiateWithFlags(&p->exec, g, 0);
      cudaGraphDestroy(g);
      if (e != cudaSuccess) return cuda_fail(e, "graph instantiate");
    }
    c.lru.emplace_front(full, std::move(p));
    x = c.lru.front().second.get();
    while (c.lru.size() > 16) c.lru.pop_back();
  }
  e = graphs ? cudaGraphLaunch(x->exec, st) : run_serial(*x, st);
  if (e != cudaSuccess) return cuda_fail(e, "x launch");
  if (info_out) {
    int h = 0;
    if ((e = cudaMemcpyAsync(&h, x->d_info, sizeof(int), cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (e = cudaStreamSynchronize(st)) != cudaSuccess)
      return cuda_fail(e, "x sync");
    *info_out = h;
  }
  return 0;
}

int parse_uplo_layout(const char* uplo) {
  if (!uplo) return -1;
  if (*uplo == 'L' || *uplo == 'l') return kLayoutN;
  if (*uplo == 'U' || *uplo == 'u') return kLayoutT;
  return -1;
}

bool device_ptr(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

std::string ptr_key(const void* p) {
  char b[32];
  snprintf(b, sizeof(b), "%p", p);
  return b;
}

XParams x_params() {
  XParams p;
  const char* v = getenv("RELAPACK_XBASE");
  if (v) p.tri_base = std::max(8, std::min(kTriMax, atoi(v)));
  v = getenv("RELAPACK_GETRF_BASE");
  if (v) p.getrf_base = std::max(1, std::min(kGetf2Max, atoi(v)));
  p.potrs_cols = std::max(0, env_int_x("RELAPACK_POTRS_COLS", p.potrs_cols));
  p.tri_rows = std::max(0, env_int_x("RELAPACK_TRI_ROWS", 0));
  p.trtri_order = env_int_x("RELAPACK_TRTRI_ORDER", p.trtri_order) == 1 ? 1 : 0;
  return p;
}

std::string params_key(const XParams& p) {
  char b[128];
  snprintf(b, sizeof(b), " tb%d st%d gb%d cl%d pc%d tr%d to%d", p.tri_base, p.split_tile, p.getrf_base,
           p.getf2_cluster, p.potrs_cols, p.tri_rows, p.trtri_order);
  return b;
}

// Triangular operations on the L-view of an n x n device matrix.
int tri_common(const char* what, const char* uplo, int n, double* A, int lda, const XParams& p,
               const std::vector<XOp>& ops, bool check, const std::string& extra, int* info) {
  const int layout = parse_uplo_layout(uplo);
  XBuffers b;
  b.base[0] = A;
  b.ld[0] = lda;
  b.layout[0] = layout;
  b.total_rows = n;
  const std::string key = std::string(what) + " n" + std::to_string(n) + " ld" + std::to_string(lda) + " l" +
                          std::to_string(layout) + " A" + ptr_key(A) + params_key(p) + extra;
  std::vector<XOp> all;
  if (check) {
    XOp c;
    c.kind = XK_CHECK;
    c.n = n;
    all.push_back(c);
  }
  all.insert(all.end(), ops.begin(), ops.end());
  return x_run(key, all, b, false, check, current_stream_or(nullptr), info);
}

int check_tri_args(const char* uplo, const char* diag, const int* n, const double* A, const int* lda, bool need_diag) {
  if (parse_uplo_layout(uplo) < 0) return -1;
  if (need_diag && !(diag && (*diag == 'N' || *diag == 'n' || *diag == 'U' || *diag == 'u'))) return -2;
  if (!n || *n < 0) return need_diag ? -3 : -2;
  if (*n > 0 && (!A || !device_ptr(A))) return need_diag ? -4 : -3;
  if (!lda || *lda < std::max(1, *n)) return need_diag ? -5 : -4;
  return 0;
}

}  // namespace

}  // namespace relapack

using namespace relapack;

extern "C" {

void relapack_dtrtri(const char* uplo, const char* diag, const int* n, double* A, const int* lda, int* info) {
  if (!info) return;
  if ((*info = check_tri_args(uplo, diag, n, A, lda, true)) != 0 || *n == 0) return;
  const XParams p = x_params();
  const int unit = (*diag == 'U' || *diag == 'u');
  std::vector<XOp> ops;
  xplan_trtri(ops, p, 0, *n, unit, 0);
  const int r = tri_common("trtri", uplo, *n, A, *lda, p, ops, !unit, unit ? " unit" : "", info);
  if (r != 0) *info = r;
}

void relapack_dtrtri_blocked(const char* uplo, const char* diag, const int* n, double* A, const int* lda, int nb,
                             int* info) {
  if (!info) return;
  if ((*info = check_tri_args(uplo, diag, n, A, lda, true)) != 0 || *n == 0) return;
  if (nb < 1) {
    *info = -6;
    return;
  }
  const XParams p = x_params();
  const int unit = (*diag == 'U' || *diag == 'u');
  std::vector<XOp> ops;
  xplan_trtri_blocked(ops, p, *n, nb, unit);
  const int r = tri_common("trtri_blocked", uplo, *n, A, *lda, p, ops, !unit,
                     std::string(unit ? " unit" : "") + " nb" + std::to_string(nb), info);
  if (r != 0) *info = r;
}

void relapack_dlauum(const char* uplo, const int* n, double* A, const int* lda, int* info) {
  if (!info) return;
  if ((*info = check_tri_args(uplo, nullptr, n, A, lda, false)) != 0 || *n == 0) return;
  const XParams p = x_params();
  std::vector<XOp> ops;
  xplan_lauum(ops, p, 0, *n, 0);
  const int r = tri_common("lauum", uplo, *n, A, *lda, p, ops, false, "", info);
  if (r != 0) *info = r;
}

void relapack_dpotri(const char* uplo, const int* n, double* A, const int* lda, int* info) {
  if (!info) return;
  if ((*info = check_tri_args(uplo, nullptr, n, A, lda, false)) != 0 || *n == 0) return;
  const XParams p = x_params();
  std::vector<XOp> ops;
  xplan_trtri(ops, p, 0, *n, 0, 0);
  xplan_lauum(ops, p, 0, *n, 0);
  const int r = tri_common("potri", uplo, *n, A, *lda, p, ops, true, "", info);
  if (r != 0) *info = r;
}

void relapack_dpotrs(const char* uplo, const int* n, const int* nrhs, const double* A, const int* lda, double* B,
                     const int* ldb, int* info) {
  if (!info) return;
  const int layout = parse_uplo_layout(uplo);
  if (layout < 0) { *info = -1; return; }
  if (!n || *n < 0) { *info = -2; return; }
  if (!nrhs || *nrhs < 0) { *info = -3; return; }
  if (*n > 0 && (!A || !device_ptr(A))) { *info = -4; return; }
  if (!lda || *lda < std::max(1, *n)) { *info = -5; return; }
  if (*n > 0 && *nrhs > 0 && (!B || !device_ptr(B))) { *info = -6; return; }
  if (!ldb || *ldb < std::max(1, *n)) { *info = -7; return; }
  *info = 0;
  if (*n == 0 || *nrhs == 0) return;
  const XParams p = x_params();
  std::vector<XOp> ops;
  xplan_potrs(ops, p, *n, *nrhs);
  XBuffers b;
  b.base[0] = const_cast<double*>(A);
  b.ld[0] = *lda;
  b.layout[0] = layout;
  b.base[1] = B;
  b.ld[1] = *ldb;
  b.layout[1] = kLayoutN;
  b.total_rows = *n;
  const std::string key = "potrs n" + std::to_string(*n) + " r" + std::to_string(*nrhs) + " ld" +
                          std::to_string(*lda) + " ldb" + std::to_string(*ldb) + " l" + std::to_string(layout) +
                          " A" + ptr_key(A) + " B" + ptr_key(B) + params_key(p);
  int r = x_run(key, ops, b, false, false, current_stream_or(nullptr), info);
  if (r != 0) *info = r;
}

void relapack_dgetrf(const int* m, const int* n, double* A, const int* lda, int* ipiv, int* info) {
  if (!info) return;
  if (!m || *m < 0) { *info = -1; return; }
  if (!n || *n < 0) { *info = -2; return; }
  if (*m > 0 && *n > 0 && (!A || !device_ptr(A))) { *info = -3; return; }
  if (!lda || *lda < std::max(1, *m)) { *info = -4; return; }
  if (std::min(*m, *n) > 0 && (!ipiv || !device_ptr(ipiv))) { *info = -5; return; }
  *info = 0;
  if (*m == 0 || *n == 0) return;
  XParams p = x_params();
  p.getrf_cols = *n;
  std::vector<XOp> ops;
  // lookahead plan (RELAPACK_GETRF_LA, window RELAPACK_GETRF_WINDOW): panel-only
  // cluster leaves for every panel height, else the plain recursion
  const int la = env_int_x("RELAPACK_GETRF_LA", 0);
  const int cl = la ? getf2_cluster_size(env_int_x("RELAPACK_GETF2_CLUSTER", 16)) : 0;
  if (la && cl > 0 && (*m + cl - 1) / cl <= kGetf2ClRows8) {
    p.getf2_cluster = cl;
    p.getrf_window = std::max(8, env_int_x("RELAPACK_GETRF_WINDOW", 256));
    p.getrf_first_piece = env_int_x("RELAPACK_GETRF_P0FIRST", 0);
    xplan_getrf_la(ops, p, *m, *n);
  } else {
    p.getf2_cluster = getf2_cluster_caps();
    xplan_getrf(ops, p, 0, 0, *m, *n, 0);
  }
  XBuffers b;
  b.base[0] = A;
  b.ld[0] = *lda;
  b.layout[0] = kLayoutN;
  b.ipiv = ipiv;
  b.total_rows = *m;
  b.total_cols = *n;
  b.cl_size = p.getf2_cluster;
  const std::string key = "getrf m" + std::to_string(*m) + " n" + std::to_string(*n) + " ld" + std::to_string(*lda) +
                          " A" + ptr_key(A) + " P" + ptr_key(ipiv) + params_key(p) + " la" + std::to_string(la) +
                          " w" + std::to_string(p.getrf_window) + " pf" + std::to_string(p.getrf_first_piece) + " rs" +
                          std::to_string(env_int_x("RELAPACK_GETRF_RESERVE", 16)) + " se" +
                          std::to_string(env_int_x("RELAPACK_GETRF_SERIAL", 1));
  int r = x_run(key, ops, b, true, false, current_stream_or(nullptr), info);
  if (r != 0) *info = r;
}

int relapack_xprofile_enable(int on) {
  g_xprof_on = on ? 1 : 0;
  return 0;
}

int relapack_xprofile_read(int kind, double* ms_total, double* flops_total, int* launches) {
  std::lock_guard<std::mutex> lk(g_xprof_mu);
  double ms = 0, fl = 0;
  int cnt = 0;
  for (const XProfRec& r : g_xprof) {
    if (r.kind != kind) continue;
    float t = 0.f;
    cudaEventSynchronize(r.b);
    cudaEventElapsedTime(&t, r.a, r.b);
    ms += t;
    fl += r.flops;
    ++cnt;
  }
  if (ms_total) *ms_total = ms;
  if (flops_total) *flops_total = fl;
  if (launches) *launches = cnt;
  return 0;
}

int relapack_xprofile_records(int max, double* out) {
  std::lock_guard<std::mutex> lk(g_xprof_mu);
  int cnt = 0;
  for (const XProfRec& r : g_xprof) {
    if (cnt >= max) break;
    float t = 0.f;
    cudaEventSynchronize(r.b);
    cudaEventElapsedTime(&t, r.a, r.b);
    double* o = out + 4 * cnt;
    o[0] = r.kind;
    o[1] = r.level;
    o[2] = r.flops;
    o[3] = t;
    ++cnt;
  }
  return cnt;
}

void relapack_xprofile_reset(void) {
  std::lock_guard<std::mutex> lk(g_xprof_mu);
  for (XProfRec& r : g_xprof) {
    cudaEventSynchronize(r.b);
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  g_xprof.clear();
}

int relapack_xplan_count(int op, int n, int nb, int* kinds_out, int max_kinds, double* flops_out) {
  // host-only introspection of the §8(f) plans: op 0 trtri, 1 trtri_blocked,
  // 2 lauum, 3 potri, 4 potrs (nrhs = nb), 5 getrf (square), 6 getrf with lookahead (window nb)
  if (n < 0) return -1;
  XParams p;
  p.potrs_cols = x_params().potrs_cols;  // the panel knobs as the executor reads them
  p.tri_rows = x_params().tri_rows;
  p.trtri_order = x_params().trtri_order;
  std::vector<XOp> ops;
  switch (op) {
    case 0: xplan_trtri(ops, p, 0, n, 0, 0); break;
    case 1: if (nb < 1) return -1; xplan_trtri_blocked(ops, p, n, nb, 0); break;
    case 2: xplan_lauum(ops, p, 0, n, 0); break;
    case 3: xplan_trtri(ops, p, 0, n, 0, 0); xplan_lauum(ops, p, 0, n, 0); break;
    case 4: xplan_potrs(ops, p, n, nb); break;
    case 5: xplan_getrf(ops, p, 0, 0, n, n, 0); break;
    case 6:  // getrf lookahead plan, 16-CTA cluster leaves, window nb (0: 256)
      p.getf2_cluster = 16;
      p.getrf_cols = n;
      if (nb > 0) p.getrf_window = nb;
      if ((n + 15) / 16 > kGetf2ClRows8) return -1;
      xplan_getrf_la(ops, p, n, n);
      break;
    default: return -1;
  }
  double fl = 0.0;
  for (size_t i = 0; i < ops.size(); ++i) {
    fl += ops[i].flops;
    if (kinds_out && (int)i < max_kinds) kinds_out[i] = ops[i].kind;
  }
  if (flops_out) *flops_out = fl;
  return (int)ops.size();
}

}  // extern "C"
