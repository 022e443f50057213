// batched.cu — K2: independent small Cholesky factorizations (CFG[4]: 131072
// SPD matrices, n in {16, 32, 48, 64}; SPEC potf2 S:219-227 per matrix, one
// call, per-matrix info).
//
// The batch is HBM-bound in aggregate but every single factorization is a
// latency-bound chain (one pivot -> rsqrt -> update per column), so the design
// keeps the load of the next matrix in flight while the current one is
// factored, and keeps enough matrices per SM to cover the chains:
//  * a bucketing pass sorts the matrices into size classes NMAX in
//    {16, 32, 48, 64} (validating n / lda and writing info -2 / -4 on the way);
//    its lists live in a library-owned workspace (no per-call allocation);
//  * one persistent kernel per class, one WARP per matrix, grid-stride over the
//    class list, no CTA-wide barriers; each warp owns TWO shared-memory slots:
//    while it factors matrix k in one slot, matrix k+1 streams into the other
//    with bulk async copies (cp.async.bulk, one per column of the lower
//    triangle, completion on an mbarrier);
//  * a slot holds the lower triangle "even-packed": column j of L (layout N)
//    or row i of L (layout T) starts at the even index below/at it, so every
//    bulk copy is 16-byte aligned and a multiple of 16 bytes; the slot is padded
//    with the identity beyond n, so every loop runs at the compile-time size
//    NMAX (the factor of [A 0; 0 I] is [L 0; 0 I]);
//  * panels of 8 columns are factored in registers (lane l holds rows l and
//    l+32; pivot and l_kj broadcast by shuffles; rsqrt chain as in potf2.cu),
//    the rank-8 trailing update runs on the FP64 tensor cores (DMMA.8x8x4 on
//    8x8 tiles of the lower triangle, K = 8), all tiles of a tile row in flight;
//  * odd n, odd lda or a base not 16-byte aligned take a plain-load path into
//    the same slot layout.
#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "chol_regs.cuh"
#include "common.cuh"
#include "kernels.h"

#ifndef RELAPACK_BATCH_MODE
#define RELAPACK_BATCH_MODE 0
#endif

namespace relapack {

#ifndef RELAPACK_BATCH_DESC_AHEAD
#define RELAPACK_BATCH_DESC_AHEAD 1
#endif
#ifndef RELAPACK_BATCH_SQUARE
#define RELAPACK_BATCH_SQUARE 1
#endif

namespace {

constexpr int kPanel = 8;
constexpr int kClasses = 4;  // NMAX = 16 (c + 1)

template <int NMAX, int LAYOUT>
struct BC {
  static constexpr int TN = NMAX / 8;
  static constexpr int WPC = 4;  // warps (matrices in flight) per CTA
  // CTAs per SM the register budget is sized for: more warps in flight hide
  // the per-matrix column chain (compile-time knobs RELAPACK_BATCH_MINB<NMAX>)
#ifndef RELAPACK_BATCH_MINB16
#define RELAPACK_BATCH_MINB16 4
#endif
#ifndef RELAPACK_BATCH_MINB32
#define RELAPACK_BATCH_MINB32 3
#endif
#ifndef RELAPACK_BATCH_MINB48
#define RELAPACK_BATCH_MINB48 3
#endif
#ifndef RELAPACK_BATCH_MINB64
#define RELAPACK_BATCH_MINB64 2
#endif
  static constexpr int MIN_BLOCKS =
      NMAX == 64 ? RELAPACK_BATCH_MINB64 : NMAX == 48 ? RELAPACK_BATCH_MINB48 : NMAX == 32 ? RELAPACK_BATCH_MINB32 : RELAPACK_BATCH_MINB16;
  // even-packed lower triangle: NMAX (NMAX/2 + 1) doubles per prefetch slot;
  // n <= 32, uplo L: room for the whole column-major square at stride SQ_LD
  // instead (the square path below)
  static constexpr bool SQ = NMAX <= 32 && LAYOUT == kLayoutN && RELAPACK_BATCH_SQUARE;
  static constexpr int SQ_LD = NMAX + 2;  // 16-byte aligned columns; DMMA-layout reads 2-way (the minimum)
  static constexpr int SLOT = SQ && NMAX * SQ_LD > NMAX * (NMAX / 2 + 1) ? NMAX * SQ_LD : NMAX * (NMAX / 2 + 1);
  static constexpr size_t SMEM = sizeof(double) * SLOT * WPC;
  // layout N: column j of L from row (j & ~1), columns back to back;
  // layout T: row i of L, columns 0 .. (i | 1), rows back to back.
  static __device__ __forceinline__ int base(int x) {
    const int m = x >> 1;
    if (LAYOUT == kLayoutN) return 2 * (m * NMAX - m * (m - 1)) + ((x & 1) ? NMAX - 2 * m : 0);
    return 2 * m * (m + 1) + ((x & 1) ? 2 * m + 2 : 0);
  }
  // offset of L(i, j), i >= j
  static __device__ __forceinline__ int off(int i, int j) {
    return LAYOUT == kLayoutN ? base(j) + i - (j & ~1) : base(i) + j;
  }
};

// x, hidden from loop-invariant code motion
__device__ __forceinline__ int opaque(int x) {
  int z;
  asm volatile("mov.u32 %0, 0;" : "=r"(z));
  return x + z;
}

// Pass 1: validate, bucket by size class (list[c * batch + pos]).
__global__ void k_bucket(int batch, const int* __restrict__ d_n, const int* __restrict__ d_lda, int* d_info,
                         int* counts, int* lists) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  const int n = d_n[b], lda = d_lda[b];
  if (n < 0 || n > RELAPACK_BATCH_NMAX_) {
    d_info[b] = -2;
    return;
  }
  if (lda < (n > 1 ? n : 1)) {
    d_info[b] = -4;
    return;
  }
  if (n == 0) {
    d_info[b] = 0;
    return;
  }
  const int c = (n - 1) / 16;
  const int pos = atomicAdd(&counts[c], 1);
  lists[(size_t)c * batch + pos] = b;
}

// 1-D bulk async copy global -> shared, completion (bytes) on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Small full-class matrices stored densely (n == lda == NMAX <= 32, uplo L):
// the per-column bulk copies would be 8..256 bytes each, so the lanes instead
// move the columns' lower parts as 16-byte cp.async chunks (a few per lane).
template <int NMAX, int LAYOUT>
__device__ __forceinline__ bool square_ok(const double* A, int n, int64_t lda) {
  return BC<NMAX, LAYOUT>::SQ && n == NMAX && lda == NMAX && (reinterpret_cast<uintptr_t>(A) & 15) == 0;
}

template <int NMAX, int LAYOUT>
__device__ __forceinline__ bool bulk_ok(const double* A, int n, int64_t lda) {
  return !square_ok<NMAX, LAYOUT>(A, n, lda) && ((n & 1) == 0) && ((lda & 1) == 0) &&
         ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
}

// Start the load of matrix (A, n, lda) into slot s: one bulk copy per column
// (layout N) / row (layout T) of L, issued by the lanes; lane 0 registers the
// byte count first.  Plain-load matrices (see bulk_ok) are loaded at wait time.
template <int NMAX, int LAYOUT>
__device__ __forceinline__ void issue_load(double* s, uint64_t* bar, const double* A, int n, int64_t lda, int lane) {
  using C = BC<NMAX, LAYOUT>;
  if (square_ok<NMAX, LAYOUT>(A, n, lda)) {
    constexpr int CH = NMAX / 2;  // 16-byte chunks per column
    __syncwarp();                 // every lane has read the previous matrix out of the slot
#pragma unroll
    for (int k = lane; k < NMAX * CH; k += 32) {
      const int col = k / CH, r2 = 2 * (k % CH);
      if (r2 + 1 < col) continue;  // wholly above the diagonal
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(s + col * C::SQ_LD + r2)),
                   "l"(A + col * NMAX + r2)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    return;
  }
  if (!bulk_ok<NMAX, LAYOUT>(A, n, lda)) return;
  fence_proxy_async_smem();  // this warp's earlier generic accesses of the slot precede the async writes
  if (lane == 0) mbar_arrive_expect_tx(bar, (uint32_t)(8 * n * (n / 2 + 1)));
  __syncwarp();
  for (int x = lane; x < n; x += 32) {
    if (LAYOUT == kLayoutN) {
      const int js = x & ~1;  // column x of L: rows js .. n-1
      bulk_g2s(s + C::base(x), A + x * lda + js, (uint32_t)(8 * (n - js)), bar);
    } else {
      const int cnt = (x + 2) & ~1;  // row x of L = column x of A: elements 0 .. cnt-1 (cnt <= n, n even)
      bulk_g2s(s + C::base(x), A + x * lda, (uint32_t)(8 * cnt), bar);
    }
  }
}

// Plain-load matrices (odd n or lda, unaligned base): the lanes copy the
// lower triangle into the slot (same layout as the bulk copies), so the
// register load below has one source.  Not unrolled: a rare path kept small.
template <int NMAX, int LAYOUT>
__device__ __forceinline__ void plain_to_slot(double* s, const double* A, int n, int64_t lda, int lane) {
  using C = BC<NMAX, LAYOUT>;
  __syncwarp();  // every lane has read the previous matrix out of the slot
#pragma unroll 1
  for (int c = 0; c < n; ++c)
    for (int r = c + lane; r < n; r += 32) s[C::off(r, c)] = A[lv_off(LAYOUT, r, c, lda)];
  __syncwarp();
}

// Registers <- the matrix from the slot; identity beyond n, 0 above the
// diagonal.  (One source only: the kernel's code size matters — the fully
// unrolled 64-class kernel is instruction-cache bound.)
template <int NMAX, int LAYOUT>
__device__ __forceinline__ void load_regs(double (&v)[RegTri<NMAX / 8>::NT][2], const double* s, bool square, int n,
                                          int lane) {
  using C = BC<NMAX, LAYOUT>;
  using T = RegTri<NMAX / 8>;
  const int g = lane >> 2, t = lane & 3;
  if (C::SQ && square) {
#pragma unroll
    for (int i = 0; i < C::TN; ++i)
#pragma unroll
      for (int k = 0; k <= i; ++k)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int r = 8 * i + g, c = 8 * k + 2 * t + q;
          v[T::id(i, k)][q] = r >= c ? s[r + c * C::SQ_LD] : (r == c ? 1.0 : 0.0);
        }
  } else {
#pragma unroll
    for (int i = 0; i < C::TN; ++i)
#pragma unroll
      for (int k = 0; k <= i; ++k)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int r = 8 * i + g, c = 8 * k + 2 * t + q;
          v[T::id(i, k)][q] = (r < n && c < n && r >= c) ? s[C::off(r, c)] : (r == c ? 1.0 : 0.0);
        }
  }
}

template <int NMAX, int LAYOUT>
__global__ void __launch_bounds__(BC<NMAX, LAYOUT>::WPC * 32, BC<NMAX, LAYOUT>::MIN_BLOCKS)
    k_batched_cls(int batch, const int* counts, const int* lists, double* const* d_A, const int* d_n,
                  const int* d_lda, int* d_info, int stagger_ns) {
  using C = BC<NMAX, LAYOUT>;
  using T = RegTri<NMAX / 8>;
  constexpr int WPC = C::WPC;
  extern __shared__ __align__(16) double smem_b[];
  __shared__ uint64_t bars[WPC];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  double* const slot = smem_b + warp * C::SLOT;
  uint64_t* bar = &bars[warp];
  if (lane == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  __syncwarp();
  const int cls = NMAX / 16 - 1;
  const int count = counts[cls];
  const int* list = lists + (size_t)cls * batch;
  const int stride = gridDim.x * WPC;
  int pos = blockIdx.x * WPC + warp;
  if (pos >= count) return;
  int b = list[pos];
  int n = d_n[b];
  int64_t lda = d_lda[b];
  double* A = d_A[b];
  issue_load<NMAX, LAYOUT>(slot, bar, A, n, lda, lane);
  // the second wave of CTAs (sharing SMs with the first) starts later, so the
  // two CTAs on an SM do not run their factorization and memory phases in
  // lockstep (RELAPACK_BATCH_STAGGER_NS; the first load is already in flight)
  if (stagger_ns > 0 && blockIdx.x >= gridDim.x / 2)
    for (int w = 0; w < stagger_ns; w += 1000) __nanosleep(1000);
  uint32_t parity = 0;
  // the next matrix's list entry, one iteration ahead (RELAPACK_BATCH_DESC_AHEAD):
  // its descriptor loads then start before this matrix's wait and register load
  constexpr bool kAhead = RELAPACK_BATCH_DESC_AHEAD && NMAX == 64;  // measured: helps the 64-class only
  int nb_ahead = (kAhead && pos + stride < count) ? list[pos + stride] : 0;
  while (pos < count) {
    double v[T::NT][2];
    const int npos = pos + stride;
    int nb = 0, nn = 0;
    int64_t nlda = 0;
    double* nA = nullptr;
    if (kAhead && npos < count) {
      nb = nb_ahead;
      nn = d_n[nb];
      nlda = d_lda[nb];
      nA = d_A[nb];
      nb_ahead = npos + stride < count ? list[npos + stride] : 0;
    }
    const bool sq = square_ok<NMAX, LAYOUT>(A, n, lda);
    const bool bulk = bulk_ok<NMAX, LAYOUT>(A, n, lda);
    if (sq) {
      asm volatile("cp.async.wait_all;\n" ::: "memory");
      __syncwarp();
    } else if (bulk) {
      mbar_wait(bar, parity);
      parity ^= 1u;
    } else {
      plain_to_slot<NMAX, LAYOUT>(slot, A, n, lda, lane);
    }
    // the slot offsets of the 72 (n = 64) register elements depend only on the
    // lane: computed from an opaque copy of it, so they are not hoisted out of
    // the matrix loop and held live across it (register spills)
    load_regs<NMAX, LAYOUT>(v, slot, sq, n, opaque(lane));
    // prefetch this warp's next matrix into the (now consumed) slot
    if (npos < count) {
      if (!kAhead) {
        nb = list[npos];
        nn = d_n[nb];
        nlda = d_lda[nb];
        nA = d_A[nb];
      }
      issue_load<NMAX, LAYOUT>(slot, bar, nA, nn, nlda, lane);
    }
    // the lower triangle of L is stored panel by panel as it becomes final
    // (only the uplo triangle is written)
    double* const Al = A + lv_off(LAYOUT, g, 2 * t, lda);
    const int64_t cs = LAYOUT == kLayoutN ? lda : 1, rs = LAYOUT == kLayoutN ? 1 : lda;  // column / row stride
    auto sink = [&](int k) {
      double* Ak = Al + 8 * k * cs;
#pragma unroll
      for (int i = k; i < C::TN; ++i)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int r = 8 * i + g, c = 8 * k + 2 * t + q;
          if (r < n && c < n && r >= c) __stcs(Ak + 8 * i * rs + q * cs, v[T::id(i, k)][q]);  // st.global.cs: streamed out, not re-read
        }
    };
#if RELAPACK_BATCH_MODE == 1  // tools/microbench only: memory phases alone
    const int fail = 0;
#pragma unroll
    for (int k = 0; k < C::TN; ++k) sink(k);
#else
    const int fail = reg_potrf<NMAX / 8>(v, lane, sink);
#endif
    if (lane == 0) d_info[b] = fail;
    pos = npos;
    b = nb;
    n = nn;
    lda = nlda;
    A = nA;
  }
}

template <int NMAX, int LAYOUT>
cudaError_t launch_cls(int batch, const int* counts, const int* lists, double* const* d_A, const int* d_n,
                       const int* d_lda, int* d_info, int dev, int sms, cudaStream_t st) {
  using C = BC<NMAX, LAYOUT>;
  static int occ[kMaxDevices] = {};  // CTAs per SM of this instantiation (0: not configured on that device)
  int& per_sm = occ[dev];
  cudaError_t e;
  if (per_sm == 0) {
    if ((e = cudaFuncSetAttribute(k_batched_cls<NMAX, LAYOUT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)C::SMEM)) != cudaSuccess)
      return e;
    int p = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p, k_batched_cls<NMAX, LAYOUT>, C::WPC * 32, C::SMEM)) !=
        cudaSuccess)
      return e;
    per_sm = p > 0 ? p : 1;
  }
  int grid = sms * per_sm;
  const int need = (batch + C::WPC - 1) / C::WPC;
  if (grid > need) grid = need;
  static const int stagger = [] {
    const char* v = getenv("RELAPACK_BATCH_STAGGER_NS");
    return v ? atoi(v) : 0;
  }();
  k_batched_cls<NMAX, LAYOUT><<<grid, C::WPC * 32, C::SMEM, st>>>(batch, counts, lists, d_A, d_n, d_lda, d_info,
                                                                  stagger);
  return cudaGetLastError();
}

template <int LAYOUT>
cudaError_t launch_classes(int batch, const int* counts, const int* lists, double* const* d_A, const int* d_n,
                           const int* d_lda, int* d_info, int dev, int sms, cudaStream_t st) {
  cudaError_t e;
  if ((e = launch_cls<64, LAYOUT>(batch, counts, lists, d_A, d_n, d_lda, d_info, dev, sms, st)) != cudaSuccess) return e;
  if ((e = launch_cls<48, LAYOUT>(batch, counts, lists, d_A, d_n, d_lda, d_info, dev, sms, st)) != cudaSuccess) return e;
  if ((e = launch_cls<32, LAYOUT>(batch, counts, lists, d_A, d_n, d_lda, d_info, dev, sms, st)) != cudaSuccess) return e;
  return launch_cls<16, LAYOUT>(batch, counts, lists, d_A, d_n, d_lda, d_info, dev, sms, st);
}

// Library-owned bucketing workspace per device (grown on demand; growing
// synchronizes the device once so no in-flight launch still uses the old one).
struct BatchWs {
  std::mutex mu;
  int* buf = nullptr;
  size_t cap = 0;  // batch entries
  int sms = 0;
  // one stream per size class, forked from / joined back into the caller's
  // stream: a class's CTAs start on the SMs the previous class's tail frees
  cudaStream_t cs[kClasses] = {};
  cudaEvent_t fork = nullptr, join[kClasses] = {};
  // end of the last call that used the workspace: a call on another stream
  // waits for it before overwriting the counts / lists
  cudaEvent_t done = nullptr;
};

static bool batch_streams() {
  static const bool v = [] {
    const char* e = getenv("RELAPACK_BATCH_STREAMS");
    return !(e && e[0] == '0');
  }();
  return v;
}
BatchWs g_bws[kMaxDevices];

}  // namespace

cudaError_t launch_potf2_batched(int layout, int batch, const int* d_n, double* const* d_A, const int* d_lda,
                                 int* d_info, cudaStream_t st) {
  if (batch <= 0) return cudaSuccess;
  int dev = 0;
  cudaError_t e;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  BatchWs& w = g_bws[dev];
  std::lock_guard<std::mutex> lk(w.mu);
  if (w.sms == 0 && (e = cudaDeviceGetAttribute(&w.sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  cudaStreamCaptureStatus capturing = cudaStreamCaptureStatusNone;
  if ((e = cudaStreamIsCapturing(st, &capturing)) != cudaSuccess) return e;
  const bool in_capture = capturing != cudaStreamCaptureStatusNone;
  const size_t ws_bytes = sizeof(int) * (kClasses + (size_t)kClasses * batch);
  int* ws = nullptr;
  if (in_capture) {
    // inside a graph capture the workspace belongs to the graph (an allocation
    // node freed by the graph's own free node): a replay never touches library
    // memory that a later eager call may regrow or another replay may share
    if ((e = cudaMallocAsync(&ws, ws_bytes, st)) != cudaSuccess) return e;
  } else {
    if ((size_t)batch > w.cap) {
      if (w.buf) {
        if ((e = cudaDeviceSynchronize()) != cudaSuccess) return e;
        cudaFree(w.buf);
        w.buf = nullptr;
        w.cap = 0;
      }
      if ((e = cudaMalloc(&w.buf, ws_bytes)) != cudaSuccess) return e;
      w.cap = (size_t)batch;
    }
    ws = w.buf;
  }
  // the lists are indexed with stride `batch` of this call
  int* counts = ws;
  int* lists = ws + kClasses;
  if (!w.done && (e = cudaEventCreateWithFlags(&w.done, cudaEventDisableTiming)) != cudaSuccess) return e;
  // eager calls: the previous eager call (any stream) has finished with the
  // library workspace before this one overwrites it
  if (!in_capture && (e = cudaStreamWaitEvent(st, w.done, 0)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(counts, 0, kClasses * sizeof(int), st)) != cudaSuccess) return e;
  k_bucket<<<(batch + 255) / 256, 256, 0, st>>>(batch, d_n, d_lda, d_info, counts, lists);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (!batch_streams()) {
    e = layout == kLayoutN ? launch_classes<kLayoutN>(batch, counts, lists, d_A, d_n, d_lda, d_info, dev, w.sms, st)
                           : launch_classes<kLayoutT>(batch, counts, lists, d_A, d_n, d_lda, d_info, dev, w.sms, st);
    if (e != cudaSuccess) return e;
    return in_capture ? cudaFreeAsync(ws, st) : cudaEventRecord(w.done, st);
  }
  if (!w.fork) {
    if ((e = cudaEventCreateWithFlags(&w.fork, cudaEventDisableTiming)) != cudaSuccess) return e;
    for (int c = 0; c < kClasses; ++c) {
      if ((e = cudaStreamCreateWithFlags(&w.cs[c], cudaStreamNonBlocking)) != cudaSuccess) return e;
      if ((e = cudaEventCreateWithFlags(&w.join[c], cudaEventDisableTiming)) != cudaSuccess) return e;
    }
  }
  if ((e = cudaEventRecord(w.fork, st)) != cudaSuccess) return e;
  for (int c = kClasses - 1; c >= 0; --c) {  // the 64-class (longest) first
    if ((e = cudaStreamWaitEvent(w.cs[c], w.fork, 0)) != cudaSuccess) return e;
    const int nmax = 16 * (c + 1);
    auto go = [&](auto lay) -> cudaError_t {
      constexpr int L = decltype(lay)::value;
      switch (nmax) {
        case 64: return launch_cls<64, L>(batch, counts, lists, d_A, d_n, d_lda, d_info, dev, w.sms, w.cs[c]);
        case 48: return launch_cls<48, L>(batch, counts, lists, d_A, d_n, d_lda, d_info, dev, w.sms, w.cs[c]);
        case 32: return launch_cls<32, L>(batch, counts, lists, d_A, d_n, d_lda, d_info, dev, w.sms, w.cs[c]);
        default: return launch_cls<16, L>(batch, counts, lists, d_A, d_n, d_lda, d_info, dev, w.sms, w.cs[c]);
      }
    };
    e = layout == kLayoutN ? go(std::integral_constant<int, kLayoutN>{}) : go(std::integral_constant<int, kLayoutT>{});
    if (e != cudaSuccess) return e;
    if ((e = cudaEventRecord(w.join[c], w.cs[c])) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(st, w.join[c], 0)) != cudaSuccess) return e;
  }
  // (not inside a capture: an event recorded there cannot be waited on later)
  return in_capture ? cudaFreeAsync(ws, st) : cudaEventRecord(w.done, st);
}

void release_batched_workspace() {
  for (int d = 0; d < kMaxDevices; ++d) {
    std::lock_guard<std::mutex> lk(g_bws[d].mu);
    BatchWs& w = g_bws[d];
    if (w.buf || w.fork) {
      int cur = 0;
      cudaGetDevice(&cur);
      cudaSetDevice(d);
      if (w.buf) cudaFree(w.buf);
      if (w.done) cudaEventDestroy(w.done);
      if (w.fork) {
        cudaEventDestroy(w.fork);
        for (int c = 0; c < kClasses; ++c) {
          cudaStreamDestroy(w.cs[c]);
          cudaEventDestroy(w.join[c]);
        }
      }
      cudaSetDevice(cur);
    }
    w.buf = nullptr;
    w.fork = nullptr;
    w.done = nullptr;
    for (int c = 0; c < kClasses; ++c) {
      w.cs[c] = nullptr;
      w.join[c] = nullptr;
    }
    g_bws[d].cap = 0;
  }
}

}  // namespace relapack
