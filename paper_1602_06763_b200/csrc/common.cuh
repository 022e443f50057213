// common.cuh — sm_100a building blocks shared by the relapack kernels:
// L-view addressing, mbarrier / TMA (cp.async.bulk.tensor) wrappers and the
// FP64 tensor-core MMA (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4).
//
// FP64 on sm_100a (measured, tools/microbench/fp64_peak.cu, profiles/): there is
// no tcgen05 kind::f64; DMMA.8x8x4 reaches 37.0 TFLOP/s vs 34.2 for DFMA
// register chains at 1965 MHz, so every dense update runs on DMMA.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace relapack {

// Layout of the L-view: the algorithm always works on
// the lower factor L.  uplo 'L': L(i,j) = A[i + j*ld] (kLayoutN, rows
// contiguous).  uplo 'U': A = U^T U, L = U^T, so L(i,j) = A[j + i*ld]
// (kLayoutT, columns contiguous).
enum : int { kLayoutN = 0, kLayoutT = 1 };

__host__ __device__ __forceinline__ int64_t lv_off(int layout, int64_t i, int64_t j, int64_t ld) {
  return layout == kLayoutN ? i + j * ld : j + i * ld;
}

// ----------------------------------------------------------------------------
// mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra LAB_WAIT;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ----------------------------------------------------------------------------
// TMA: 2-D tiled bulk tensor load global -> shared, completion on an mbarrier.
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// A descriptor in global memory modified through the generic proxy (the
// plan's first node rebases it with tensormap.replace): acquire it for the
// tensormap proxy before the first TMA that uses it.
__device__ __forceinline__ void tma_acquire_desc(const CUtensorMap* map) {
  asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;\n" ::"l"(reinterpret_cast<uint64_t>(map))
               : "memory");
}

__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// ----------------------------------------------------------------------------
// FP64 tensor core: D(8x8) += A(8x4) * B(4x8).  Lane l: a = A[l/4][l%4],
// b = B[l%4][l/4], d = {D[l/4][2(l%4)], D[l/4][2(l%4)+1]}.
__device__ __forceinline__ void dmma_884(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// 1/sqrt(d) for a positive normal d: hardware approximation (MUFU.RSQ64H,
// relative error < 2^-22) + one branch-free third-order correction
//   e = 1 - d y^2,   y <- y (1 + e/2 + 3e^2/8)
// (truncation ~ 5e^3/16 < 2^-66; ~1 ulp after rounding): four dependent FP64
// operations after the MUFU instead of six for two Newton steps — this is on
// the per-column critical path of every base-case factorization.
// The MUFU flushes subnormal inputs to zero (.ftz).  Pivots follow the same
// flush-to-zero semantics (reading R15): a pivot d is accepted only
// if d >= kMinPivot (the smallest normal double), so a subnormal pivot is
// reported through info like d <= 0 instead of turning into inf / NaN factors
// with info = 0 — the same single compare the !(d > 0) test was, off the chain.
constexpr double kMinPivot = 0x1p-1022;

__device__ __forceinline__ double rsqrt_nr(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  const double p = d * y;
  const double e = fma(-p, y, 1.0);
  const double t = fma(0.375, e, 0.5);
  return fma(y * e, t, y);
}


// sqrt(d) from y ~ 1/sqrt(d): r = d*y corrected by one fma-exact residual step
// (branch-free; exact for perfect squares, within an ulp otherwise).
__device__ __forceinline__ double sqrt_from_rsqrt(double d, double y) {
  const double r = d * y;
  const double e = fma(-r, r, d);
  return fma(e, 0.5 * y, r);
}

// Per-launch timeline record (tools/trace_timeline.py): earliest CTA start and
// latest CTA end in %globaltimer ns; null when tracing is off.
struct TraceRec {
  unsigned long long t0, t1;
};

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void trace_begin(TraceRec* tr) {
  if (tr && threadIdx.x == 0) atomicMin(&tr->t0, globaltimer_ns());
}

// Call at the end of a kernel by every thread (contains a barrier when on).
__device__ __forceinline__ void trace_end(TraceRec* tr) {
  if (tr) {
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(&tr->t1, globaltimer_ns());
  }
}

// Pointer-independent plan graphs (driver.cu): the run's info word and the
// matrix base live in one 16-byte PlanState written by the graph's first node;
// the plan's kernels get byte offsets instead of pointers and a d_info tagged
// with bit 0 pointing at the PlanState, and add the base they read together
// with the info word (one load, no extra latency).  An untagged d_info is a
// plain info word and the pointer arguments are absolute (base 0).
struct alignas(16) PlanState {
  int info;
  int pad;
  unsigned long long base;
};

__device__ __forceinline__ int* untag(const int* d_info) {
  return reinterpret_cast<int*>(reinterpret_cast<uintptr_t>(d_info) & ~uintptr_t(1));
}

struct KState {
  int info;
  uintptr_t base;
};

// Every plan kernel starts here: wait for the grids it depends on
// (programmatic dependent launch: a no-op unless the graph edge into this
// node is programmatic, driver.cu capture_dag), then read the info word (and,
// in a pointer-independent plan, the matrix base).
__device__ __forceinline__ KState ld_state(const int* d_info) {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  const uintptr_t t = reinterpret_cast<uintptr_t>(d_info);
  KState s;
  if (t & 1) {
    unsigned a, b, c, d;
    asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                 : "l"(t & ~uintptr_t(1))
                 : "memory");
    s.info = (int)a;
    s.base = ((uintptr_t)d << 32) | c;
  } else {
    s.info = *reinterpret_cast<const volatile int*>(d_info);
    s.base = 0;
  }
  return s;
}

__device__ __forceinline__ int ld_info(const int* d_info) { return ld_state(d_info).info; }

// The matrix base again (a cached load of the PlanState; 0 for an untagged
// d_info), for uses before the kernel's first barrier.
__device__ __forceinline__ uintptr_t plan_base(const int* d_info) {
  const uintptr_t t = reinterpret_cast<uintptr_t>(d_info);
  return (t & 1) ? reinterpret_cast<const PlanState*>(t & ~uintptr_t(1))->base : 0;
}

template <class T>
__device__ __forceinline__ T* rebase(T* p, uintptr_t base) {
  return reinterpret_cast<T*>(reinterpret_cast<uintptr_t>(p) + base);
}

// Let the dependent grids launch (they still wait for this grid's completion
// in ld_info): issued when a CTA's main work is done, so their launch
// latency overlaps this grid's stores.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

}  // namespace relapack
