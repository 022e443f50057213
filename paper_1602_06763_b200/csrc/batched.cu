// batched.cu — K2: independent small Cholesky factorizations (CFG[4]: 131072
// SPD matrices, n in {16, 32, 48, 64}; SPEC potf2 S:219-227 per matrix, one
// call, per-matrix info).
//
// The batch is HBM-bound in aggregate but every single factorization is a
// latency-bound chain (one pivot -> rsqrt -> update per column), so the design
// maximises matrices in flight per SM and strips integer overhead:
//  * a bucketing pass sorts the matrices into size classes NMAX in
//    {16, 32, 48, 64} (validating n / lda and writing info -2 / -4 on the way);
//  * one kernel per class, one WARP per matrix, persistent grid-stride over the
//    class list, no CTA-wide barriers;
//  * the matrix sits in shared memory padded with the identity beyond n, so
//    every loop runs at the compile-time size NMAX (factor of [A 0; 0 I] =
//    [L 0; 0 I]); NMAX >= 48 as a packed lower triangle (12 matrices per SM),
//    smaller classes as an odd-stride square;
//  * panels of 8 columns are factored in registers (lane l holds rows l and
//    l+32; pivot and l_kj broadcast by shuffles; rsqrt chain as in potf2.cu),
//    the rank-8 trailing update runs on the FP64 tensor cores (DMMA.8x8x4 on
//    8x8 tiles of the lower triangle, K = 8), all tiles of a tile row in flight;
//  * cp.async loads / coalesced stores along the contiguous index of either layout.
#include "common.cuh"
#include "kernels.h"

namespace relapack {

namespace {

constexpr int kPanel = 8;
constexpr int kClasses = 4;  // NMAX = 16 (c + 1)

template <int NMAX>
struct BC {
  static constexpr int LDS = NMAX + 1;
  static constexpr int R = (NMAX + 31) / 32;                 // panel rows per lane
  static constexpr int WPC = 4;                              // warps (matrices) per CTA
  // NMAX >= 48: packed lower triangle (column j at colbase(j) + i), so 12+
  // matrices stay resident per SM; smaller classes: odd-stride square.
  static constexpr bool PACKED = NMAX >= 48;
  static constexpr int PER_WARP = PACKED ? NMAX * (NMAX + 1) / 2 : NMAX * LDS;
  static constexpr size_t SMEM = sizeof(double) * PER_WARP * WPC;
  // offset of element (i, j), i >= j for the packed layout
  static __device__ __forceinline__ int off(int i, int j) {
    return PACKED ? j * NMAX - ((j * (j + 1)) >> 1) + i : i + j * LDS;
  }
};

// Factor the NMAX x NMAX lower triangle in s (s[i + j*LDS]); returns the
// 1-based first failing column (< n by construction of the padding) or 0.
template <int NMAX>
__device__ int factor_warp(double* s, int lane) {
  using C = BC<NMAX>;
  constexpr int R = C::R;
  const int g = lane >> 2, t = lane & 3;
  int fail = 0;
#pragma unroll(NMAX <= 32 ? NMAX / kPanel : 1)
  for (int j0 = 0; j0 < NMAX; j0 += kPanel) {
    // ---- panel [j0, j0 + 8): rows i_r = lane + 32 r in registers
    double x[R][kPanel];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = lane + 32 * r;
#pragma unroll
      for (int c = 0; c < kPanel; ++c) x[r][c] = (i < NMAX && i >= j0 + c) ? s[C::off(i, j0 + c)] : 0.0;
    }
    double dpiv[kPanel], rpiv[kPanel];
    double dnext = (R > 1 && j0 >= 32) ? x[R - 1][0] : x[0][0];
#pragma unroll
    for (int c = 0; c < kPanel; ++c) {
      const int j = j0 + c;
      const double d = __shfl_sync(0xffffffffu, dnext, j & 31);
      dpiv[c] = d;
      const double rinv = rsqrt_nr(d);
      rpiv[c] = rinv;
#pragma unroll
      for (int r = 0; r < R; ++r) x[r][c] *= rinv;
      if (c + 1 < kPanel) {
        const int jn = j + 1;
        const double xn = (R > 1 && jn >= 32) ? x[R - 1][c] : x[0][c];
        const double an = (R > 1 && jn >= 32) ? x[R - 1][c + 1] : x[0][c + 1];
        dnext = an - xn * xn;
#pragma unroll
        for (int c2 = c + 1; c2 < kPanel; ++c2) {
          const int jj = j0 + c2;
          const double l = __shfl_sync(0xffffffffu, (R > 1 && jj >= 32) ? x[R - 1][c] : x[0][c], jj & 31);
#pragma unroll
          for (int r = 0; r < R; ++r) x[r][c2] -= x[r][c] * l;
        }
      }
    }
#pragma unroll
    for (int c = kPanel - 1; c >= 0; --c)
      if (!(dpiv[c] > 0.0)) fail = j0 + c + 1;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = lane + 32 * r;
#pragma unroll
      for (int c = 0; c < kPanel; ++c) {
        if (i == j0 + c) x[r][c] = sqrt_from_rsqrt(dpiv[c], rpiv[c]);
        if (i < NMAX && i >= j0 + c) s[C::off(i, j0 + c)] = x[r][c];
      }
    }
    __syncwarp();
    if (fail) return fail;
    // ---- trailing update A22 -= P2 P2^T on 8x8 tiles (lower), K = 8; the
    // tiles of one tile row are independent DMMA chains issued together
    const int r0 = j0 + kPanel;
    constexpr int TK = NMAX / 8 - 1;
    for (int ti = 0; r0 + 8 * ti < NMAX; ++ti) {
      const int ia = r0 + 8 * ti + g;
      double a[2];
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) a[ks] = -s[C::off(ia, j0 + 4 * ks + t)];
      double c0[TK], c1[TK];
#pragma unroll
      for (int tk = 0; tk < TK; ++tk) {
        // positions above the diagonal (diagonal tile, g < 2t + c) are don't-care;
        // the packed layout does not store them at all
        const int jc = r0 + 8 * tk + 2 * t;
        if (tk <= ti) {
          c0[tk] = (jc <= ia) ? s[C::off(ia, jc)] : 0.0;
          c1[tk] = (jc + 1 <= ia) ? s[C::off(ia, jc + 1)] : 0.0;
        }
      }
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
#pragma unroll
        for (int tk = 0; tk < TK; ++tk) {
          if (tk <= ti) dmma_884(c0[tk], c1[tk], a[ks], s[C::off(r0 + 8 * tk + g, j0 + 4 * ks + t)]);
        }
      }
#pragma unroll
      for (int tk = 0; tk < TK; ++tk) {
        const int jc = r0 + 8 * tk + 2 * t;
        if (tk <= ti && jc <= ia) s[C::off(ia, jc)] = c0[tk];
        if (tk <= ti && jc + 1 <= ia) s[C::off(ia, jc + 1)] = c1[tk];
      }
    }
    __syncwarp();
  }
  return fail;
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

template <int NMAX>
__global__ void __launch_bounds__(BC<NMAX>::WPC * 32) k_batched_cls(int layout, int batch, const int* counts,
                                                                     const int* lists, double* const* d_A,
                                                                     const int* d_n, const int* d_lda, int* d_info) {
  using C = BC<NMAX>;
  constexpr int WPC = C::WPC;
  extern __shared__ double smem_b[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* s = smem_b + warp * C::PER_WARP;
  const uint32_t sbase = smem_u32(s);
  const int cls = NMAX / 16 - 1;
  const int count = counts[cls];
  const int* list = lists + (size_t)cls * batch;
  for (int pos = blockIdx.x * WPC + warp; pos < count; pos += gridDim.x * WPC) {
    const int b = list[pos];
    const int n = d_n[b];
    const int64_t lda = d_lda[b];
    double* A = d_A[b];
    // ---- stage: identity padding, then cp.async of the lower triangle
    for (int e = lane; e < NMAX * NMAX; e += 32) {
      const int i = e % NMAX, j = e / NMAX;
      if ((i >= n || j >= n) && i >= j) s[C::off(i, j)] = (i == j) ? 1.0 : 0.0;
    }
    for (int o = 0; o < n; ++o) {
      const int cnt = layout == kLayoutN ? n - o : o + 1;
      for (int q = lane; q < cnt; q += 32) {
        const int i = layout == kLayoutN ? o + q : o, j = layout == kLayoutN ? o : q;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sbase + 8u * (uint32_t)C::off(i, j)),
                     "l"(A + lv_off(layout, i, j, lda))
                     : "memory");
      }
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncwarp();
    const int fail = factor_warp<NMAX>(s, lane);
    for (int o = 0; o < n; ++o) {
      const int cnt = layout == kLayoutN ? n - o : o + 1;
      for (int q = lane; q < cnt; q += 32) {
        const int i = layout == kLayoutN ? o + q : o, j = layout == kLayoutN ? o : q;
        A[lv_off(layout, i, j, lda)] = s[C::off(i, j)];
      }
    }
    if (lane == 0) d_info[b] = fail;
    __syncwarp();
  }
}

template <int NMAX>
cudaError_t launch_cls(int layout, int batch, const int* counts, const int* lists, double* const* d_A, const int* d_n,
                       const int* d_lda, int* d_info, cudaStream_t st) {
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_batched_cls<NMAX>, BC<NMAX>::WPC * 32,
                                                                BC<NMAX>::SMEM);
  if (e != cudaSuccess) return e;
  int sms = 148;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int grid = sms * (per_sm > 0 ? per_sm : 1);
  const int need = (batch + BC<NMAX>::WPC - 1) / BC<NMAX>::WPC;
  if (grid > need) grid = need;
  k_batched_cls<NMAX><<<grid, BC<NMAX>::WPC * 32, BC<NMAX>::SMEM, st>>>(layout, batch, counts, lists, d_A, d_n, d_lda,
                                                                       d_info);
  return cudaGetLastError();
}

template <int NMAX>
cudaError_t configure_cls() {
  return cudaFuncSetAttribute(k_batched_cls<NMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BC<NMAX>::SMEM);
}

}  // namespace

cudaError_t configure_batched() {
  cudaError_t e;
  if ((e = configure_cls<16>()) != cudaSuccess) return e;
  if ((e = configure_cls<32>()) != cudaSuccess) return e;
  if ((e = configure_cls<48>()) != cudaSuccess) return e;
  return configure_cls<64>();
}

cudaError_t launch_potf2_batched(int layout, int batch, const int* d_n, double* const* d_A, const int* d_lda,
                                 int* d_info, cudaStream_t st) {
  if (batch <= 0) return cudaSuccess;
  static bool configured[kMaxDevices] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  cudaError_t e;
  if (dev >= 0 && dev < kMaxDevices && !configured[dev]) {
    if ((e = configure_batched()) != cudaSuccess) return e;
    configured[dev] = true;
  }
  // stream-ordered workspace: 4 class counters + 4 lists of up to `batch` indices
  int* ws = nullptr;
  const size_t bytes = sizeof(int) * (kClasses + (size_t)kClasses * batch);
  if ((e = cudaMallocAsync(&ws, bytes, st)) != cudaSuccess) return e;
  int* counts = ws;
  int* lists = ws + kClasses;
  if ((e = cudaMemsetAsync(counts, 0, kClasses * sizeof(int), st)) != cudaSuccess) return e;
  k_bucket<<<(batch + 255) / 256, 256, 0, st>>>(batch, d_n, d_lda, d_info, counts, lists);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if ((e = launch_cls<64>(layout, batch, counts, lists, d_A, d_n, d_lda, d_info, st)) != cudaSuccess) return e;
  if ((e = launch_cls<48>(layout, batch, counts, lists, d_A, d_n, d_lda, d_info, st)) != cudaSuccess) return e;
  if ((e = launch_cls<32>(layout, batch, counts, lists, d_A, d_n, d_lda, d_info, st)) != cudaSuccess) return e;
  if ((e = launch_cls<16>(layout, batch, counts, lists, d_A, d_n, d_lda, d_info, st)) != cudaSuccess) return e;
  return cudaFreeAsync(ws, st);
}

}  // namespace relapack
