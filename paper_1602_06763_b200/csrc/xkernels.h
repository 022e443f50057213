// xkernels.h — launch interface of the §8(f) base-case kernels (xkernels.cu).
// Internal to the library.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace relapack {

constexpr int kTriMax = 64;        // widest triangular block of k_tri_rows / k_trti2 / k_lauu2
constexpr int kGetf2Max = 32;      // widest getrf panel of k_getf2
constexpr int kGetf2Threads = 256;
constexpr int kGetf2RowThreads = 128;  // threads on the panel rows; the rest swap rows outside the panel
// register panels of k_getf2_clr: rows per CTA for panel widths 32 / 16 / 8
constexpr int kGetf2ClRows32 = 512, kGetf2ClRows16 = 1024, kGetf2ClRows8 = 2048;

enum XTriMode : int {
  kTriSolveLT = 0,  // x := alpha x T^{-T}   (x T^T = alpha b, forward)
  kTriSolveL = 1,   // x := alpha x T^{-1}   (x T = alpha b, backward)
  kTriMulL = 2,     // x := alpha x T
  kTriMulLT = 3     // x := alpha x T^T
};

struct XTriArgs {
  const double* T;  // t x t lower-triangular block (lower part read only)
  int64_t ldt;
  int lt;           // layout of T
  double* B;        // m x t
  int64_t ldb;
  int lb;           // layout of B
  int m, t;
  int mode, unit;
  double alpha;
  const int* d_info;
};

struct XBlockArgs {   // k_trti2 / k_lauu2: one n x n lower-triangular block
  double* A;
  int64_t ld;
  int layout, n, unit;
  const int* d_info;
};

struct XGetf2Args {
  double* P;          // m x w panel, layout 0
  int64_t ld;
  int m, w, rows_per_cta;
  int* ipiv;          // w entries: pivot_base + panel-relative row
  int pivot_base;
  int* getrf_info;    // atomicMin(info_base + j + 1) on a zero pivot
  int info_base;
  unsigned* bar;      // grid barrier counter, zero at launch
  double* cand_val;   // 2 x grid
  int* cand_idx;      // 2 x grid
  double* cand_rows;  // 2 x grid x kGetf2Max
  double* diag_row;   // 2 x kGetf2Max
  double* A0;         // element (panel row 0, column 0) of the matrix: the interchanges apply to every column
  int ncols, c0;      // the matrix's columns; the panel's first column
  const int* d_info;
  // epoch-stamped exchange (poll != 0): 16-byte records {value, epoch} read
  // until their epoch is this column's — no grid barrier, no fence
  int poll;
  unsigned epoch_base;       // (replay << 16) | (op << 6) is added on the device (replay: *replay)
  const unsigned* replay;    // the plan's replay counter (incremented by its prologue)
  void* prec;                // [2][grid] candidate records {|a|, (epoch << 32) | row}
  void* prow;                // [2][grid][kGetf2Max] candidate-row records {a, epoch}
  void* pdiag;               // [2][kGetf2Max] row-j records {a, epoch}
};

// Cluster panel (k_getf2_clr): the same LU with partial pivoting of an m x w
// panel held by ONE thread-block cluster (C CTAs, rows split evenly), the
// per-column exchange through distributed shared memory and the hardware
// cluster barrier; interchanges outside the panel are left to k_permute.
struct XGetf2ClArgs {
  double* P;  // m x w panel, layout 0
  int64_t ld;
  int m, w, rows_per_cta;
  int* ipiv;
  int pivot_base;
  int* getrf_info;
  int info_base;
  const int* d_info;
};

// Row interchanges of one panel (pivots ipiv[k0 .. k0 + npiv), panel-relative
// row = ipiv - base) applied as one permutation to columns [0, ncols) of A
// (A = element (panel row 0, first column), layout 0): a warp per column
// gathers the at most 2 npiv affected rows and scatters them permuted.
struct XPermArgs {
  double* A;
  int64_t ld;
  int ncols;
  const int* ipiv;
  int k0, npiv, base;
  const int* d_info;
};

struct XLaswpArgs {
  double* A;      // columns [0, ncols) of the matrix, layout 0
  int64_t ld;
  int ncols;
  const int* ipiv;  // ipiv[k] - base = row interchanged with row k
  int k0, k1, base;
  const int* d_info;
};

cudaError_t launch_tri_rows(const XTriArgs& a, cudaStream_t st);
cudaError_t launch_trti2(const XBlockArgs& a, cudaStream_t st);
cudaError_t launch_lauu2(const XBlockArgs& a, cudaStream_t st);
cudaError_t launch_diag_check(const double* A, int64_t ld, int layout, int n, int* d_info, cudaStream_t st);
size_t getf2_smem(int rows_per_cta);
cudaError_t launch_getf2(const XGetf2Args& a, int grid, cudaStream_t st);
cudaError_t launch_laswp(const XLaswpArgs& a, cudaStream_t st);
// cluster size C (16 or 8; 0: no cluster can be scheduled); configures the
// cluster panel kernels once per device
int getf2_cluster_caps();
int getf2_cluster_size(int want);
cudaError_t launch_getf2_cl(const XGetf2ClArgs& a, int csize, cudaStream_t st);
cudaError_t launch_permute(const XPermArgs& a, cudaStream_t st);
cudaError_t configure_xkernels();

}  // namespace relapack
