// dist.cu — multi-GPU mode.  Placeholder until the NCCL path lands.
#include <cuda_runtime.h>

#include "../../include/relapack.h"
#include "driver_internal.h"

extern "C" {
int relapack_comm_unique_id(char uid[128]) {
  relapack::set_error("relapack_comm_unique_id: multi-GPU mode not built yet");
  return -1000;
}
int relapack_comm_init(relapack_comm_t** comm, const char uid[128], int nranks, int rank, int device) {
  relapack::set_error("relapack_comm_init: multi-GPU mode not built yet");
  return -1000;
}
void relapack_comm_destroy(relapack_comm_t* comm) {}
void relapack_dpotrf_dist(const char* uplo, const int* n, double* A, const int* lda, int nb, int dist_min,
                          relapack_comm_t* comm, int* info) {
  relapack::set_error("relapack_dpotrf_dist: multi-GPU mode not built yet");
  if (info) *info = -1000;
}
}
