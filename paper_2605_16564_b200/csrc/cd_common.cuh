// cd_common.cuh — declarations shared by the batched CD kernels (cd.cu,
// cd_block.cu): the argument block, flags, tile-run codes, dispatch helpers.
#pragma once
#include "pam_common.cuh"

namespace pam {

constexpr int CD_REG_ROWS = 8192;  // rows a register-resident residual covers (cd_kernel, G = 8)

enum : int { CD_COLSQ_GIVEN = 1, CD_R_GIVEN = 2, CD_WRITE_R = 4 };

struct CdArgs {
  int64_t S;
  const int64_t* order;
  const int64_t* row_off;
  double* y;  // targets (or residual when CD_R_GIVEN); residual written back with CD_WRITE_R
  const int64_t* dict_off;
  const int32_t* m_cur;
  const int64_t* w_off;
  const int32_t* ld;
  const double* W;
  const double* lam1;
  const double* lam2;
  const double* tol;
  const int32_t* max_iters;
  const int32_t* active;
  double* beta;
  double* col_sq;
  int32_t* sweeps;
  int32_t* converged;
  double* objective;
  double* hist;
  const int64_t* hist_off;
  int flags;
  // tile-packed design matrices (tiles.cu); null = dense column-major W
  const unsigned long long* tile_mask;
  const int64_t* col_off;
  const int32_t* perm;  // tile mode: packed position -> local row (nullable = identity)
  unsigned* queue;      // work counter in the caller's workspace (zeroed by the launcher)
  double* rbuf;         // large-fit residual scratch (sum N doubles, workspace)
};

// Run code of a tile mask made of one contiguous run (tiles.cu run_cover):
// a0 | la << 8  (run = tiles [a0, a0+la))
__device__ __forceinline__ int tile_code(unsigned long long mk) {
  if (mk == 0ull) return 0;
  const int a0 = __ffsll(static_cast<long long>(mk)) - 1;
  return a0 | (__popcll(mk) << 8);
}
__device__ __forceinline__ int code_tiles(int code) { return (code >> 8) & 0xff; }

// 16-lane (half-warp) reductions of the two-fits-per-warp kernels
__device__ __forceinline__ double half_sum(double v) {
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double half_max(double v) {
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

inline int sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

// blocked few-fit CD (cd_block.cu)
int64_t cd_block_workspace_bytes(int64_t S, int64_t total_slots);
int launch_cd_block(const CdArgs& a, int max_rows, void* block_ws, cudaStream_t stream);

}  // namespace pam
