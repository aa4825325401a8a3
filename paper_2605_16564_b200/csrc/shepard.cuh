// shepard.cuh — the Shepard-normalised Gaussian evaluation shared by the
// residual (K3) and global-evaluation (K4) kernels.
//
// v(x) = (sum_m e_m beta_m) / (sum_m e_m),  e_m = exp(L_m(x) - max_m L_m(x))
// (reference rbf.py:152-167).  Two passes over the dictionary (max, then the
// normalised sums) exactly as the reference does it, so every exponent is
// exp(L - max) with max the true row maximum.  The dictionary is staged
// through shared memory in chunks of SH_CHUNK entries (centre, 1/(2w^2),
// beta) and read as warp-uniform broadcasts.
#pragma once
#include "pam_common.cuh"

namespace pam {

constexpr int SH_CHUNK = 512;

template <int D>
struct ShepardSmem {
  double c[SH_CHUNK * D];
  double inv[SH_CHUNK];
  double beta[SH_CHUNK];
};

// Cooperative (whole-block) staging of dictionary entries [j0, j0+cnt).
template <int D>
__device__ __forceinline__ void stage_dict(ShepardSmem<D>& sm, const double* centres,
                                           const double* widths, const double* beta, int64_t doff,
                                           int j0, int cnt) {
  __syncthreads();
  for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
#pragma unroll
    for (int k = 0; k < D; ++k) sm.c[t * D + k] = centres[(doff + j0 + t) * D + k];
    sm.inv[t] = inv_two_sigma_sq(widths[doff + j0 + t]);
    sm.beta[t] = beta ? beta[doff + j0 + t] : 0.0;
  }
  __syncthreads();
}

// Block-cooperative Shepard evaluation: every thread of the block calls this
// with its own point (live=false threads still participate in the barriers).
// Returns v; sets *den_out to the Shepard denominator.
template <int D>
__device__ double shepard_eval_block(ShepardSmem<D>& sm, const double* x, bool live,
                                     const double* centres, const double* widths,
                                     const double* beta, int64_t doff, int M, double* den_out) {
  double mx = -INFINITY;
  for (int j0 = 0; j0 < M; j0 += SH_CHUNK) {
    const int cnt = min(SH_CHUNK, M - j0);
    stage_dict<D>(sm, centres, widths, beta, doff, j0, cnt);
    if (live)
      for (int t = 0; t < cnt; ++t) mx = fmax(mx, log_feature<D>(x, &sm.c[t * D], sm.inv[t]));
  }
  double num = 0.0, den = 0.0;
  for (int j0 = 0; j0 < M; j0 += SH_CHUNK) {
    const int cnt = min(SH_CHUNK, M - j0);
    if (M > SH_CHUNK) stage_dict<D>(sm, centres, widths, beta, doff, j0, cnt);
    if (live)
      for (int t = 0; t < cnt; ++t) {
        const double e = exp(__dsub_rn(log_feature<D>(x, &sm.c[t * D], sm.inv[t]), mx));
        num = fma(e, sm.beta[t], num);
        den = __dadd_rn(den, e);
      }
  }
  *den_out = den;
  return num / den;
}

__device__ __forceinline__ bool shepard_degenerate(double den) {
  return !isfinite(den) || den <= 0.0;
}

}  // namespace pam
