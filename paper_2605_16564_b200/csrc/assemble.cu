// assemble.cu — K1: batched Shepard-normalised Gaussian design matrices.
//
// Replaces shepard_features = shepard_normalize(assemble_features(...))
// (reference rbf.py:79-91, 123-149) for every subdomain of a ragged batch in
// one launch.  Thread per sample row (so the column-major W store is
// coalesced across the warp), the subdomain's centres and 1/(2 w^2) staged
// through shared memory in chunks and read as warp broadcasts.  Three passes
// over the dictionary per row: row max of L, row sum of exp(L - max), then
// the normalised store W[i,j] = exp(L - max) / sum (true division, as numpy's
// `w /= w.sum(...)`, rbf.py:143).  The exponent L is bit-identical to the
// reference (pam_common.cuh: log_feature); exp is CUDA's correctly-rounded-
// to-1-ulp libdevice exp.
//
// Roofline: HBM-write bound when W is materialised (8 B per entry written,
// 2 exps per entry on the FP64 pipe).  It runs once per adaptive round and is
// <1% of the fit (the CD kernel re-reads W thousands of times).
#include "pam_common.cuh"

namespace pam {

constexpr int ASM_THREADS = 128;
constexpr int ASM_CHUNK = 512;  // dictionary entries staged per smem chunk

template <int D>
__global__ void __launch_bounds__(ASM_THREADS)
assemble_kernel(const int64_t* __restrict__ row_off, const double* __restrict__ pts,
                const int64_t* __restrict__ dict_off, const int32_t* __restrict__ m_cur,
                const double* __restrict__ centres, const double* __restrict__ widths,
                const int64_t* __restrict__ w_off, const int32_t* __restrict__ ld,
                const int32_t* __restrict__ active, int mode, double* __restrict__ W) {
  __shared__ double s_c[ASM_CHUNK * D];
  __shared__ double s_inv[ASM_CHUNK];

  const int64_t s = blockIdx.y;
  if (active != nullptr && active[s] == 0) return;
  const int64_t r0 = row_off[s];
  const int64_t n = row_off[s + 1] - r0;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * ASM_THREADS + threadIdx.x;
  if (static_cast<int64_t>(blockIdx.x) * ASM_THREADS >= n) return;  // whole block idle
  const bool live = i < n;
  const int M = m_cur[s];
  const int64_t doff = dict_off[s];
  double* Ws = W + w_off[s];
  const int64_t lds = ld[s];

  double x[D];
#pragma unroll
  for (int k = 0; k < D; ++k) x[k] = live ? pts[(r0 + i) * D + k] : 0.0;

  auto stage = [&](int j0, int cnt) {
    __syncthreads();
    for (int t = threadIdx.x; t < cnt; t += ASM_THREADS) {
#pragma unroll
      for (int k = 0; k < D; ++k) s_c[t * D + k] = centres[(doff + j0 + t) * D + k];
      s_inv[t] = inv_two_sigma_sq(widths[doff + j0 + t]);
    }
    __syncthreads();
  };

  if (mode != 0) {
    // raw features (rbf.py:79-91, 123-128): mode 1 = L, mode 2 = exp(L)
    for (int j0 = 0; j0 < M; j0 += ASM_CHUNK) {
      const int cnt = min(ASM_CHUNK, M - j0);
      stage(j0, cnt);
      if (live)
        for (int t = 0; t < cnt; ++t) {
          const double L = log_feature<D>(x, &s_c[t * D], s_inv[t]);
          Ws[static_cast<int64_t>(j0 + t) * lds + i] = (mode == 1) ? L : exp(L);
        }
    }
    return;
  }
  // pass 1: row max of L
  double mx = -INFINITY;
  for (int j0 = 0; j0 < M; j0 += ASM_CHUNK) {
    const int cnt = min(ASM_CHUNK, M - j0);
    stage(j0, cnt);
    for (int t = 0; t < cnt; ++t) mx = fmax(mx, log_feature<D>(x, &s_c[t * D], s_inv[t]));
  }
  // pass 2: row sum of exp(L - max)
  double sum = 0.0;
  for (int j0 = 0; j0 < M; j0 += ASM_CHUNK) {
    const int cnt = min(ASM_CHUNK, M - j0);
    stage(j0, cnt);
    for (int t = 0; t < cnt; ++t)
      sum = __dadd_rn(sum, exp(__dsub_rn(log_feature<D>(x, &s_c[t * D], s_inv[t]), mx)));
  }
  // pass 3: normalised store, column-major (coalesced across the warp's rows)
  for (int j0 = 0; j0 < M; j0 += ASM_CHUNK) {
    const int cnt = min(ASM_CHUNK, M - j0);
    stage(j0, cnt);
    if (live) {
      for (int t = 0; t < cnt; ++t) {
        const double e = exp(__dsub_rn(log_feature<D>(x, &s_c[t * D], s_inv[t]), mx));
        Ws[static_cast<int64_t>(j0 + t) * lds + i] = __ddiv_rn(e, sum);
      }
    }
  }
}

// y = log(values) with the positivity check of fit_log_field (elastic_net.py:197-205)
__global__ void log_values_kernel(const double* __restrict__ v, int64_t n, double* __restrict__ y,
                                  int64_t* err) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double a = v[i];
    if (!(a > 0.0)) {
      report_error(err, PAM_ERR_NONPOSITIVE, i);
      y[i] = 0.0;
    } else {
      y[i] = log(a);
    }
  }
}

__global__ void err_reset_kernel(int64_t* err) {
  err[0] = 0;
  err[1] = INT64_MAX;
}

}  // namespace pam

using namespace pam;

extern "C" int pam_err_reset(int64_t* err, void* stream) {
  if (!err) return PAM_ERR_ARG;
  err_reset_kernel<<<1, 1, 0, as_stream(stream)>>>(err);
  PAM_LAUNCH_CHECK("err_reset_kernel");
  return PAM_OK;
}

extern "C" int pam_log_values_f64(const double* values, int64_t n, double* y, int64_t* err,
                                  void* stream) {
  if (n < 0) return PAM_ERR_ARG;
  if (n == 0) return PAM_OK;
  const int threads = 256;
  const int64_t blocks = std::min<int64_t>(ceil_div(n, threads), 148 * 16);
  log_values_kernel<<<(unsigned)blocks, threads, 0, as_stream(stream)>>>(values, n, y, err);
  PAM_LAUNCH_CHECK("log_values_kernel");
  return PAM_OK;
}

extern "C" int pam_assemble_f64(int dim, int64_t S, const int64_t* row_off, const double* pts,
                                const int64_t* dict_off, const int32_t* m_cur,
                                const double* centres, const double* widths,
                                const int64_t* w_off, const int32_t* ld, const int32_t* active,
                                int32_t max_rows, int mode, double* W, void* stream) {
  if (S < 0 || max_rows < 0 || dim < 1 || dim > 3) return PAM_ERR_ARG;
  if (S == 0 || max_rows == 0) return PAM_OK;
  if (S > 65535) {
    // grid.y limit: split the batch
    for (int64_t s0 = 0; s0 < S; s0 += 65535) {
      const int64_t cnt = std::min<int64_t>(65535, S - s0);
      int st = pam_assemble_f64(dim, cnt, row_off + s0, pts, dict_off + s0, m_cur + s0, centres,
                                widths, w_off + s0, ld + s0, active ? active + s0 : nullptr,
                                max_rows, mode, W, stream);
      if (st != PAM_OK) return st;
    }
    return PAM_OK;
  }
  dim3 grid((unsigned)ceil_div(max_rows, ASM_THREADS), (unsigned)S);
  cudaStream_t st = as_stream(stream);
  switch (dim) {
    case 1:
      assemble_kernel<1><<<grid, ASM_THREADS, 0, st>>>(row_off, pts, dict_off, m_cur, centres,
                                                       widths, w_off, ld, active, mode, W);
      break;
    case 2:
      assemble_kernel<2><<<grid, ASM_THREADS, 0, st>>>(row_off, pts, dict_off, m_cur, centres,
                                                       widths, w_off, ld, active, mode, W);
      break;
    default:
      assemble_kernel<3><<<grid, ASM_THREADS, 0, st>>>(row_off, pts, dict_off, m_cur, centres,
                                                       widths, w_off, ld, active, mode, W);
      break;
  }
  PAM_LAUNCH_CHECK("assemble_kernel");
  return PAM_OK;
}
