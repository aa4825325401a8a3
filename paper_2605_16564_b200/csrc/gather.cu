// gather.cu — batch construction and standalone row normalisation.
//
// pam_gather_cells_f64 replaces Partition.subdomain_fields ->
// FieldData.subdomain (reference partition.py:41-42, fields.py:61-73): the
// reference masks all n_cells centroids once per box (O(n_cells * S) on the
// host); here every output row computes its global cell directly from the
// structured layout (boxes are unions of whole cells, partition.py:83-92)
// and recomputes the centroid with the mesh formula (geometry.py:122-132)
// using round-to-nearest intrinsics, so coordinates are bit-identical.
//
// pam_row_normalize_f64 replaces shepard_normalize on an explicit feature
// matrix (rbf.py:131-144): one warp per row.
#include "pam_common.cuh"

#include <algorithm>

namespace pam {

template <int D>
__global__ void gather_kernel(const int64_t* __restrict__ counts, const int32_t* __restrict__ shape,
                              const double* __restrict__ lo, const double* __restrict__ d,
                              const double* __restrict__ values, int64_t S,
                              const int64_t* __restrict__ row_off, double* __restrict__ pts,
                              double* __restrict__ vals, int64_t* __restrict__ cell_idx) {
  const int64_t total = row_off[S];
  int64_t nloc[3] = {1, 1, 1}, ncnt[3] = {1, 1, 1};
  int p[3] = {1, 1, 1};
#pragma unroll
  for (int k = 0; k < D; ++k) {
    ncnt[k] = counts[k];
    p[k] = shape[k];
    nloc[k] = ncnt[k] / p[k];
  }
  const int64_t per = nloc[0] * nloc[1] * nloc[2];
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = g / per;  // equal-size boxes (make_partition requires divisibility)
    const int64_t t = g - s * per;
    const int64_t sx = s % p[0];
    const int64_t sy = (s / p[0]) % p[1];
    const int64_t sz = s / ((int64_t)p[0] * p[1]);
    int64_t ix = sx * nloc[0] + t % nloc[0];
    int64_t iy = sy * nloc[1] + (t / nloc[0]) % nloc[1];
    int64_t iz = sz * nloc[2] + t / (nloc[0] * nloc[1]);
    const int64_t cell = (iz * ncnt[1] + iy) * ncnt[0] + ix;
    const int64_t ii[3] = {ix, iy, iz};
#pragma unroll
    for (int k = 0; k < D; ++k)
      pts[g * D + k] = __dadd_rn(lo[k], __dmul_rn(__dadd_rn((double)ii[k], 0.5), d[k]));
    vals[g] = values[cell];
    cell_idx[g] = cell;
  }
}

__global__ void row_normalize_kernel(int64_t N, int64_t M, const double* __restrict__ in, int mode,
                                     double* __restrict__ out, int64_t* err) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (row >= N) return;
  const double* r = in + row * M;
  double* o = out + row * M;
  if (mode == 1) {
    double mx = -INFINITY;
    for (int64_t j = lane; j < M; j += 32) mx = fmax(mx, r[j]);
    mx = warp_max(mx);
    double sum = 0.0;
    for (int64_t j = lane; j < M; j += 32) sum += exp(__dsub_rn(r[j], mx));
    sum = warp_sum(sum);
    for (int64_t j = lane; j < M; j += 32) o[j] = __ddiv_rn(exp(__dsub_rn(r[j], mx)), sum);
  } else {
    double sum = 0.0;
    for (int64_t j = lane; j < M; j += 32) sum += r[j];
    sum = warp_sum(sum);
    if (!(sum > 0.0)) {
      if (lane == 0) report_error(err, PAM_ERR_DEGENERATE, row);
      return;
    }
    for (int64_t j = lane; j < M; j += 32) o[j] = __ddiv_rn(r[j], sum);
  }
}

}  // namespace pam

using namespace pam;

extern "C" int pam_gather_cells_f64(int dim, const int64_t* counts, const int32_t* shape,
                                    const double* lo, const double* d, const double* values,
                                    int64_t S, const int64_t* row_off, double* pts_out,
                                    double* vals_out, int64_t* cell_idx_out, void* stream) {
  if (dim < 1 || dim > 3 || S < 1) return PAM_ERR_ARG;
  cudaStream_t st = as_stream(stream);
  const int threads = 256, blocks = 148 * 8;
  if (dim == 1)
    gather_kernel<1><<<blocks, threads, 0, st>>>(counts, shape, lo, d, values, S, row_off, pts_out,
                                                 vals_out, cell_idx_out);
  else if (dim == 2)
    gather_kernel<2><<<blocks, threads, 0, st>>>(counts, shape, lo, d, values, S, row_off, pts_out,
                                                 vals_out, cell_idx_out);
  else
    gather_kernel<3><<<blocks, threads, 0, st>>>(counts, shape, lo, d, values, S, row_off, pts_out,
                                                 vals_out, cell_idx_out);
  PAM_LAUNCH_CHECK("gather_kernel");
  return PAM_OK;
}

extern "C" int pam_row_normalize_f64(int64_t N, int64_t M, const double* in, int mode, double* out,
                                     int64_t* err, void* stream) {
  if (N < 0 || M < 1) return PAM_ERR_ARG;
  if (N == 0) return PAM_OK;
  const int threads = 256;
  const int64_t blocks = ceil_div(N * 32, threads);
  row_normalize_kernel<<<(unsigned)blocks, threads, 0, as_stream(stream)>>>(N, M, in, mode, out, err);
  PAM_LAUNCH_CHECK("row_normalize_kernel");
  return PAM_OK;
}
