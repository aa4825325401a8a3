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

namespace pam {
// one thread per destination dictionary entry: subdomain s's first
// cnt[s] = src_off[s+1]-src_off[s] slots receive entries src_off[s].. in order
__global__ void dict_scatter_kernel(int dim, int64_t S, const int64_t* __restrict__ src_off,
                                    const double* __restrict__ src_centres,
                                    const double* __restrict__ src_widths,
                                    const double* __restrict__ sigma, const int32_t* __restrict__ src_gens,
                                    const int64_t* __restrict__ dict_off, double* __restrict__ centres,
                                    double* __restrict__ widths, int32_t* __restrict__ gens) {
  const int64_t total = src_off[S];
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    // owning subdomain by binary search over src_off (S+1 ascending offsets)
    int64_t lo = 0, hi = S;
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (src_off[mid] <= g) lo = mid;
      else hi = mid;
    }
    const int64_t s = lo;
    const int64_t dst = dict_off[s] + (g - src_off[s]);
    for (int k = 0; k < dim; ++k) centres[dst * dim + k] = src_centres[g * dim + k];
    widths[dst] = src_widths ? src_widths[g] : sigma[s];
    gens[dst] = src_gens ? src_gens[g] : 0;
  }
}
}  // namespace pam

extern "C" int pam_dict_scatter_f64(int dim, int64_t S, const int64_t* src_off, const double* src_centres,
                                    const double* src_widths, const double* sigma, const int32_t* src_gens,
                                    const int64_t* dict_off, double* centres, double* widths, int32_t* gens,
                                    void* stream) {
  if (dim < 1 || dim > 3 || S < 0 || (src_widths == nullptr && sigma == nullptr)) return PAM_ERR_ARG;
  if (S == 0) return PAM_OK;
  dict_scatter_kernel<<<148 * 8, 256, 0, as_stream(stream)>>>(dim, S, src_off, src_centres, src_widths, sigma,
                                                              src_gens, dict_off, centres, widths, gens);
  PAM_LAUNCH_CHECK("dict_scatter_kernel");
  return PAM_OK;
}

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

// ---------------------------------------------------------------------------
// On-device generator of BASELINE config 5 inputs: unit
// boxes of a gx x gy x gz tiling (x fastest), n_pts uniform samples per box,
// 1-4 planar interfaces through uniform points with uniform normals and
// per-region levels 10^U[-3,3], and a jittered (lx, ly, lz) centre lattice
// (offsets U(-1/4, 1/4) of the spacing, clamped to the box).  Same
// distributions as workloads.config5 (host, numpy), different random stream:
// counter-based SplitMix64 hashes of (seed, box, stream, index), so the data
// are identical for any launch shape and deterministic.
namespace pam {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// uniform double in [0, 1) from (seed, box, stream, index)
__device__ __forceinline__ double u01(uint64_t seed, uint64_t box, uint32_t stream, uint64_t i) {
  const uint64_t h = mix64(seed ^ mix64(box * 0x100000001B3ull + stream) ^ mix64(i + 0x632BE59BD9B4E019ull));
  return static_cast<double>(h >> 11) * 0x1.0p-53;
}

struct C5Box {
  int k;
  double lo[3];
  double nrm[4][3];
  double thr[4][3];
  double lev[16];
};

__device__ void c5_box(uint64_t seed, int64_t s, int gx, int gy, C5Box& b) {
  b.lo[0] = static_cast<double>(s % gx);
  b.lo[1] = static_cast<double>((s / gx) % gy);
  b.lo[2] = static_cast<double>(s / (static_cast<int64_t>(gx) * gy));
  b.k = 1 + min(3, static_cast<int>(u01(seed, s, 1, 0) * 4.0));
  for (int p = 0; p < b.k; ++p) {
    // uniform direction: normalised Gaussian triple (Box-Muller)
    double v[3], nn = 0.0;
    for (int c = 0; c < 3; ++c) {
      const double u1 = 1.0 - u01(seed, s, 2, 6 * p + 2 * c), u2 = u01(seed, s, 2, 6 * p + 2 * c + 1);
      v[c] = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
      nn += v[c] * v[c];
    }
    nn = sqrt(nn);
    for (int c = 0; c < 3; ++c) {
      b.nrm[p][c] = v[c] / nn;
      b.thr[p][c] = b.lo[c] + u01(seed, s, 3, 3 * p + c);
    }
  }
  for (int r = 0; r < (1 << b.k); ++r) b.lev[r] = exp10(-3.0 + 6.0 * u01(seed, s, 4, r));
}

__global__ void c5_points_kernel(int64_t first, int64_t n_sub, int n_pts, int gx, int gy, uint64_t seed,
                                 double* pts, double* vals) {
  __shared__ C5Box b;
  for (int64_t ls = blockIdx.x; ls < n_sub; ls += gridDim.x) {
    const int64_t s = first + ls;  // global box index (random stream), ls = output slot
    __syncthreads();
    if (threadIdx.x == 0) c5_box(seed, s, gx, gy, b);
    __syncthreads();
    for (int i = threadIdx.x; i < n_pts; i += blockDim.x) {
      const int64_t row = ls * n_pts + i;
      double x[3];
      for (int c = 0; c < 3; ++c) {
        x[c] = b.lo[c] + u01(seed, s, 5, 3 * static_cast<uint64_t>(i) + c);
        pts[row * 3 + c] = x[c];
      }
      int region = 0;
      for (int p = 0; p < b.k; ++p) {
        double side = 0.0;
        for (int c = 0; c < 3; ++c) side += (x[c] - b.thr[p][c]) * b.nrm[p][c];
        region |= (side > 0.0 ? 1 : 0) << p;
      }
      vals[row] = b.lev[region];
    }
  }
}

__global__ void c5_centres_kernel(int64_t first, int64_t n_sub, int lx, int ly, int lz, int gx, int gy,
                                  uint64_t seed, double* cen) {
  const int M = lx * ly * lz;
  const double h[3] = {1.0 / lx, 1.0 / ly, 1.0 / lz};
  const int64_t total = n_sub * M;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = first + e / M;
    const int m = static_cast<int>(e % M);
    const int li[3] = {m % lx, (m / lx) % ly, m / (lx * ly)};
    const double lo[3] = {static_cast<double>(s % gx), static_cast<double>((s / gx) % gy),
                          static_cast<double>(s / (static_cast<int64_t>(gx) * gy))};
    for (int c = 0; c < 3; ++c) {
      const double j = (u01(seed, s, 6, 3 * static_cast<uint64_t>(m) + c) - 0.5) * 0.5 * h[c];
      const double v = lo[c] + (li[c] + 0.5) * h[c] + j;
      cen[e * 3 + c] = fmin(fmax(v, lo[c]), lo[c] + 1.0);
    }
  }
}

}  // namespace pam

extern "C" int pam_c5_generate_f64(int64_t first_box, int64_t n_sub, int32_t n_pts, int32_t lx, int32_t ly,
                                   int32_t lz, int32_t gx, int32_t gy, uint64_t seed, double* points,
                                   double* values, double* centres, void* stream) {
  if (first_box < 0 || n_sub < 1 || n_pts < 1 || lx < 1 || ly < 1 || lz < 1 || gx < 1 || gy < 1) return PAM_ERR_ARG;
  cudaStream_t st = as_stream(stream);
  const int blocks = static_cast<int>(std::min<int64_t>(n_sub, 148 * 16));
  c5_points_kernel<<<blocks, 256, 0, st>>>(first_box, n_sub, n_pts, gx, gy, seed, points, values);
  PAM_LAUNCH_CHECK("c5_points_kernel");
  c5_centres_kernel<<<148 * 8, 256, 0, st>>>(first_box, n_sub, lx, ly, lz, gx, gy, seed, centres);
  PAM_LAUNCH_CHECK("c5_centres_kernel");
  return PAM_OK;
}
