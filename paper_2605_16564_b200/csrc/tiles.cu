// tiles.cu — K1t: tile-packed Shepard design matrices for the CD stream.
//
// Same W as K1 (assemble.cu; reference rbf.py:79-91, 123-149) but stored for
// the coordinate-descent kernel as a column-major sequence of 32-row TILES,
// keeping only tiles that hold at least one entry >= tau:
//
//   * rows are visited in a caller-supplied permutation `perm` (the engine
//     uses a recursive coordinate bisection of the sample points, so a tile
//     is a spatially compact blob of 32 cells and a narrow Gaussian touches
//     few tiles);
//   * tile_mask[col] (uint64) has bit k set when tile k of that column is
//     stored; col_off[col] is the column's offset (doubles) inside the
//     subdomain's packed block; stored tiles are contiguous per column, so
//     the CD kernel fetches a column with ONE cp.async.bulk of
//     popcount(mask) * 256 bytes.
//
// Entries below tau are dropped.  A dropped entry changes a CD dot product
// z_j = sum_i W_ij r_i by at most tau * sum_i |r_i|.  The default tau = 1e-16
// is below the FP64 unit roundoff of a row of W (rows sum to 1): zeroing every
// entry below it moves the reference's adaptive fits by ~1e-13 relative
// (tests/test_oracle_pins.py), five orders below the parity tolerance;
// tau = 2^-100 drops only entries invisible to FP64 sums, tau = 0 keeps every
// tile (exact dense streaming, K1 semantics).
//
// Three launches: (A) row max/sum + tile masks (ballot per warp = per tile),
// (B) per-subdomain exclusive scan of popcounts -> col_off, (C) packed store.
#include "pam_common.cuh"

#include <algorithm>

namespace pam {

constexpr int TL_THREADS = 128;
constexpr int TL_CHUNK = 512;

template <int D>
struct TileSmem {
  double c[TL_CHUNK * D];
  double inv[TL_CHUNK];
};

template <int D>
__device__ __forceinline__ void tl_stage(TileSmem<D>& sm, const double* centres, const double* widths,
                                         int64_t doff, int j0, int cnt) {
  __syncthreads();
  for (int t = threadIdx.x; t < cnt; t += TL_THREADS) {
#pragma unroll
    for (int k = 0; k < D; ++k) sm.c[t * D + k] = centres[(doff + j0 + t) * D + k];
    sm.inv[t] = inv_two_sigma_sq(widths[doff + j0 + t]);
  }
  __syncthreads();
}

struct TileArgs {
  const int64_t* row_off;
  const double* pts;
  const int32_t* perm;  // position -> local canonical row (nullable = identity)
  const int64_t* dict_off;
  const int32_t* m_cur;
  const double* centres;
  const double* widths;
  const int64_t* w_off;
  const int32_t* active;
  double tau;
  double* rowmax;  // per packed position
  double* rowsum;
  unsigned long long* tile_mask;  // per dictionary slot
  int64_t* col_off;               // per dictionary slot (doubles, relative to w_off)
  int64_t* packed_total;          // per subdomain: doubles stored (nullable)
  double* W;
};

// (A) row statistics + tile masks
template <int D>
__global__ void __launch_bounds__(TL_THREADS) tile_mask_kernel(const TileArgs a) {
  __shared__ TileSmem<D> sm;
  const int64_t s = blockIdx.y;
  if (a.active != nullptr && a.active[s] == 0) return;
  const int64_t r0 = a.row_off[s];
  const int n = static_cast<int>(a.row_off[s + 1] - r0);
  const int p = blockIdx.x * TL_THREADS + threadIdx.x;
  if (static_cast<int>(blockIdx.x) * TL_THREADS >= n) return;
  const bool live = p < n;
  const int row = live ? (a.perm ? a.perm[r0 + p] : p) : 0;
  const int M = a.m_cur[s];
  const int64_t doff = a.dict_off[s];
  const int lane = threadIdx.x & 31;
  const int tile = p >> 5;
  double x[D];
#pragma unroll
  for (int k = 0; k < D; ++k) x[k] = live ? a.pts[(r0 + row) * D + k] : 0.0;

  double mx = -INFINITY;
  for (int j0 = 0; j0 < M; j0 += TL_CHUNK) {
    const int cnt = min(TL_CHUNK, M - j0);
    tl_stage<D>(sm, a.centres, a.widths, doff, j0, cnt);
    for (int t = 0; t < cnt; ++t) mx = fmax(mx, log_feature<D>(x, &sm.c[t * D], sm.inv[t]));
  }
  double sum = 0.0;
  for (int j0 = 0; j0 < M; j0 += TL_CHUNK) {
    const int cnt = min(TL_CHUNK, M - j0);
    if (M > TL_CHUNK) tl_stage<D>(sm, a.centres, a.widths, doff, j0, cnt);
    for (int t = 0; t < cnt; ++t)
      sum = __dadd_rn(sum, exp(__dsub_rn(log_feature<D>(x, &sm.c[t * D], sm.inv[t]), mx)));
  }
  if (live) {
    a.rowmax[r0 + p] = mx;
    a.rowsum[r0 + p] = sum;
  }
  for (int j0 = 0; j0 < M; j0 += TL_CHUNK) {
    const int cnt = min(TL_CHUNK, M - j0);
    if (M > TL_CHUNK) tl_stage<D>(sm, a.centres, a.widths, doff, j0, cnt);
    for (int t = 0; t < cnt; ++t) {
      const double w =
          __ddiv_rn(exp(__dsub_rn(log_feature<D>(x, &sm.c[t * D], sm.inv[t]), mx)), sum);
      const unsigned keep = __ballot_sync(0xffffffffu, live && !(w < a.tau));
      if (lane == 0 && keep) atomicOr(&a.tile_mask[doff + j0 + t], 1ull << tile);
    }
  }
}

// Smallest superset of mask m made of one contiguous run of set bits: the
// tiles between a column's first and last kept tile are stored too (with
// their exact small values), so the CD addresses a column with one base.
__device__ __forceinline__ unsigned long long run_cover(unsigned long long m) {
  if (m == 0ull) return 0ull;
  const int t0 = __ffsll(static_cast<long long>(m)) - 1;
  const int t1 = 63 - __clzll(static_cast<long long>(m));
  const unsigned long long upto = (t1 >= 63) ? ~0ull : ((2ull << t1) - 1ull);
  return upto & ~((1ull << t0) - 1ull);
}

// (B) per-subdomain exclusive scan of 32 * popcount(mask) over the columns
constexpr int SC_THREADS = 256;
__global__ void __launch_bounds__(SC_THREADS) tile_scan_kernel(const TileArgs a) {
  __shared__ int64_t part[SC_THREADS];
  const int64_t s = blockIdx.x;
  if (a.active != nullptr && a.active[s] == 0) return;
  const int M = a.m_cur[s];
  const int64_t doff = a.dict_off[s];
  const int per = (M + SC_THREADS - 1) / SC_THREADS;
  const int lo = threadIdx.x * per, hi = min(M, lo + per);
  // Run cover (+~12% bytes at C4 over exact masks; one base and one
  // predicate per tile in the CD kernels, which are issue-bound)
  for (int j = lo; j < hi; ++j) a.tile_mask[doff + j] = run_cover(a.tile_mask[doff + j]);
  int64_t acc = 0;
  for (int j = lo; j < hi; ++j) acc += 32 * __popcll(a.tile_mask[doff + j]);
  part[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t run = 0;
    for (int k = 0; k < SC_THREADS; ++k) {
      const int64_t v = part[k];
      part[k] = run;
      run += v;
    }
  }
  __syncthreads();
  int64_t run = part[threadIdx.x];
  for (int j = lo; j < hi; ++j) {
    a.col_off[doff + j] = run;
    run += 32 * __popcll(a.tile_mask[doff + j]);
  }
  if (threadIdx.x == SC_THREADS - 1 && a.packed_total != nullptr) a.packed_total[s] = run;
}

// (C) packed store of the kept tiles (padding rows of a kept tile are zero)
template <int D>
__global__ void __launch_bounds__(TL_THREADS) tile_store_kernel(const TileArgs a) {
  __shared__ TileSmem<D> sm;
  const int64_t s = blockIdx.y;
  if (a.active != nullptr && a.active[s] == 0) return;
  const int64_t r0 = a.row_off[s];
  const int n = static_cast<int>(a.row_off[s + 1] - r0);
  const int p = blockIdx.x * TL_THREADS + threadIdx.x;
  if (static_cast<int>(blockIdx.x) * TL_THREADS >= n) return;
  const bool live = p < n;
  const int row = live ? (a.perm ? a.perm[r0 + p] : p) : 0;
  const int M = a.m_cur[s];
  const int64_t doff = a.dict_off[s];
  const int lane = threadIdx.x & 31;
  const int tile = p >> 5;
  double* Ws = a.W + a.w_off[s];
  double x[D];
#pragma unroll
  for (int k = 0; k < D; ++k) x[k] = live ? a.pts[(r0 + row) * D + k] : 0.0;
  const double mx = live ? a.rowmax[r0 + p] : 0.0;
  const double sum = live ? a.rowsum[r0 + p] : 1.0;
  const unsigned long long below = (1ull << tile) - 1ull;
  for (int j0 = 0; j0 < M; j0 += TL_CHUNK) {
    const int cnt = min(TL_CHUNK, M - j0);
    tl_stage<D>(sm, a.centres, a.widths, doff, j0, cnt);
    for (int t = 0; t < cnt; ++t) {
      const unsigned long long mask = a.tile_mask[doff + j0 + t];  // warp-uniform
      if (!((mask >> tile) & 1ull)) continue;
      double w = 0.0;
      if (live)
        w = __ddiv_rn(exp(__dsub_rn(log_feature<D>(x, &sm.c[t * D], sm.inv[t]), mx)), sum);
      const int slot = __popcll(mask & below);
      Ws[a.col_off[doff + j0 + t] + slot * 32 + lane] = w;
    }
  }
}

}  // namespace pam

using namespace pam;

extern "C" int pam_assemble_tiles_f64(int dim, int64_t S, const int64_t* row_off, const double* pts,
                                      const int32_t* perm, const int64_t* dict_off,
                                      const int32_t* m_cur, const double* centres,
                                      const double* widths, const int64_t* w_off,
                                      const int32_t* active, int32_t max_rows, double tau,
                                      double* rowmax, double* rowsum, uint64_t* tile_mask,
                                      int64_t* col_off, int64_t* packed_total,
                                      int64_t total_slots, double* W, void* stream) {
  if (S < 0 || max_rows < 0 || dim < 1 || dim > 3 || max_rows > 1024) return PAM_ERR_ARG;
  if (S == 0 || max_rows == 0) return PAM_OK;
  cudaStream_t st = as_stream(stream);
  PAM_CUDA_CHECK(cudaMemsetAsync(tile_mask, 0, total_slots * sizeof(uint64_t), st));
  for (int64_t s0 = 0; s0 < S; s0 += 65535) {
    const int64_t cnt = std::min<int64_t>(65535, S - s0);
    TileArgs a{row_off + s0, pts, perm, dict_off + s0, m_cur + s0, centres, widths, w_off + s0,
               active ? active + s0 : nullptr, tau, rowmax, rowsum,
               reinterpret_cast<unsigned long long*>(tile_mask), col_off,
               packed_total ? packed_total + s0 : nullptr, W};
    dim3 grid((unsigned)ceil_div(max_rows, TL_THREADS), (unsigned)cnt);
    if (dim == 1) tile_mask_kernel<1><<<grid, TL_THREADS, 0, st>>>(a);
    else if (dim == 2) tile_mask_kernel<2><<<grid, TL_THREADS, 0, st>>>(a);
    else tile_mask_kernel<3><<<grid, TL_THREADS, 0, st>>>(a);
    PAM_LAUNCH_CHECK("tile_mask_kernel");
    tile_scan_kernel<<<(unsigned)cnt, SC_THREADS, 0, st>>>(a);
    PAM_LAUNCH_CHECK("tile_scan_kernel");
    if (dim == 1) tile_store_kernel<1><<<grid, TL_THREADS, 0, st>>>(a);
    else if (dim == 2) tile_store_kernel<2><<<grid, TL_THREADS, 0, st>>>(a);
    else tile_store_kernel<3><<<grid, TL_THREADS, 0, st>>>(a);
    PAM_LAUNCH_CHECK("tile_store_kernel");
  }
  return PAM_OK;
}
