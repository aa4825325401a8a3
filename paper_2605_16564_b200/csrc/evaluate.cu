// evaluate.cu — K4: fused global evaluation of the piecewise surrogate.
//
// Replaces GlobalSurrogate.evaluate (reference partition.py:132-143) =
// locate_many (geometry.py:242-258) + per-owner LocalSurrogate.evaluate
// (rbf.py:152-192).  Pipeline (all on one stream, no host round trip):
//
//   1. locate: per point, per axis, the unique box index i with
//      edges[i] <= x < edges[i+1] (<= on the global upper face) — the
//      half-open rule of Box.contains_many evaluated against host-identical
//      edges, so ownership is bit-exact.  Points outside every
//      box report the FIRST offending index (atomicMin).
//   2. counting sort of point ids by owner (histogram, exclusive scan,
//      scatter) so each subdomain's dictionary is read from HBM once per
//      128-point tile and served to the tile from shared memory.
//   3. eval: per tile, per owner run, the two-pass Shepard sum with the
//      dictionary staged in smem; exp() of the blend when log_transform;
//      results scattered back to input order.
//
// Roofline: FP64-pipe bound (M*(3d+4+E) flops per point vs 8d+8 bytes).
#include "shepard.cuh"

#include <algorithm>

namespace pam {

constexpr int EVAL_TILE = 128;

template <int D>
__global__ void locate_kernel(int64_t P, const double* __restrict__ pts,
                              const int32_t* __restrict__ shape, const double* __restrict__ edges,
                              int64_t* __restrict__ owner, int64_t* err) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < P;
       j += (int64_t)gridDim.x * blockDim.x) {
    int64_t own = 0, stride = 1;
    bool ok = true;
    const double* e = edges;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const int p = shape[k];
      const double x = pts[j * D + k];
      // largest i in [0, p-1] with e[i] <= x
      int lo = 0, hi = p - 1;
      if (!(x >= e[0])) ok = false;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (e[mid] <= x) lo = mid; else hi = mid - 1;
      }
      const bool last = (lo == p - 1);
      if (last ? !(x <= e[p]) : !(x < e[lo + 1])) ok = false;
      own += stride * lo;
      stride *= p;
      e += p + 1;
    }
    if (!ok) {
      report_error(err, PAM_ERR_OUTSIDE, j);
      own = -1;
    }
    owner[j] = own;
  }
}

__global__ void histogram_kernel(int64_t P, const int64_t* __restrict__ owner,
                                 unsigned long long* __restrict__ counts) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < P;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = owner[j];
    if (o >= 0) atomicAdd(&counts[o], 1ull);
  }
}

// exclusive scan over S counts, single CTA (S up to a few 1e5)
constexpr int SCAN_THREADS = 1024;
__global__ void __launch_bounds__(SCAN_THREADS)
scan_kernel(int64_t S, const unsigned long long* __restrict__ counts,
            unsigned long long* __restrict__ start, unsigned long long* __restrict__ cursor) {
  __shared__ unsigned long long part[SCAN_THREADS];
  const int64_t per = (S + SCAN_THREADS - 1) / SCAN_THREADS;
  const int64_t lo = threadIdx.x * per, hi = min(S, lo + per);
  unsigned long long acc = 0;
  for (int64_t i = lo; i < hi; ++i) acc += counts[i];
  part[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long run = 0;
    for (int k = 0; k < SCAN_THREADS; ++k) {
      const unsigned long long v = part[k];
      part[k] = run;
      run += v;
    }
  }
  __syncthreads();
  unsigned long long run = part[threadIdx.x];
  for (int64_t i = lo; i < hi; ++i) {
    start[i] = run;
    cursor[i] = run;
    run += counts[i];
  }
  if (threadIdx.x == SCAN_THREADS - 1) start[S] = run;  // last range ends at the total
}

__global__ void scatter_kernel(int64_t P, const int64_t* __restrict__ owner,
                               unsigned long long* __restrict__ cursor, int64_t* __restrict__ perm,
                               int64_t* __restrict__ sorted_owner) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < P;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = owner[j];
    if (o < 0) continue;
    const unsigned long long pos = atomicAdd(&cursor[o], 1ull);
    perm[pos] = j;
    sorted_owner[pos] = o;
  }
}

template <int D>
__global__ void __launch_bounds__(EVAL_TILE)
eval_kernel(int64_t P, const double* __restrict__ pts, const int64_t* __restrict__ perm,
            const int64_t* __restrict__ sorted_owner, const int64_t* __restrict__ dict_off,
            const int32_t* __restrict__ m_cur, const double* __restrict__ centres,
            const double* __restrict__ widths, const double* __restrict__ beta,
            const int32_t* __restrict__ log_flag, double* __restrict__ out, int64_t* err) {
  __shared__ ShepardSmem<D> sm;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * EVAL_TILE;
  const int64_t tend = min(P, t0 + EVAL_TILE);
  const int64_t mine = t0 + threadIdx.x;
  const bool have = mine < tend;
  const int64_t my_owner = have ? sorted_owner[mine] : -1;
  const int64_t j = have ? perm[mine] : 0;
  double x[D];
#pragma unroll
  for (int k = 0; k < D; ++k) x[k] = have ? pts[j * D + k] : 0.0;
  int64_t cur = t0;
  while (cur < tend) {
    const int64_t s = sorted_owner[cur];  // block-uniform
    const bool live = have && my_owner == s;
    double den;
    const double v = shepard_eval_direct<D>(sm, x, live, centres, widths, beta, dict_off[s],
                                            m_cur[s], &den);
    if (live) {
      if (shepard_degenerate(den)) report_error(err, PAM_ERR_DEGENERATE, j);
      out[j] = log_flag[s] ? exp(v) : v;
    }
    // advance past this owner's run (sorted => contiguous)
    int64_t nxt = cur;
    while (nxt < tend && sorted_owner[nxt] == s) ++nxt;
    cur = nxt;
  }
}

// single-dictionary Shepard evaluation (rbf.py:152-167 / 190-192); same
// arithmetic as eval_kernel, so LocalSurrogate and GlobalSurrogate agree bit for bit
template <int D>
__global__ void __launch_bounds__(EVAL_TILE)
shepard_single_kernel(int64_t P, const double* __restrict__ pts, int M,
                      const double* __restrict__ centres, const double* __restrict__ widths,
                      const double* __restrict__ beta, int exp_out, double* __restrict__ out,
                      int64_t* err) {
  __shared__ ShepardSmem<D> sm;
  const int64_t j = static_cast<int64_t>(blockIdx.x) * EVAL_TILE + threadIdx.x;
  const bool live = j < P;
  double x[D];
#pragma unroll
  for (int k = 0; k < D; ++k) x[k] = live ? pts[j * D + k] : 0.0;
  double den;
  const double v = shepard_eval_direct<D>(sm, x, live, centres, widths, beta, 0, M, &den);
  if (live) {
    if (shepard_degenerate(den)) report_error(err, PAM_ERR_DEGENERATE, j);
    out[j] = exp_out ? exp(v) : v;
  }
}

int grid_for(int64_t n, int threads) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), 148 * 32));
}

}  // namespace pam

using namespace pam;

extern "C" int64_t pam_eval_workspace_bytes(int64_t P, int64_t S) {
  // owner, perm, sorted_owner (P each) + counts, cursor (S) + start (S+1)
  return 3 * P * 8 + (3 * S + 1) * 8 + 256;
}

extern "C" int pam_locate_f64(int dim, int64_t P, const double* pts, const int32_t* shape,
                              const double* edges, int64_t* owner, int64_t* err, void* stream) {
  if (dim < 1 || dim > 3 || P < 0) return PAM_ERR_ARG;
  if (P == 0) return PAM_OK;
  cudaStream_t st = as_stream(stream);
  const int g = grid_for(P, 256);
  if (dim == 1) locate_kernel<1><<<g, 256, 0, st>>>(P, pts, shape, edges, owner, err);
  else if (dim == 2) locate_kernel<2><<<g, 256, 0, st>>>(P, pts, shape, edges, owner, err);
  else locate_kernel<3><<<g, 256, 0, st>>>(P, pts, shape, edges, owner, err);
  PAM_LAUNCH_CHECK("locate_kernel");
  return PAM_OK;
}

extern "C" int pam_eval_f64(int dim, int64_t P, const double* pts, const int32_t* shape,
                            const double* edges, int64_t S, const int64_t* dict_off,
                            const int32_t* m_cur, const double* centres, const double* widths,
                            const double* beta, const int32_t* log_flag, double* out, void* work,
                            int64_t* err, void* stream) {
  if (dim < 1 || dim > 3 || P < 0 || S < 1 || !work) return PAM_ERR_ARG;
  if (P == 0) return PAM_OK;
  cudaStream_t st = as_stream(stream);
  char* w = static_cast<char*>(work);
  int64_t* owner = reinterpret_cast<int64_t*>(w);
  int64_t* perm = owner + P;
  int64_t* sorted_owner = perm + P;
  unsigned long long* counts = reinterpret_cast<unsigned long long*>(sorted_owner + P);
  unsigned long long* cursor = counts + S;
  unsigned long long* start = cursor + S;
  int rc = pam_locate_f64(dim, P, pts, shape, edges, owner, err, stream);
  if (rc != PAM_OK) return rc;
  PAM_CUDA_CHECK(cudaMemsetAsync(counts, 0, S * sizeof(unsigned long long), st));
  const int g = grid_for(P, 256);
  histogram_kernel<<<g, 256, 0, st>>>(P, owner, counts);
  PAM_LAUNCH_CHECK("histogram_kernel");
  scan_kernel<<<1, SCAN_THREADS, 0, st>>>(S, counts, start, cursor);
  PAM_LAUNCH_CHECK("scan_kernel");
  // points that failed to locate are not scattered; pad the tail so every
  // sorted slot is defined (error path only: the caller raises).
  PAM_CUDA_CHECK(cudaMemsetAsync(sorted_owner, 0, P * sizeof(int64_t), st));
  PAM_CUDA_CHECK(cudaMemsetAsync(perm, 0, P * sizeof(int64_t), st));
  scatter_kernel<<<g, 256, 0, st>>>(P, owner, cursor, perm, sorted_owner);
  PAM_LAUNCH_CHECK("scatter_kernel");
  const int64_t tiles = ceil_div(P, EVAL_TILE);
  if (tiles > 0x7fffffffLL) return PAM_ERR_ARG;
  if (dim == 1)
    eval_kernel<1><<<(unsigned)tiles, EVAL_TILE, 0, st>>>(P, pts, perm, sorted_owner, dict_off, m_cur,
                                                          centres, widths, beta, log_flag, out, err);
  else if (dim == 2)
    eval_kernel<2><<<(unsigned)tiles, EVAL_TILE, 0, st>>>(P, pts, perm, sorted_owner, dict_off, m_cur,
                                                          centres, widths, beta, log_flag, out, err);
  else
    eval_kernel<3><<<(unsigned)tiles, EVAL_TILE, 0, st>>>(P, pts, perm, sorted_owner, dict_off, m_cur,
                                                          centres, widths, beta, log_flag, out, err);
  PAM_LAUNCH_CHECK("eval_kernel");
  return PAM_OK;
}

extern "C" int pam_shepard_eval_f64(int dim, int64_t P, const double* pts, int64_t M,
                                    const double* centres, const double* widths,
                                    const double* beta, int32_t exp_out, double* out, int64_t* err,
                                    void* stream) {
  if (dim < 1 || dim > 3 || P < 0 || M < 1 || M > 0x7fffffff) return PAM_ERR_ARG;
  if (P == 0) return PAM_OK;
  cudaStream_t st = as_stream(stream);
  const int64_t tiles = ceil_div(P, EVAL_TILE);
  if (dim == 1)
    shepard_single_kernel<1><<<(unsigned)tiles, EVAL_TILE, 0, st>>>(P, pts, (int)M, centres, widths,
                                                                    beta, exp_out, out, err);
  else if (dim == 2)
    shepard_single_kernel<2><<<(unsigned)tiles, EVAL_TILE, 0, st>>>(P, pts, (int)M, centres, widths,
                                                                    beta, exp_out, out, err);
  else
    shepard_single_kernel<3><<<(unsigned)tiles, EVAL_TILE, 0, st>>>(P, pts, (int)M, centres, widths,
                                                                    beta, exp_out, out, err);
  PAM_LAUNCH_CHECK("shepard_single_kernel");
  return PAM_OK;
}
