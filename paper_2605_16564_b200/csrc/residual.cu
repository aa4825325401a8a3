// residual.cu — K3: adaptive-refinement residual, L2 misfit parts, stable
// top-K marking and enrichment for a ragged batch of subdomains.
//
// Replaces (reference) residual_indicators (adaptive.py:133-138) over
// cell_quadrature (geometry.py:204-224), l2_misfit_parts (fields.py:113-121),
// mark (adaptive.py:141-152), _nearest_entry + enrich (adaptive.py:155-210)
// and the dictionary append of fit_adaptive (adaptive.py:267-269).
//
// Determinism: every reduction is a fixed-order tree inside one CTA (no
// floating-point atomics), so reports are bit-reproducible run to run.
// Tie-sensitive quantities (nearest-entry distances, candidate centres,
// duplicate tests) use round-to-nearest intrinsics only (no FMA), matching
// numpy bit for bit; marking compares the residuals exactly.
#include "shepard.cuh"

#include <algorithm>

namespace pam {

constexpr int RES_THREADS = 128;

// ---- K3a: per-cell residual indicator R_i -----------------------------------
template <int D>
__global__ void __launch_bounds__(RES_THREADS)
residual_kernel(const int64_t* __restrict__ row_off, const double* __restrict__ pts,
                const double* __restrict__ values, const int64_t* __restrict__ dict_off,
                const int32_t* __restrict__ m_cur, const double* __restrict__ centres,
                const double* __restrict__ widths, const double* __restrict__ beta,
                const int32_t* __restrict__ quad_order, const double* __restrict__ qoff,
                const double* __restrict__ qw, int log_flag, const int32_t* __restrict__ active,
                double* __restrict__ R, int64_t* err) {
  __shared__ ShepardSmem<D> sm;
  const int64_t s = blockIdx.y;
  if (active != nullptr && active[s] == 0) return;
  const int64_t r0 = row_off[s];
  const int64_t n = row_off[s + 1] - r0;
  if (static_cast<int64_t>(blockIdx.x) * RES_THREADS >= n) return;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * RES_THREADS + threadIdx.x;
  const bool live = i < n;
  const int M = m_cur[s];
  const int64_t doff = dict_off[s];
  const int order = quad_order[s];
  const int nq = (order == 1) ? 1 : (1 << D);
  const int q0 = (order == 1) ? 0 : 1;  // qoff rows: [order-1 point, order-2 points...]

  double c[D];
#pragma unroll
  for (int k = 0; k < D; ++k) c[k] = live ? pts[(r0 + i) * D + k] : 0.0;
  const double kt = live ? values[r0 + i] : 0.0;

  double acc = 0.0;
  for (int q = 0; q < nq; ++q) {
    double x[D];
#pragma unroll
    for (int k = 0; k < D; ++k) x[k] = __dadd_rn(c[k], qoff[(q0 + q) * D + k]);
    double den;
    const double v = shepard_eval_block<D>(sm, x, live, centres, widths, beta, doff, M, &den);
    if (live) {
      if (shepard_degenerate(den)) report_error(err, PAM_ERR_DEGENERATE, r0 + i);
      const double ks = log_flag ? exp(v) : v;
      const double diff = __dsub_rn(ks, kt);
      const double term = __dmul_rn(__dmul_rn(diff, diff), qw[q0 + q]);
      acc = (q == 0) ? term : __dadd_rn(acc, term);
    }
  }
  if (live) R[r0 + i] = acc;
}

// ---- K3b: per-subdomain reductions: num = sum R, den = sum(w) * sum(K^2),
//      rmax = max R (fields.py:113-121; adaptive.py:244-246) -----------------
constexpr int RED_THREADS = 256;
__global__ void __launch_bounds__(RED_THREADS)
reduce_kernel(const int64_t* __restrict__ row_off, const double* __restrict__ R,
              const double* __restrict__ values, const int32_t* __restrict__ quad_order,
              const double* __restrict__ qw, int dim, const int32_t* __restrict__ active,
              double* __restrict__ parts, double* __restrict__ rmax) {
  __shared__ double s_sum[RED_THREADS / 32], s_sq[RED_THREADS / 32], s_max[RED_THREADS / 32];
  const int64_t s = blockIdx.x;
  if (active != nullptr && active[s] == 0) return;
  const int64_t r0 = row_off[s];
  const int64_t n = row_off[s + 1] - r0;
  double sum = 0.0, sq = 0.0, mx = -INFINITY;
  for (int64_t i = threadIdx.x; i < n; i += RED_THREADS) {
    const double r = R[r0 + i];
    const double v = values[r0 + i];
    sum += r;
    sq = fma(v, v, sq);
    mx = fmax(mx, r);
  }
  sum = warp_sum(sum);
  sq = warp_sum(sq);
  mx = warp_max(mx);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s_sum[w] = sum;
    s_sq[w] = sq;
    s_max[w] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0, m = -INFINITY;
    for (int k = 0; k < RED_THREADS / 32; ++k) {
      a += s_sum[k];
      b += s_sq[k];
      m = fmax(m, s_max[k]);
    }
    const int order = quad_order[s];
    const int nq = (order == 1) ? 1 : (1 << dim);
    const int q0 = (order == 1) ? 0 : 1;
    double wsum = 0.0;
    for (int q = 0; q < nq; ++q) wsum += qw[q0 + q];
    parts[2 * s] = a;
    parts[2 * s + 1] = wsum * b;
    rmax[s] = m;
  }
}

// ---- K3c: stable top-K by (R desc, index asc), R > 0 only -------------------
constexpr int MARK_THREADS = 256;
constexpr int MARK_TILE = 2048;
__global__ void __launch_bounds__(MARK_THREADS)
mark_kernel(const int64_t* __restrict__ row_off, const double* __restrict__ R,
            const int32_t* __restrict__ k_top, const int32_t* __restrict__ active, int kcap,
            int32_t* __restrict__ marked, int32_t* __restrict__ n_marked) {
  __shared__ double tile[MARK_TILE];
  __shared__ int s_pos;
  const int64_t s = blockIdx.x;
  if (active != nullptr && active[s] == 0) return;
  const int64_t r0 = row_off[s];
  const int n = static_cast<int>(row_off[s + 1] - r0);
  const int K = min(k_top[s], kcap);
  if (threadIdx.x == 0) s_pos = 0;
  // rank_i = #{j : R_j > R_i} + #{j < i : R_j == R_i}; marked[rank_i] = i
  for (int base = 0; base < n; base += MARK_THREADS) {
    const int i = base + threadIdx.x;
    const double ri = (i < n) ? R[r0 + i] : 0.0;
    int rank = 0;
    for (int t0 = 0; t0 < n; t0 += MARK_TILE) {
      const int cnt = min(MARK_TILE, n - t0);
      __syncthreads();
      for (int t = threadIdx.x; t < cnt; t += MARK_THREADS) tile[t] = R[r0 + t0 + t];
      __syncthreads();
      if (i < n && ri > 0.0) {
        for (int t = 0; t < cnt; ++t) {
          const double rj = tile[t];
          rank += (rj > ri) || (rj == ri && (t0 + t) < i);
        }
      }
    }
    if (i < n && ri > 0.0) {
      if (rank < K) marked[s * (int64_t)kcap + rank] = i;
      atomicAdd(&s_pos, 1);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) n_marked[s] = min(s_pos, K);
}

// ---- K3d: enrichment ----------------------------------------------------------
constexpr int ENR_THREADS = 256;
constexpr double DUPLICATE_TOL = 1e-12;  // adaptive.py:27

struct EnrichArgs {
  const int64_t* row_off;
  const double* pts;
  const int32_t* marked;
  const int32_t* n_marked;
  int kcap;
  const double* eta;
  const int32_t* m_q;
  int mq_cap;
  const double* offsets;
  const double* cell_size;
  const double* box_lo;
  const double* box_hi;
  const int64_t* dict_off;
  const int32_t* dict_cap;
  int32_t* m_cur;
  double* centres;
  double* widths;
  int32_t* gens;
  double* beta;
  int gen;
  const int32_t* active;
  int32_t* n_added;
  int64_t* err;
};

// lexicographic (d2, width, idx) minimum
struct NearKey {
  double d2, w;
  int idx;
};
__device__ __forceinline__ bool near_less(const NearKey& a, const NearKey& b) {
  if (a.d2 != b.d2) return a.d2 < b.d2;
  if (a.w != b.w) return a.w < b.w;
  return a.idx < b.idx;
}

template <int D>
__global__ void __launch_bounds__(ENR_THREADS) enrich_kernel(const EnrichArgs a) {
  extern __shared__ __align__(16) unsigned char enr_smem[];
  const int64_t s = blockIdx.x;
  if (a.active != nullptr && a.active[s] == 0) return;
  const int K = a.n_marked[s];
  const int mq = a.m_q[s];
  const int ncand = K * mq;
  double* cand = reinterpret_cast<double*>(enr_smem);     // ncand * D
  double* cw = cand + (size_t)a.kcap * a.mq_cap * D;      // ncand
  int* keep = reinterpret_cast<int*>(cw + (size_t)a.kcap * a.mq_cap);  // ncand
  __shared__ int s_scan[ENR_THREADS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = ENR_THREADS / 32;
  const int M = a.m_cur[s];
  const int64_t doff = a.dict_off[s];
  const int64_t r0 = a.row_off[s];
  const double eta = a.eta[s];

  // phase 1: one warp per marked cell: parent, width, candidates, duplicate test
  for (int t = warp; t < K; t += nwarps) {
    const int cell = a.marked[s * (int64_t)a.kcap + t];
    double xt[D];
#pragma unroll
    for (int k = 0; k < D; ++k) xt[k] = a.pts[(r0 + cell) * D + k];
    NearKey best{INFINITY, INFINITY, 0x7fffffff};
    for (int m = lane; m < M; m += 32) {
      NearKey key{sqdist_npsum<D>(&a.centres[(doff + m) * D], xt), a.widths[doff + m], m};
      if (near_less(key, best)) best = key;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      NearKey other{__shfl_xor_sync(0xffffffffu, best.d2, o), __shfl_xor_sync(0xffffffffu, best.w, o),
                    __shfl_xor_sync(0xffffffffu, best.idx, o)};
      if (near_less(other, best)) best = other;
    }
    const double width = __dmul_rn(eta, a.widths[doff + best.idx]);
    for (int q = 0; q < mq; ++q) {
      double c[D];
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const double off = a.offsets[((size_t)s * a.mq_cap + q) * D + k];
        double v = __dadd_rn(xt[k], __dmul_rn(off, a.cell_size[k]));
        v = fmin(fmax(v, a.box_lo[s * D + k]), a.box_hi[s * D + k]);  // np.clip (geometry.py:68-70)
        c[k] = v;
      }
      // duplicate only against the EXISTING dictionary (adaptive.py:200-205)
      bool dup = false;
      for (int m = lane; m < M && !dup; m += 32) {
        bool same = fabs(__dsub_rn(a.widths[doff + m], width)) <= DUPLICATE_TOL;
#pragma unroll
        for (int k = 0; k < D; ++k)
          same = same && (fabs(__dsub_rn(a.centres[(doff + m) * D + k], c[k])) <= DUPLICATE_TOL);
        dup = same;
      }
      dup = __any_sync(0xffffffffu, dup);
      if (lane == 0) {
        const int id = t * mq + q;
#pragma unroll
        for (int k = 0; k < D; ++k) cand[id * D + k] = c[k];
        cw[id] = width;
        keep[id] = dup ? 0 : 1;
      }
    }
  }
  __syncthreads();
  // phase 2: ordered compaction (marked order, then offset order)
  const int per = (ncand + ENR_THREADS - 1) / ENR_THREADS;
  const int lo = threadIdx.x * per, hi = min(ncand, lo + per);
  int cnt = 0;
  for (int id = lo; id < hi; ++id) cnt += keep[id];
  s_scan[threadIdx.x] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int k = 0; k < ENR_THREADS; ++k) {
      const int v = s_scan[k];
      s_scan[k] = run;
      run += v;
    }
    if (M + run > a.dict_cap[s]) {
      report_error(a.err, PAM_ERR_UNSUPPORTED, s);
      run = 0;
      for (int k = 0; k < ENR_THREADS; ++k) s_scan[k] = 0;
    }
    a.n_added[s] = run;
  }
  __syncthreads();
  const int total_added = a.n_added[s];
  if (total_added > 0) {
    int pos = M + s_scan[threadIdx.x];
    for (int id = lo; id < hi; ++id) {
      if (!keep[id]) continue;
      const int64_t slot = doff + pos;
#pragma unroll
      for (int k = 0; k < D; ++k) a.centres[slot * D + k] = cand[id * D + k];
      a.widths[slot] = cw[id];
      a.gens[slot] = a.gen;
      a.beta[slot] = 0.0;  // warm start zero-extension (adaptive.py:268)
      ++pos;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) a.m_cur[s] = M + total_added;
}

size_t enrich_smem_bytes(int kcap, int mq_cap, int dim) {
  const size_t n = (size_t)kcap * mq_cap;
  return n * dim * sizeof(double) + n * sizeof(double) + n * sizeof(int);
}

}  // namespace pam

using namespace pam;

extern "C" int pam_residual_f64(int dim, int64_t S, const int64_t* row_off, const double* pts,
                                const double* values, const int64_t* dict_off,
                                const int32_t* m_cur, const double* centres,
                                const double* widths, const double* beta,
                                const int32_t* quad_order, const double* qoff, const double* qw,
                                int32_t log_flag, const int32_t* active, int32_t max_rows,
                                double* R, double* parts, double* rmax, int64_t* err,
                                void* stream) {
  if (S < 0 || dim < 1 || dim > 3 || max_rows < 0) return PAM_ERR_ARG;
  if (S == 0) return PAM_OK;
  cudaStream_t st = as_stream(stream);
  for (int64_t s0 = 0; s0 < S; s0 += 65535) {
    const int64_t cnt = std::min<int64_t>(65535, S - s0);
    dim3 grid((unsigned)ceil_div(std::max(max_rows, 1), RES_THREADS), (unsigned)cnt);
    const int32_t* act = active ? active + s0 : nullptr;
    switch (dim) {
      case 1:
        residual_kernel<1><<<grid, RES_THREADS, 0, st>>>(row_off + s0, pts, values, dict_off + s0,
                                                         m_cur + s0, centres, widths, beta,
                                                         quad_order + s0, qoff, qw, log_flag, act,
                                                         R, err);
        break;
      case 2:
        residual_kernel<2><<<grid, RES_THREADS, 0, st>>>(row_off + s0, pts, values, dict_off + s0,
                                                         m_cur + s0, centres, widths, beta,
                                                         quad_order + s0, qoff, qw, log_flag, act,
                                                         R, err);
        break;
      default:
        residual_kernel<3><<<grid, RES_THREADS, 0, st>>>(row_off + s0, pts, values, dict_off + s0,
                                                         m_cur + s0, centres, widths, beta,
                                                         quad_order + s0, qoff, qw, log_flag, act,
                                                         R, err);
        break;
    }
    PAM_LAUNCH_CHECK("residual_kernel");
  }
  reduce_kernel<<<(unsigned)S, RED_THREADS, 0, st>>>(row_off, R, values, quad_order, qw, dim,
                                                     active, parts, rmax);
  PAM_LAUNCH_CHECK("reduce_kernel");
  return PAM_OK;
}

extern "C" int pam_mark_f64(int64_t S, const int64_t* row_off, const double* R,
                            const int32_t* k_top, const int32_t* active, int32_t kcap,
                            int32_t* marked, int32_t* n_marked, void* stream) {
  if (S < 0 || kcap < 1) return PAM_ERR_ARG;
  if (S == 0) return PAM_OK;
  mark_kernel<<<(unsigned)S, MARK_THREADS, 0, as_stream(stream)>>>(row_off, R, k_top, active, kcap,
                                                                   marked, n_marked);
  PAM_LAUNCH_CHECK("mark_kernel");
  return PAM_OK;
}

extern "C" int pam_enrich_f64(int dim, int64_t S, const int64_t* row_off, const double* pts,
                              const int32_t* marked, const int32_t* n_marked, int32_t kcap,
                              const double* eta, const int32_t* m_q, int32_t mq_cap,
                              const double* offsets, const double* cell_size,
                              const double* box_lo, const double* box_hi,
                              const int64_t* dict_off, const int32_t* dict_cap, int32_t* m_cur,
                              double* centres, double* widths, int32_t* gens, double* beta,
                              int32_t gen, const int32_t* active, int32_t* n_added,
                              int64_t* err, void* stream) {
  if (S < 0 || dim < 1 || dim > 3 || kcap < 1 || mq_cap < 1) return PAM_ERR_ARG;
  if (S == 0) return PAM_OK;
  const size_t smem = enrich_smem_bytes(kcap, mq_cap, dim);
  if (smem > 200 * 1024) {
    set_last_error("pam_enrich_f64: k_top * m_q too large for the shared-memory candidate list");
    return PAM_ERR_UNSUPPORTED;
  }
  EnrichArgs a{row_off, pts,    marked,  n_marked, kcap,   eta,   m_q,   mq_cap,
               offsets, cell_size, box_lo, box_hi, dict_off, dict_cap, m_cur, centres,
               widths,  gens,   beta,    gen,      active, n_added, err};
  cudaStream_t st = as_stream(stream);
  switch (dim) {
    case 1:
      PAM_CUDA_CHECK(cudaFuncSetAttribute(enrich_kernel<1>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      enrich_kernel<1><<<(unsigned)S, ENR_THREADS, smem, st>>>(a);
      break;
    case 2:
      PAM_CUDA_CHECK(cudaFuncSetAttribute(enrich_kernel<2>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      enrich_kernel<2><<<(unsigned)S, ENR_THREADS, smem, st>>>(a);
      break;
    default:
      PAM_CUDA_CHECK(cudaFuncSetAttribute(enrich_kernel<3>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      enrich_kernel<3><<<(unsigned)S, ENR_THREADS, smem, st>>>(a);
      break;
  }
  PAM_LAUNCH_CHECK("enrich_kernel");
  return PAM_OK;
}
