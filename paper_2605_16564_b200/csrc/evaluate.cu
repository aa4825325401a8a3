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
//      scatter; 32-bit indices when P and S fit) so each subdomain's
//      dictionary is read once per 128-point warp tile (from L2) and served
//      to the warp from shared memory.
//   3. eval: one warp per 128 sorted points (4 per lane), per owner run the one-pass
//      Shepard sum with a table-driven FP64 exp (below); exp() of the blend
//      when log_transform; results scattered back to input order.
//
// Roofline: FP64-pipe bound (M*(3d+4+E) flops per point vs 8d+8 bytes).
#include "shepard.cuh"

#include <string.h>

#include <algorithm>
#include <type_traits>

namespace pam {

template <int D, typename IdxT>
__global__ void locate_kernel(int64_t P, const double* __restrict__ pts,
                              const int32_t* __restrict__ shape, const double* __restrict__ edges,
                              IdxT* __restrict__ owner, int64_t* err) {
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
    owner[j] = static_cast<IdxT>(own);
  }
}

// Arbitrary half-open boxes (geometry.py:54-66, 242-258): per point the boxes are
// tested in order; owner = the first box containing it.  A second containing box
// records min over points of (second box << 40 | point) in flags[0] (the
// reference raises for the FIRST box, in order, that re-claims a point, and within
// it the smallest point index); a point in no box records its index in flags[1].
template <int D, typename IdxT>
__global__ void locate_boxes_kernel(int64_t P, const double* __restrict__ pts, int64_t S,
                                    const double* __restrict__ lo, const double* __restrict__ hi,
                                    const int32_t* __restrict__ open_hi, IdxT* __restrict__ owner,
                                    unsigned long long* flags) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < P;
       j += (int64_t)gridDim.x * blockDim.x) {
    double x[D];
#pragma unroll
    for (int k = 0; k < D; ++k) x[k] = pts[j * D + k];
    int64_t own = -1;
    for (int64_t i = 0; i < S; ++i) {
      bool in = true;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const double l = lo[i * D + k], h = hi[i * D + k];
        in = in && (x[k] >= l) && (open_hi[i * D + k] ? (x[k] < h) : (x[k] <= h));
      }
      if (in) {
        if (own < 0) {
          own = i;
        } else {
          atomicMin(flags, (static_cast<unsigned long long>(i) << 40) | static_cast<unsigned long long>(j));
          break;
        }
      }
    }
    if (own < 0) atomicMin(flags + 1, static_cast<unsigned long long>(j));
    owner[j] = static_cast<IdxT>(own);
  }
}

// error word from the two flags: a doubly claimed point wins over an unclaimed one
// (the reference checks claims inside its box loop, coverage after it)
__global__ void locate_boxes_finish_kernel(const unsigned long long* flags, int64_t* err) {
  if (flags[0] != ~0ull) report_error(err, PAM_ERR_CLAIMED, static_cast<int64_t>(flags[0]));
  else if (flags[1] != ~0ull) report_error(err, PAM_ERR_OUTSIDE, static_cast<int64_t>(flags[1]));
}

// unsigned counterpart for atomicAdd (int32 -> unsigned, int64 -> unsigned long long)
template <typename IdxT>
using UIdx = std::conditional_t<sizeof(IdxT) == 8, unsigned long long, unsigned int>;

template <typename IdxT>
__global__ void histogram_kernel(int64_t P, const IdxT* __restrict__ owner, IdxT* __restrict__ counts) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < P;
       j += (int64_t)gridDim.x * blockDim.x) {
    const IdxT o = owner[j];
    if (o >= 0) atomicAdd(reinterpret_cast<UIdx<IdxT>*>(&counts[o]), 1u);
  }
}

// exclusive scan over S counts, single CTA (S up to a few 1e5); start[S] =
// number of located points (the evaluation's sorted length)
constexpr int SCAN_THREADS = 1024;
template <typename IdxT>
__global__ void __launch_bounds__(SCAN_THREADS)
scan_kernel(int64_t S, const IdxT* __restrict__ counts, IdxT* __restrict__ start, IdxT* __restrict__ cursor) {
  __shared__ IdxT part[SCAN_THREADS];
  const int64_t per = (S + SCAN_THREADS - 1) / SCAN_THREADS;
  const int64_t lo = threadIdx.x * per, hi = min(S, lo + per);
  IdxT acc = 0;
  for (int64_t i = lo; i < hi; ++i) acc += counts[i];
  part[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    IdxT run = 0;
    for (int k = 0; k < SCAN_THREADS; ++k) {
      const IdxT v = part[k];
      part[k] = run;
      run += v;
    }
  }
  __syncthreads();
  IdxT run = part[threadIdx.x];
  for (int64_t i = lo; i < hi; ++i) {
    start[i] = run;
    cursor[i] = run;
    run += counts[i];
  }
  if (threadIdx.x == SCAN_THREADS - 1) start[S] = run;  // last range ends at the total
}

template <typename IdxT>
__global__ void scatter_kernel(int64_t P, const IdxT* __restrict__ owner, IdxT* __restrict__ cursor,
                               IdxT* __restrict__ perm, IdxT* __restrict__ sorted_owner) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < P;
       j += (int64_t)gridDim.x * blockDim.x) {
    const IdxT o = owner[j];
    if (o < 0) continue;
    const IdxT pos = static_cast<IdxT>(
        atomicAdd(reinterpret_cast<UIdx<IdxT>*>(&cursor[o]), 1u));
    perm[pos] = static_cast<IdxT>(j);
    sorted_owner[pos] = o;
  }
}

// ----------------------------------------------------------------------------
// K4 evaluation kernel: one WARP per 32*PT consecutive owner-sorted points
// (PT points per lane), no block-wide barriers.  For each owner run inside the
// warp the owner's dictionary is streamed 32 entries at a time: lane l loads
// entry j0+l, converts it to (centre, g = K/(2w^2), beta) in a per-warp shared
// block, and every lane then reads the entries as broadcasts and accumulates
// its PT points (register blocking: one staged entry feeds PT points).
//
// exp() of the (<= 0) log-feature uses a table-driven FP64 exponential that
// spends 11 FP64 instructions instead of libdevice's ~20 (the FP64 pipe is the
// binding roofline):
//   t = -g * d^2 = L * 2048/ln2 with g = K/(2w^2), K = 2048/ln2,
//   n = rint(t) by the 1.5*2^52 shift (one DFMA), f = t - n in [-1/2, 1/2]
//   exactly rounded by one DFMA, 2^(f/2048) by a degree-3 polynomial
//   (truncation <= 3.4e-17 relative), 2^(n/2048) = 2^(n>>11) * T[n & 2047]
//   with T in shared memory and 2^(n>>11) added into T's exponent field by an
//   integer add (no FP64 op).  Terms below 2^-1022 are exactly 0; a point
//   whose every term underflows (den < 1e-280, ~27 widths from all entries) is
//   redone with the reference's exact max-shifted two-pass form.
// Per-term relative error ~1e-16*(1+|L|), the same order as the reference's
// own rounding of L (rbf.py:87-90); values agree with the oracle to ~1e-14.

constexpr int XT_BITS = 11;
constexpr int XT = 1 << XT_BITS;
constexpr int EVAL_WARPS = 8;  // warps per CTA
constexpr double EXP_K = 2954.639443740597;   // 2048 / ln 2
constexpr double EXP_C1 = 3.384507717577858e-04;   // ln2/2048 (exact scaling of ln2)
constexpr double EXP_C2 = 5.72744624517204e-08;    // (ln2/2048)^2 / 2
constexpr double EXP_C3 = 6.461528672932365e-12;   // (ln2/2048)^3 / 6
constexpr double EXP_SHIFT = 6755399441055744.0;   // 1.5 * 2^52
constexpr long long EXP_SHIFT_BITS = 0x4338000000000000LL;
constexpr long long EXP_NMIN = -1022LL * XT;        // 2^(n/2048) >= 2^-1022

// table word j: the bits of 2^(j/2048) with (j << 9) subtracted from the high
// word, so hi + (n << 9) == hi(2^(j/2048)) + ((n >> 11) << 20) for
// n = 2048 (n >> 11) + j: one integer multiply-add applies the 2^(n >> 11)
// scale (see ensure_exp2_table)
__device__ unsigned long long g_exp2_table[XT];

// exp(-g * d2) with g = K/(2 w^2) -- see the block comment above
__device__ __forceinline__ double exp_neg_scaled(double d2, double g, const unsigned long long* tab) {
  const double s = fma(d2, -g, EXP_SHIFT);
  const double nd = s - EXP_SHIFT;
  const double f = fma(-g, d2, -nd);
  const long long sb = __double_as_longlong(s);
  const unsigned lo = static_cast<unsigned>(sb);
  const unsigned long long tw = tab[lo & (XT - 1)];
  const unsigned hi = static_cast<unsigned>(tw >> 32) + (lo << 9);
  const double Ts = __hiloint2double(static_cast<int>(hi), static_cast<int>(static_cast<unsigned>(tw)));
  const double p = fma(f, fma(f, fma(f, EXP_C3, EXP_C2), EXP_C1), 1.0);
  // terms below 2^-1022 (and |t| beyond the shift trick's range, where f and
  // the scale are meaningless) are exactly 0: a select, not an FP64 op
  return (sb >= EXP_SHIFT_BITS + EXP_NMIN) ? Ts * p : 0.0;
}

// the reference's exact max-shifted two-pass Shepard sum (rbf.py:152-167) for
// one point, reading the dictionary from global memory (underflow fallback)
template <int D>
__device__ double shepard_exact_point(const double* x, const double* centres, const double* widths,
                                      const double* beta, int64_t doff, int M, double* den_out) {
  double mx = -INFINITY;
  for (int t = 0; t < M; ++t) {
    double c[D];
#pragma unroll
    for (int k = 0; k < D; ++k) c[k] = centres[(doff + t) * D + k];
    mx = fmax(mx, log_feature<D>(x, c, inv_two_sigma_sq(widths[doff + t])));
  }
  double num = 0.0, den = 0.0;
  for (int t = 0; t < M; ++t) {
    double c[D];
#pragma unroll
    for (int k = 0; k < D; ++k) c[k] = centres[(doff + t) * D + k];
    const double e = exp(__dsub_rn(log_feature<D>(x, c, inv_two_sigma_sq(widths[doff + t])), mx));
    num = fma(e, beta[doff + t], num);
    den = __dadd_rn(den, e);
  }
  *den_out = den;
  return num / den;
}

// sorted_owner == nullptr: single-dictionary mode (LocalSurrogate.evaluate /
// shepard_eval, rbf.py:152-192): every point belongs to dictionary 0 of
// size single_m, log transform = single_exp.  perm == nullptr: identity.
template <int D, int PT, typename IdxT>
__global__ void __launch_bounds__(EVAL_WARPS * 32)
eval_kernel(int64_t P, const double* __restrict__ pts, const IdxT* __restrict__ perm,
            const IdxT* __restrict__ sorted_owner, const IdxT* __restrict__ n_sorted,
            const int64_t* __restrict__ dict_off,
            const int32_t* __restrict__ m_cur, const double* __restrict__ centres,
            const double* __restrict__ widths, const double* __restrict__ beta,
            const int32_t* __restrict__ log_flag, int single_m, int single_exp,
            double* __restrict__ out, int64_t* err, unsigned long long* queue) {
  constexpr int REC = (D + 2 + 1) & ~1;  // staged record: centre, g, beta (16-byte aligned)
  __shared__ unsigned long long tab[XT];
  __shared__ __align__(16) double stage[EVAL_WARPS][32 * REC];
  for (int i = threadIdx.x; i < XT; i += blockDim.x) tab[i] = g_exp2_table[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  double* const st = stage[warp];
  // sorted mode: only the located points were sorted (start[S]); the rest is
  // the error path (the caller raises)
  if (n_sorted) P = static_cast<int64_t>(*n_sorted);
  const int64_t n_tiles = (P + 32 * PT - 1) / (32 * PT);
  // persistent warps pulling 32*PT-point tiles from a queue counter in the
  // caller's workspace (balanced whatever the owner-run mix of a tile and
  // however many CTAs are resident; no global state, so concurrent calls on
  // different streams are independent); queue == nullptr: one tile per warp
  int64_t tile = static_cast<int64_t>(blockIdx.x) * EVAL_WARPS + warp;
  while (true) {
    if (queue) {
      unsigned long long tq = 0;
      if (lane == 0) tq = atomicAdd(queue, 1ull);
      tile = static_cast<int64_t>(__shfl_sync(0xffffffffu, tq, 0));
    }
    if (tile >= n_tiles) break;
    const int64_t base = tile * (32 * PT);
    bool have[PT];
    int64_t own[PT], idx[PT];
    double x[PT][D];
#pragma unroll
    for (int p = 0; p < PT; ++p) {
      const int64_t pos = base + 32 * p + lane;
      have[p] = pos < P;
      own[p] = have[p] ? (sorted_owner ? static_cast<int64_t>(sorted_owner[pos]) : 0) : INT64_MAX;
      idx[p] = have[p] ? (perm ? static_cast<int64_t>(perm[pos]) : pos) : 0;
#pragma unroll
      for (int k = 0; k < D; ++k) x[p][k] = have[p] ? pts[idx[p] * D + k] : 0.0;
    }
    // owners are nondecreasing along the sorted positions: lane 0's first
    // point holds the tile's smallest owner
    int64_t cur = __shfl_sync(0xffffffffu, own[0], 0);
    while (true) {
      const int64_t s = cur;
      const int64_t doff = dict_off ? dict_off[s] : 0;
      const int M = m_cur ? m_cur[s] : single_m;
      double num[PT], den[PT];
#pragma unroll
      for (int p = 0; p < PT; ++p) num[p] = den[p] = 0.0;
      for (int j0 = 0; j0 < M; j0 += 32) {
        const int cnt = min(32, M - j0);
        __syncwarp();
        if (lane < cnt) {
          const int64_t e = doff + j0 + lane;
          double* r = st + lane * REC;
#pragma unroll
          for (int k = 0; k < D; ++k) r[k] = centres[e * D + k];
          r[D] = __dmul_rn(inv_two_sigma_sq(widths[e]), EXP_K);
          r[D + 1] = beta[e];
        }
        __syncwarp();
#pragma unroll 2
        for (int t = 0; t < cnt; ++t) {
          // broadcast 16-byte loads of the staged record
          double rec[REC];
#pragma unroll
          for (int q = 0; q < REC / 2; ++q) {
            const double2 v = reinterpret_cast<const double2*>(st + t * REC)[q];
            rec[2 * q] = v.x;
            rec[2 * q + 1] = v.y;
          }
          const double g = rec[D], b = rec[D + 1];
#pragma unroll
          for (int p = 0; p < PT; ++p) {
            double d2 = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) {
              const double dk = x[p][k] - rec[k];
              d2 = fma(dk, dk, d2);
            }
            const double e = exp_neg_scaled(d2, g, tab);
            num[p] = fma(e, b, num[p]);
            den[p] += e;
          }
        }
      }
      const int lf = log_flag ? log_flag[s] : single_exp;
#pragma unroll
      for (int p = 0; p < PT; ++p) {
        if (have[p] && own[p] == s) {
          double dn = den[p], v;
          if (dn >= 1e-280) {
            v = num[p] / dn;
          } else {
            v = shepard_exact_point<D>(x[p], centres, widths, beta, doff, M, &dn);
          }
          if (shepard_degenerate(dn)) report_error(err, PAM_ERR_DEGENERATE, idx[p]);
          out[idx[p]] = lf ? exp(v) : v;
        }
      }
      // next owner present in this tile
      int64_t nxt = INT64_MAX;
#pragma unroll
      for (int p = 0; p < PT; ++p)
        if (own[p] > s && own[p] < nxt) nxt = own[p];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const int64_t other = __shfl_xor_sync(0xffffffffu, nxt, o);
        nxt = other < nxt ? other : nxt;
      }
      if (nxt == INT64_MAX) break;
      cur = nxt;
    }
    if (!queue) break;
  }
}

constexpr int EVAL_PT = 4;  // points per lane (register blocking; 2 measured slower)
constexpr int MAX_DEVICES = 64;

int current_device(int* dev) {
  PAM_CUDA_CHECK(cudaGetDevice(dev));
  if (*dev < 0 || *dev >= MAX_DEVICES) {
    set_last_error("device ordinal beyond the library's per-device tables");
    return PAM_ERR_ARG;
  }
  return PAM_OK;
}

// the 2^(j/2048) table is uploaded once per device (the __device__ symbol
// exists per device)
int ensure_exp2_table() {
  static bool done[MAX_DEVICES] = {};
  int dev = 0;
  const int rc = current_device(&dev);
  if (rc != PAM_OK) return rc;
  if (done[dev]) return PAM_OK;
  unsigned long long h[XT];
  for (int j = 0; j < XT; ++j) {
    const double t = static_cast<double>(exp2l(static_cast<long double>(j) / XT));
    unsigned long long b;
    memcpy(&b, &t, sizeof(b));
    h[j] = b - (static_cast<unsigned long long>(static_cast<unsigned>(j) << 9) << 32);
  }
  PAM_CUDA_CHECK(cudaMemcpyToSymbol(g_exp2_table, h, sizeof(h)));
  done[dev] = true;
  return PAM_OK;
}

template <int D, typename IdxT>
int launch_eval(cudaStream_t st, int64_t P, const double* pts, const IdxT* perm,
                const IdxT* sorted_owner, const IdxT* n_sorted, const int64_t* dict_off, const int32_t* m_cur,
                const double* centres, const double* widths, const double* beta,
                const int32_t* log_flag, int single_m, int single_exp, double* out, int64_t* err,
                unsigned long long* queue) {
  int rc = ensure_exp2_table();
  if (rc != PAM_OK) return rc;
  constexpr int PT = EVAL_PT;
  auto kernel = eval_kernel<D, PT, IdxT>;
  static int grid_cap[MAX_DEVICES] = {};  // resident CTAs of one wave, per device
  int dev = 0;
  rc = current_device(&dev);
  if (rc != PAM_OK) return rc;
  if (grid_cap[dev] == 0) {
    int sms = 148, per_sm = 1;
    PAM_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    // maximum shared-memory carve-out, so the occupancy the grid is sized for
    // is the one the SM actually grants
    PAM_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    PAM_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, EVAL_WARPS * 32, 0));
    grid_cap[dev] = sms * std::max(per_sm, 1);
  }
  // with a queue: a persistent grid of one wave; without: one tile per warp
  const int64_t tiles_ctas = ceil_div(P, static_cast<int64_t>(EVAL_WARPS) * 32 * PT);
  const int64_t ctas = queue ? std::min<int64_t>(grid_cap[dev], tiles_ctas) : tiles_ctas;
  if (ctas > 0x7fffffffLL) return PAM_ERR_ARG;
  if (queue) PAM_CUDA_CHECK(cudaMemsetAsync(queue, 0, sizeof(unsigned long long), st));
  kernel<<<(unsigned)ctas, EVAL_WARPS * 32, 0, st>>>(P, pts, perm, sorted_owner, n_sorted, dict_off, m_cur,
                                                     centres, widths, beta, log_flag, single_m, single_exp,
                                                     out, err, queue);
  PAM_LAUNCH_CHECK("eval_kernel");
  return PAM_OK;
}

int grid_for(int64_t n, int threads) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), 148 * 32));
}

}  // namespace pam

using namespace pam;

extern "C" int64_t pam_eval_workspace_bytes(int64_t P, int64_t S) {
  // owner, perm, sorted_owner (P each) + counts, cursor (S) + start (S+1);
  // the slack holds the evaluation kernel's tile-queue counter
  return 3 * P * 8 + (3 * S + 1) * 8 + 256;
}

extern "C" int pam_locate_f64(int dim, int64_t P, const double* pts, const int32_t* shape,
                              const double* edges, int64_t* owner, int64_t* err, void* stream) {
  if (dim < 1 || dim > 3 || P < 0) return PAM_ERR_ARG;
  if (P == 0) return PAM_OK;
  cudaStream_t st = as_stream(stream);
  const int g = grid_for(P, 256);
  if (dim == 1) locate_kernel<1, int64_t><<<g, 256, 0, st>>>(P, pts, shape, edges, owner, err);
  else if (dim == 2) locate_kernel<2, int64_t><<<g, 256, 0, st>>>(P, pts, shape, edges, owner, err);
  else locate_kernel<3, int64_t><<<g, 256, 0, st>>>(P, pts, shape, edges, owner, err);
  PAM_LAUNCH_CHECK("locate_kernel");
  return PAM_OK;
}

namespace pam {
// locate -> counting sort by owner -> evaluation, with IdxT-wide indices
// (int32 whenever P and S fit: half the sort traffic and 32-bit atomics)
template <typename IdxT>
int locate_boxes(int dim, int64_t P, const double* pts, int64_t S, const double* lo, const double* hi,
                 const int32_t* open_hi, IdxT* owner, unsigned long long* flags, int64_t* err,
                 cudaStream_t st) {
  PAM_CUDA_CHECK(cudaMemsetAsync(flags, 0xff, 2 * sizeof(unsigned long long), st));
  const int g = grid_for(P, 256);
  if (dim == 1) locate_boxes_kernel<1, IdxT><<<g, 256, 0, st>>>(P, pts, S, lo, hi, open_hi, owner, flags);
  else if (dim == 2) locate_boxes_kernel<2, IdxT><<<g, 256, 0, st>>>(P, pts, S, lo, hi, open_hi, owner, flags);
  else locate_boxes_kernel<3, IdxT><<<g, 256, 0, st>>>(P, pts, S, lo, hi, open_hi, owner, flags);
  PAM_LAUNCH_CHECK("locate_boxes_kernel");
  locate_boxes_finish_kernel<<<1, 1, 0, st>>>(flags, err);
  PAM_LAUNCH_CHECK("locate_boxes_finish_kernel");
  return PAM_OK;
}

// shape/edges != null: tensor-grid boxes; else the S boxes (lo, hi, open_hi)
template <typename IdxT>
int eval_pipeline(int dim, int64_t P, const double* pts, const int32_t* shape, const double* edges,
                  const double* box_lo, const double* box_hi, const int32_t* box_open,
                  int64_t S, const int64_t* dict_off, const int32_t* m_cur, const double* centres,
                  const double* widths, const double* beta, const int32_t* log_flag, double* out,
                  void* work, int64_t* err, cudaStream_t st) {
  char* w = static_cast<char*>(work);
  IdxT* owner = reinterpret_cast<IdxT*>(w);
  IdxT* perm = owner + P;
  IdxT* sorted_owner = perm + P;
  IdxT* counts = sorted_owner + P;
  IdxT* cursor = counts + S;
  IdxT* start = cursor + S;
  // the tile-queue counter, 8-byte aligned after start[S]
  unsigned long long* queue = reinterpret_cast<unsigned long long*>(
      (reinterpret_cast<uintptr_t>(start + S + 1) + 7) & ~static_cast<uintptr_t>(7));
  const int g = grid_for(P, 256);
  if (shape != nullptr) {
    if (dim == 1) locate_kernel<1, IdxT><<<g, 256, 0, st>>>(P, pts, shape, edges, owner, err);
    else if (dim == 2) locate_kernel<2, IdxT><<<g, 256, 0, st>>>(P, pts, shape, edges, owner, err);
    else locate_kernel<3, IdxT><<<g, 256, 0, st>>>(P, pts, shape, edges, owner, err);
    PAM_LAUNCH_CHECK("locate_kernel");
  } else {
    const int rc = locate_boxes<IdxT>(dim, P, pts, S, box_lo, box_hi, box_open, owner, queue + 1, err, st);
    if (rc != PAM_OK) return rc;
  }
  PAM_CUDA_CHECK(cudaMemsetAsync(counts, 0, S * sizeof(IdxT), st));
  histogram_kernel<IdxT><<<g, 256, 0, st>>>(P, owner, counts);
  PAM_LAUNCH_CHECK("histogram_kernel");
  scan_kernel<IdxT><<<1, SCAN_THREADS, 0, st>>>(S, counts, start, cursor);
  PAM_LAUNCH_CHECK("scan_kernel");
  // points that failed to locate are not scattered: the evaluation covers
  // the start[S] located ones (error path: the caller raises)
  scatter_kernel<IdxT><<<g, 256, 0, st>>>(P, owner, cursor, perm, sorted_owner);
  PAM_LAUNCH_CHECK("scatter_kernel");
  const IdxT* n_sorted = start + S;
  if (dim == 1)
    return launch_eval<1, IdxT>(st, P, pts, perm, sorted_owner, n_sorted, dict_off, m_cur, centres, widths,
                                beta, log_flag, 0, 0, out, err, queue);
  if (dim == 2)
    return launch_eval<2, IdxT>(st, P, pts, perm, sorted_owner, n_sorted, dict_off, m_cur, centres, widths,
                                beta, log_flag, 0, 0, out, err, queue);
  return launch_eval<3, IdxT>(st, P, pts, perm, sorted_owner, n_sorted, dict_off, m_cur, centres, widths,
                              beta, log_flag, 0, 0, out, err, queue);
}
}  // namespace pam

extern "C" int pam_eval_f64(int dim, int64_t P, const double* pts, const int32_t* shape,
                            const double* edges, int64_t S, const int64_t* dict_off,
                            const int32_t* m_cur, const double* centres, const double* widths,
                            const double* beta, const int32_t* log_flag, double* out, void* work,
                            int64_t* err, void* stream) {
  if (dim < 1 || dim > 3 || P < 0 || S < 1 || !work) return PAM_ERR_ARG;
  if (P == 0) return PAM_OK;
  cudaStream_t st = as_stream(stream);
  if (P < 0x7fffffffLL && S < 0x7fffffffLL)
    return eval_pipeline<int32_t>(dim, P, pts, shape, edges, nullptr, nullptr, nullptr, S, dict_off, m_cur,
                                  centres, widths, beta, log_flag, out, work, err, st);
  return eval_pipeline<int64_t>(dim, P, pts, shape, edges, nullptr, nullptr, nullptr, S, dict_off, m_cur,
                                centres, widths, beta, log_flag, out, work, err, st);
}

extern "C" int pam_locate_boxes_f64(int dim, int64_t P, const double* pts, int64_t S, const double* box_lo,
                                    const double* box_hi, const int32_t* box_open, int64_t* owner,
                                    void* work, int64_t* err, void* stream) {
  if (dim < 1 || dim > 3 || P < 0 || S < 1 || S >= (1LL << 23) || P >= (1LL << 40) || !work) return PAM_ERR_ARG;
  if (P == 0) return PAM_OK;
  return locate_boxes<int64_t>(dim, P, pts, S, box_lo, box_hi, box_open, owner,
                               static_cast<unsigned long long*>(work), err, as_stream(stream));
}

extern "C" int pam_eval_boxes_f64(int dim, int64_t P, const double* pts, const double* box_lo,
                                  const double* box_hi, const int32_t* box_open, int64_t S,
                                  const int64_t* dict_off, const int32_t* m_cur, const double* centres,
                                  const double* widths, const double* beta, const int32_t* log_flag,
                                  double* out, void* work, int64_t* err, void* stream) {
  if (dim < 1 || dim > 3 || P < 0 || S < 1 || S >= (1LL << 23) || P >= (1LL << 40) || !work) return PAM_ERR_ARG;
  if (!box_lo || !box_hi || !box_open) return PAM_ERR_ARG;
  if (P == 0) return PAM_OK;
  cudaStream_t st = as_stream(stream);
  if (P < 0x7fffffffLL)
    return eval_pipeline<int32_t>(dim, P, pts, nullptr, nullptr, box_lo, box_hi, box_open, S, dict_off, m_cur,
                                  centres, widths, beta, log_flag, out, work, err, st);
  return eval_pipeline<int64_t>(dim, P, pts, nullptr, nullptr, box_lo, box_hi, box_open, S, dict_off, m_cur,
                                centres, widths, beta, log_flag, out, work, err, st);
}

extern "C" int pam_shepard_eval_f64(int dim, int64_t P, const double* pts, int64_t M,
                                    const double* centres, const double* widths,
                                    const double* beta, int32_t exp_out, double* out, int64_t* err,
                                    void* stream) {
  if (dim < 1 || dim > 3 || P < 0 || M < 1 || M > 0x7fffffff) return PAM_ERR_ARG;
  if (P == 0) return PAM_OK;
  cudaStream_t st = as_stream(stream);
  const int m = static_cast<int>(M);
  if (dim == 1)
    return launch_eval<1, int64_t>(st, P, pts, nullptr, nullptr, nullptr, nullptr, nullptr, centres, widths, beta,
                          nullptr, m, exp_out, out, err, nullptr);
  if (dim == 2)
    return launch_eval<2, int64_t>(st, P, pts, nullptr, nullptr, nullptr, nullptr, nullptr, centres, widths, beta,
                          nullptr, m, exp_out, out, err, nullptr);
  return launch_eval<3, int64_t>(st, P, pts, nullptr, nullptr, nullptr, nullptr, nullptr, centres, widths, beta,
                        nullptr, m, exp_out, out, err, nullptr);
}
