// gram.cu — K2: batched FP64 Gram products and the Gram-form CD (K2b') for
// subdomains whose dictionary is smaller than their sample count (M < N).
//
// The reference CD (elastic_net.py:113-161) works in residual form: per
// coordinate a length-N dot W_j.r and an AXPY r -= d W_j, i.e. N*M doubles
// streamed per sweep.  With c = W^T y - G beta (G = W^T W) the same
// cyclic updates read only column j of G:  z = col_sq_j beta_j + c_j,
// c -= d G[:, j]  — M*M doubles per sweep instead of N*M (C1: 4x fewer,
// C5 at M=64: 16x fewer, and the whole G of a small-M subdomain stays
// L2-resident across sweeps).  The decisions (cyclic order, soft threshold,
// division, stop rule) are the reference's; only the rounding of the
// accumulated inner products differs (~1e-12 relative in beta).
// FP64 throughout: an FP32/TF32 Gram fails the tolerance by 1e4-1e6 (F3).
//
//   gram_kernel     G = W^T W (symmetric: upper tiles computed, mirrored),
//                   32x32 output tiles, W chunks staged in shared memory.
//   gemv_t_kernel   q = W^T y, one warp per column.
//   cd_gram_kernel  one warp per subdomain, c in registers (lane l owns
//                   coordinates l + 32t), G columns streamed by cp.async.bulk
//                   (several columns per ring slot when M is small).
#include "pam_common.cuh"

#include <algorithm>

namespace pam {


// ---- G = W^T W -------------------------------------------------------------
// Register-blocked FP64 tiles: a CTA of 256 threads computes one 64 x 64 block
// (jb <= kb: the upper block triangle, mirrored on store) of G_s = W_s^T W_s,
// each thread a 4 x 4 micro-tile (rows ty + 16u, columns tx + 16v: the two
// operand fetches of a k-step are 4 + 4 conflict-free shared loads feeding 16
// DFMA, vs 5 loads per 4 DFMA in a 32 x 32 one-output-per-thread tile).  W is
// column-major with its rows (sample points) contiguous, so a K-chunk of 16
// rows x 64 columns is staged with coalesced loads.  Each G entry is one
// fixed-order FP64 sum over the rows (deterministic; SURVEY F3 rules out lower
// precision).  gram_kernel ncu (r02, C5 M=512): FP64 pipe 27 % for the 32 x 32
// version.
constexpr int GB = 64;  // output block
constexpr int GK = 16;  // rows per K-chunk
__global__ void __launch_bounds__(256)
gram_kernel(const int64_t* __restrict__ row_off, const int32_t* __restrict__ m_cur,
            const int64_t* __restrict__ w_off, const int32_t* __restrict__ ld,
            const int64_t* __restrict__ g_off, const int32_t* __restrict__ ldg,
            const int32_t* __restrict__ active, const double* __restrict__ W,
            double* __restrict__ G) {
  __shared__ double A[GK][GB + 2];
  __shared__ double B[GK][GB + 2];
  const int64_t s = blockIdx.y;
  if (active != nullptr && active[s] == 0) return;
  const int M = m_cur[s];
  const int T = (M + GB - 1) / GB;
  // decode upper-triangular block pair (jb <= kb) from blockIdx.x
  int pair = blockIdx.x, jb = 0;
  while (jb < T && pair >= T - jb) {
    pair -= T - jb;
    ++jb;
  }
  if (jb >= T) return;
  const int kb = jb + pair;
  const int n = static_cast<int>(row_off[s + 1] - row_off[s]);
  const double* Ws = W + w_off[s];
  const int64_t lds = ld[s];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;  // 16 x 16 threads, 4 x 4 outputs each
  double acc[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
  // staging: thread -> (row i = tid % 16, column c = tid / 16 + 16 q), q < 4
  const int si = tid & 15, sc = tid >> 4;
  for (int i0 = 0; i0 < n; i0 += GK) {
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = sc + 16 * q;
      const int i = i0 + si;
      const int cj = jb * GB + c, ck = kb * GB + c;
      A[si][c] = (i < n && cj < M) ? Ws[(int64_t)cj * lds + i] : 0.0;
      B[si][c] = (i < n && ck < M) ? Ws[(int64_t)ck * lds + i] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < GK; ++i) {
      double av[4], bv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) av[u] = A[i][ty + 16 * u];
#pragma unroll
      for (int v = 0; v < 4; ++v) bv[v] = B[i][tx + 16 * v];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(av[u], bv[v], acc[u][v]);
    }
  }
  double* Gs = G + g_off[s];
  const int64_t ldgs = ldg[s];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int j = jb * GB + ty + 16 * u;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int k = kb * GB + tx + 16 * v;
      if (j < M && k < M) {
        Gs[(int64_t)k * ldgs + j] = acc[u][v];
        if (jb != kb) Gs[(int64_t)j * ldgs + k] = acc[u][v];
      }
    }
  }
}

// ---- q = W^T y, col_sq = diag(G) -------------------------------------------
__global__ void gemv_t_kernel(const int64_t* __restrict__ row_off, const int32_t* __restrict__ m_cur,
                              const int64_t* __restrict__ dict_off, const int64_t* __restrict__ w_off,
                              const int32_t* __restrict__ ld, const int64_t* __restrict__ g_off,
                              const int32_t* __restrict__ ldg, const int32_t* __restrict__ active,
                              const double* __restrict__ W, const double* __restrict__ y,
                              const double* __restrict__ G, double* __restrict__ q,
                              double* __restrict__ col_sq) {
  const int64_t s = blockIdx.y;
  if (active != nullptr && active[s] == 0) return;
  const int M = m_cur[s];
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= M) return;
  const int64_t r0 = row_off[s];
  const int n = static_cast<int>(row_off[s + 1] - r0);
  const double* col = W + w_off[s] + (int64_t)warp * ld[s];
  double acc = 0.0;
  for (int i = lane; i < n; i += 32) acc = fma(col[i], y[r0 + i], acc);
  acc = warp_sum(acc);
  if (lane == 0) {
    q[dict_off[s] + warp] = acc;
    col_sq[dict_off[s] + warp] = G[g_off[s] + (int64_t)warp * ldg[s] + warp];
  }
}

// ---- Gram-form cyclic CD ------------------------------------------------------
struct GramArgs {
  int64_t S;
  const int64_t* order;
  const int64_t* dict_off;
  const int32_t* m_cur;
  const int64_t* g_off;
  const int32_t* ldg;
  const double* G;
  const double* q;
  const double* col_sq;
  const double* lam1;
  const double* lam2;
  const double* tol;
  const int32_t* max_iters;
  const int32_t* active;
  double* beta;
  int32_t* sweeps;
  int32_t* converged;
  unsigned* queue;  // work counter in the caller's workspace
};

// Lean covariance-form CD.  MT: coordinates per lane (M <= 32*MT, MT even);
// SLOT: doubles per ring slot (cps = SLOT / ldg columns per slot).
//
// Paired layout: lane l owns coordinates 64u + 2l + {0,1} in c[2u], c[2u+1],
// so each AXPY element pair is one 16-byte shared load.  The coordinate loop
// is NOT unrolled over chunks (an unrolled loop over MT chunks overflowed the
// instruction cache at M = 512, 0.57 of HBM): the current 64-coordinate
// chunk's two values live in (cur0, cur1), selected once per chunk and
// updated alongside c, so c_j is one shuffle away.  Per-chunk parameters
// (beta, col_sq, 1/(col_sq+lam2)) are prefetched one chunk ahead into a
// per-warp shared block; the division is the reciprocal plus one FMA
// correction, as in cd.cu's lean kernel.
template <int MT, int STAGES, int WPC, int SLOT>
__global__ void __launch_bounds__(WPC * 32, 1) cd_gram_kernel(const GramArgs a) {
  static_assert(MT % 2 == 0, "paired layout");
  constexpr int MP = MT / 2;  // 16-byte pairs per lane
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  double* const ring = reinterpret_cast<double*>(smem_raw) + static_cast<size_t>(warp) * STAGES * SLOT;
  uint64_t* const bars =
      reinterpret_cast<uint64_t*>(reinterpret_cast<double*>(smem_raw) + WPC * STAGES * SLOT) + warp * STAGES;
  double* const pblk = reinterpret_cast<double*>(
                           reinterpret_cast<uint64_t*>(reinterpret_cast<double*>(smem_raw) + WPC * STAGES * SLOT) +
                           WPC * STAGES) +
                       warp * 192;
  double* const pb = pblk;          // [64] beta of the chunk
  double* const pc = pblk + 64;     // [64] col_sq
  double* const pinv = pblk + 128;  // [64] 1 / (col_sq + lam2)
  if (lane == 0) {
    for (int i = 0; i < STAGES; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncwarp();
  const uint32_t ring_s = smem_u32(ring);
  const uint32_t bar_s = smem_u32(bars);
  int ist = 0, cst = 0;  // issue / consume ring slots
  uint32_t ph = 0;       // consume phase parity
  const unsigned total_warps = gridDim.x * WPC;
  unsigned item = warp * gridDim.x + blockIdx.x;

  while (item < a.S) {
    const int64_t s = a.order ? a.order[item] : static_cast<int64_t>(item);
    if (a.active == nullptr || a.active[s] != 0) {
      const int M = a.m_cur[s];
      const int64_t doff = a.dict_off[s];
      const double* Gs = a.G + a.g_off[s];
      const int ldgs = a.ldg[s];
      const int cps = max(1, SLOT / ldgs);     // columns per ring slot
      const int groups = (M + cps - 1) / cps;  // slots per pass over G
      const double lam1 = a.lam1[s], lam2 = a.lam2[s], tol = a.tol[s];
      const int max_iters = a.max_iters[s];
      double* betas = a.beta + doff;

      double c[MT];
#pragma unroll
      for (int u = 0; u < MP; ++u) {
        const int k = 64 * u + 2 * lane;
        c[2 * u] = (k < M) ? a.q[doff + k] : 0.0;
        c[2 * u + 1] = (k + 1 < M) ? a.q[doff + k + 1] : 0.0;
      }
      // issue side: group stream = [prologue] + max_iters passes (32-bit: host envelope)
      const int total = (max_iters + 1) * groups;
      int issued = 0, next_group = 0;
      auto issue_one = [&](double dep) {
        if (lane == 0) {
          const int c0 = next_group * cps;
          const int nc = min(cps, M - c0);
          // one column per slot: copy only the current M entries (even, for the
          // 16-byte size rule) -- the leading dimension may exceed the slot
          // for wide dictionaries that grow across rounds
          const uint32_t nb = (cps == 1 ? static_cast<uint32_t>((M + 1) & ~1)
                                        : static_cast<uint32_t>(nc) * ldgs) * sizeof(double);
          const uint32_t bar = bar_s + ist * 8;
          mbar_expect_s(bar, nb);
          bulk_g2s_dep(ring_s + ist * (SLOT * 8), Gs + (int64_t)c0 * ldgs, nb, bar, dep);
        }
        if (++ist == STAGES) ist = 0;
        ++issued;
        if (++next_group == groups) next_group = 0;
      };
      for (int q0 = 0; q0 < STAGES && issued < total; ++q0) issue_one(0.0);
      int consumed = 0;
      int in_slot = cps;  // columns left in the current slot (cps -> acquire next)
      uint32_t col_s = 0;
      // shared address of column j (columns arrive in order; slot acquired on demand)
      auto column = [&]() -> uint32_t {
        if (in_slot == cps) {
          mbar_wait_s(bar_s + cst * 8, ph);
          col_s = ring_s + cst * (SLOT * 8);
          in_slot = 0;
        } else {
          col_s += ldgs * 8;
        }
        ++in_slot;
        return col_s;
      };
      // after the last use of a column: free its slot when it was the slot's last
      auto release = [&](bool last_col_of_pass, double dep) {
        if (in_slot == cps || last_col_of_pass) {
          in_slot = cps;
          if (++cst == STAGES) {
            cst = 0;
            ph ^= 1u;
          }
          ++consumed;
          if (issued < total) issue_one(dep);
        }
      };
      auto axpy = [&](uint32_t col, double d) {
        double dep = 0.0;
#pragma unroll
        for (int u = 0; u < MP; ++u) {
          double g0, g1;
          lds_v2(col + 16u * lane + 512u * u, g0, g1);
          c[2 * u] = fma(-d, g0, c[2 * u]);
          c[2 * u + 1] = fma(-d, g1, c[2 * u + 1]);
          dep += g0;
        }
        return dep;
      };

      // prologue: c = q - G beta0 (warm start, adaptive.py:268)
      for (int j = 0; j < M; ++j) {
        const uint32_t col = column();
        const double b0 = betas[j];
        double dep = 0.0;
        if (b0 != 0.0) dep = axpy(col, b0);
        else {
          double g0, g1;
          lds_v2(col + 16u * lane, g0, g1);  // the slot is read before it is refilled
          dep = g0;
        }
        release(j == M - 1, dep);
      }

      const int nchunk = (M + 63) / 64;
      double nb0 = 0.0, nb1 = 0.0, nc0 = 0.0, nc1 = 0.0;
      auto fetch = [&](int q) {
        const int k0 = 64 * q + lane, k1 = k0 + 32;
        nb0 = (k0 < M) ? betas[k0] : 0.0;
        nb1 = (k1 < M) ? betas[k1] : 0.0;
        nc0 = (k0 < M) ? a.col_sq[doff + k0] : 0.0;
        nc1 = (k1 < M) ? a.col_sq[doff + k1] : 0.0;
      };
      fetch(0);
      int sweeps_done = 0, conv = 0;
      for (int sw = 0; sw < max_iters; ++sw) {
        double max_delta = 0.0, acc_max = 0.0;
        for (int q = 0; q < nchunk; ++q) {
          const int nc = min(64, M - 64 * q);
          __syncwarp();
          // one chunk: the block keeps the updated betas across sweeps (a
          // prefetch would read them before this sweep's write-back)
          if (sw == 0 || nchunk > 1) {
            pb[lane] = nb0;
            pb[32 + lane] = nb1;
            pc[lane] = nc0;
            pc[32 + lane] = nc1;
            const double d0 = __dadd_rn(nc0, lam2), d1 = __dadd_rn(nc1, lam2);
            pinv[lane] = d0 > 0.0 ? __ddiv_rn(1.0, d0) : 0.0;
            pinv[32 + lane] = d1 > 0.0 ? __ddiv_rn(1.0, d1) : 0.0;
            if (nchunk > 1) fetch(q + 1 < nchunk ? q + 1 : 0);
          }
          __syncwarp();
          // this chunk's pair of c values (runtime q -> static selects, once per chunk)
          double cur0 = 0.0, cur1 = 0.0;
#pragma unroll
          for (int u = 0; u < MP; ++u) {
            if (u == q) {
              cur0 = c[2 * u];
              cur1 = c[2 * u + 1];
            }
          }
          for (int r = 0; r < nc; ++r) {
            const int j = 64 * q + r;
            const uint32_t col = column();
            const double cj = __shfl_sync(0xffffffffu, (r & 1) ? cur1 : cur0, r >> 1);
            const double b_old = pb[r];
            const double cs = pc[r];
            const double inv = pinv[r];
            const double dn = __dadd_rn(cs, lam2);
            const double z = __dadd_rn(__dmul_rn(cs, b_old), cj);
            const double np_ = __dsub_rn(z, lam1), nn_ = __dadd_rn(z, lam1);
            const double qp = __dmul_rn(np_, inv), qn = __dmul_rn(nn_, inv);
            const double bp = fma(fma(-qp, dn, np_), inv, qp);
            const double bn = fma(fma(-qn, dn, nn_), inv, qn);
            const double b_new = np_ > 0.0 ? bp : (nn_ < 0.0 ? bn : 0.0);
            const double d = __dsub_rn(b_new, b_old);
            double dep;
            {
              double g0, g1;
              lds_v2(col + 16u * lane + 512u * q, g0, g1);
              cur0 = fma(-d, g0, cur0);
              cur1 = fma(-d, g1, cur1);
              dep = axpy(col, d) + g0;
            }
            if (lane == 0) pb[r] = b_new;
            const double ad = fabs(d);
            max_delta = ad > max_delta ? ad : max_delta;
            release(j == M - 1, dep);
          }
          __syncwarp();
          const int k0 = 64 * q + lane, k1 = k0 + 32;
          if (k0 < M) {
            betas[k0] = pb[lane];
            acc_max = fmax(acc_max, fabs(pb[lane]));
          }
          if (k1 < M) {
            betas[k1] = pb[32 + lane];
            acc_max = fmax(acc_max, fabs(pb[32 + lane]));
          }
        }
        const double mabs = warp_max(acc_max);
        sweeps_done = sw + 1;
        if (max_delta <= __dmul_rn(tol, fmax(mabs, 1.0))) {
          conv = 1;
          break;
        }
      }
      while (consumed < issued) {  // drain the prefetched groups of the pass that will not run
        mbar_wait_s(bar_s + cst * 8, ph);
        if (++cst == STAGES) {
          cst = 0;
          ph ^= 1u;
        }
        ++consumed;
      }
      __syncwarp();
      if (lane == 0) {
        a.sweeps[s] = sweeps_done;
        a.converged[s] = conv;
      }
    }
    unsigned nxt = 0;
    if (lane == 0) nxt = atomicAdd(a.queue, 1u) + total_warps;
    item = __shfl_sync(0xffffffffu, nxt, 0);
  }
}

template <int MT, int STAGES, int WPC, int SLOT>
int launch_gram_cd(const GramArgs& a, cudaStream_t stream) {
  const size_t smem = static_cast<size_t>(WPC) * STAGES * (SLOT * sizeof(double) + sizeof(uint64_t)) +
                      static_cast<size_t>(WPC) * 192 * sizeof(double);
  // per device and per function; set on every launch (cheap)
  PAM_CUDA_CHECK(cudaFuncSetAttribute(cd_gram_kernel<MT, STAGES, WPC, SLOT>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev = 0, sms = 148;
  PAM_CUDA_CHECK(cudaGetDevice(&dev));
  PAM_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  PAM_CUDA_CHECK(cudaMemsetAsync(a.queue, 0, sizeof(unsigned), stream));
  const int64_t ctas = std::max<int64_t>(1, std::min<int64_t>(sms, ceil_div(a.S, 1)));
  cd_gram_kernel<MT, STAGES, WPC, SLOT><<<(unsigned)ctas, WPC * 32, smem, stream>>>(a);
  PAM_LAUNCH_CHECK("cd_gram_kernel");
  return PAM_OK;
}

}  // namespace pam

using namespace pam;

extern "C" int pam_gram_f64(int64_t S, const int64_t* row_off, const int32_t* m_cur,
                            const int64_t* dict_off, const int64_t* w_off, const int32_t* ld,
                            const int64_t* g_off, const int32_t* ldg, const int32_t* active,
                            int32_t max_m, const double* W, const double* y, double* G, double* q,
                            double* col_sq, void* stream) {
  if (S < 0 || max_m < 0) return PAM_ERR_ARG;
  if (S == 0 || max_m == 0) return PAM_OK;
  cudaStream_t st = as_stream(stream);
  const int T = (max_m + GB - 1) / GB;
  for (int64_t s0 = 0; s0 < S; s0 += 65535) {
    const int64_t cnt = std::min<int64_t>(65535, S - s0);
    const int32_t* act = active ? active + s0 : nullptr;
    gram_kernel<<<dim3(T * (T + 1) / 2, (unsigned)cnt), 256, 0, st>>>(
        row_off + s0, m_cur + s0, w_off + s0, ld + s0, g_off + s0, ldg + s0, act, W, G);
    PAM_LAUNCH_CHECK("gram_kernel");
    gemv_t_kernel<<<dim3((unsigned)ceil_div((int64_t)max_m * 32, 256), (unsigned)cnt), 256, 0, st>>>(
        row_off + s0, m_cur + s0, dict_off + s0, w_off + s0, ld + s0, g_off + s0, ldg + s0, act, W,
        y, G, q, col_sq);
    PAM_LAUNCH_CHECK("gemv_t_kernel");
  }
  return PAM_OK;
}

extern "C" int pam_cd_gram_f64(int64_t S, const int64_t* order, const int64_t* dict_off,
                               const int32_t* m_cur, const int64_t* g_off, const int32_t* ldg,
                               const double* G, const double* q, const double* col_sq,
                               const double* lam1, const double* lam2, const double* tol,
                               const int32_t* max_iters, const int32_t* active, int32_t max_m,
                               double* beta, int32_t* sweeps, int32_t* converged, void* work,
                               void* stream) {
  if (S < 0 || max_m < 0 || work == nullptr) return PAM_ERR_ARG;
  if (S == 0) return PAM_OK;
  GramArgs a{S, order, dict_off, m_cur, g_off, ldg, G, q, col_sq, lam1, lam2, tol, max_iters,
             active, beta, sweeps, converged, static_cast<unsigned*>(work)};
  cudaStream_t st = as_stream(stream);
  // ldg <= SLOT is required: ldg = M_cap rounded to 16
  if (max_m <= 64) return launch_gram_cd<2, 3, 16, 512>(a, st);  // 8 columns per 4 KB copy (3 % faster than 24 warps x 2 KB)
  if (max_m <= 128) return launch_gram_cd<4, 3, 16, 512>(a, st);
  if (max_m <= 256) return launch_gram_cd<8, 3, 16, 512>(a, st);
  if (max_m <= 512) return launch_gram_cd<16, 3, 16, 512>(a, st);
  // wide dictionaries, chosen by the host only for batches of few fits (one
  // per SM), where the residual form is bound by one fit's per-column chain:
  // c in up to 192 registers, one warp per CTA (= per SM) with an 8-deep ring
  // of G columns (up to 196 KB in flight: one SM must pull ~100 GB/s)
  if (max_m <= 1024) return launch_gram_cd<32, 8, 1, 1024>(a, st);
  if (max_m <= 2048) return launch_gram_cd<64, 8, 1, 2048>(a, st);
  if (max_m <= 2304) return launch_gram_cd<72, 8, 1, 2304>(a, st);
  if (max_m <= 3072) return launch_gram_cd<96, 8, 1, 3072>(a, st);
  set_last_error("pam_cd_gram_f64: Gram-form CD supports M <= 3072 (use the residual form)");
  return PAM_ERR_UNSUPPORTED;
}
