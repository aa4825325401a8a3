// cd.cu — K2b: batched cyclic coordinate descent for the Elastic Net.
//
// Replaces fit() + _cd_sweeps_jit (reference elastic_net.py:66-161) for a
// whole ragged batch of subdomain fits.  Semantics kept exactly: residual
// form, fixed cyclic order j = 0..M-1, z = col_sq_j*beta_j + W_j.r,
// b_new = sign(z) max(|z|-lam1, 0) / (col_sq_j + lam2) (true division),
// r -= (b_new - b_old) W_j only when b_new != b_old, per-sweep objective
// 0.5 r.r + lam1 |b|_1 + 0.5 lam2 |b|^2, stop when
// max|delta| <= tol * max(1, max|beta|) or after max_iters sweeps
// (non-convergence is flagged, not an error).  Only the order of the length-N
// dot products differs from the reference's sequential sums (SURVEY F2:
// ~1e-12 relative in beta).
//
// B200 mapping.  One warp owns one subdomain fit for its whole life: the
// residual r lives in registers (lane l holds rows l, l+32, ...), the
// design matrix is streamed column by column (column-major, so a column is
// one contiguous N*8-byte run) from HBM into a per-warp shared-memory ring
// by the TMA bulk-copy engine (cp.async.bulk + mbarrier complete_tx), STAGES
// columns ahead of the consumer.  The prologue pass (col_sq and the warm-start
// residual) and all sweeps are one continuous column stream, so there is no
// pipeline bubble between sweeps.  Warps pull subdomains from a dynamic queue
// (longest first, host-ordered) so the ragged batch stays balanced.  Each
// sweep reads N*M*8 bytes: the kernel is HBM-bandwidth bound (SURVEY §8d,
// K2b), ~2 FMA per 8 bytes.
#include "pam_common.cuh"

#include <stdlib.h>

#include <algorithm>

namespace pam {

__device__ unsigned int g_cd_queue;

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
};

// named barrier over the G warps of one subdomain group (G > 1 only)
__device__ __forceinline__ void group_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// R: rows per thread, STAGES: ring depth, WPC: warps per CTA, G: warps per
// subdomain group (rows of a subdomain split over the G*32 threads).
template <int R, int STAGES, int WPC, int G, bool TILES, bool KEEPW = true, bool LDGSTS = false>
__global__ void __launch_bounds__(WPC * 32, 1) cd_kernel(const CdArgs a) {
  static_assert(!LDGSTS || (G == 1 && STAGES == 3), "LDGSTS staging: one warp, 3 stages");
  static_assert(!TILES || G == 1, "tile-packed columns are consumed one warp per subdomain");
  constexpr int GT = G * 32;         // threads per group
  constexpr int LDMAX = R * GT;      // rows per ring slot
  constexpr int NGROUPS = WPC / G;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int grp = warp / G;          // group within the CTA
  const int wig = warp % G;          // warp within group
  const int gt = threadIdx.x - grp * GT;  // thread within group
  double* ring = reinterpret_cast<double*>(smem_raw) + static_cast<size_t>(grp) * STAGES * LDMAX;
  uint64_t* bars =
      reinterpret_cast<uint64_t*>(reinterpret_cast<double*>(smem_raw) + NGROUPS * STAGES * LDMAX) +
      grp * STAGES;
  double* red = reinterpret_cast<double*>(
                    reinterpret_cast<uint64_t*>(reinterpret_cast<double*>(smem_raw) +
                                                NGROUPS * STAGES * LDMAX) +
                    NGROUPS * STAGES) +
                grp * (2 * G + 1);  // double-buffered cross-warp partials + queue slot
  const int bar_id = 1 + grp;
  // per-warp column-parameter block (G == 1): beta, col_sq, tile mask of the
  // current 32-column chunk, read by warp-uniform smem broadcasts
  constexpr bool PSM = (G == 1);
  double* prm_base = reinterpret_cast<double*>(smem_raw) +
                     (static_cast<size_t>(NGROUPS) * STAGES * LDMAX) + NGROUPS * STAGES +
                     NGROUPS * (2 * G + 1);
  double* pb = prm_base + grp * 128;
  double* pc = pb + 32;
  double* pinv = pb + 64;  // 1 / (col_sq + lam2): division by reciprocal + one FMA correction
  unsigned* pm = reinterpret_cast<unsigned*>(pb + 96);

  auto sync_group = [&]() {
    if (G == 1) __syncwarp();
    else group_bar(bar_id, GT);
  };
  int red_buf = 0;
  auto group_sum = [&](double v) -> double {
    v = warp_sum(v);
    if (G == 1) return v;
    if (lane == 0) red[red_buf * G + wig] = v;
    group_bar(bar_id, GT);
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < G; ++w) t += red[red_buf * G + w];
    red_buf ^= 1;
    return t;
  };

  if (gt == 0) {
    for (int st = 0; st < STAGES; ++st) mbar_init(&bars[st], 1);
    fence_mbar_init();
    fence_proxy_async_smem();
  }
  sync_group();

  uint32_t g_issue = 0, g_cons = 0;  // running ring counters (stage = g % STAGES)
  const unsigned total_groups = gridDim.x * NGROUPS;
  unsigned item = grp * gridDim.x + blockIdx.x;  // spread the first items over SMs

  while (item < a.S) {
    const int64_t s = a.order ? a.order[item] : static_cast<int64_t>(item);
    if (a.active == nullptr || a.active[s] != 0) {
      const int64_t r0 = a.row_off[s];
      const int N = static_cast<int>(a.row_off[s + 1] - r0);
      const int M = a.m_cur[s];
      const int64_t doff = a.dict_off[s];
      const double* Ws = a.W + a.w_off[s];
      const int64_t ld = a.ld[s];
      const double lam1 = a.lam1[s], lam2 = a.lam2[s], tol = a.tol[s];
      const int max_iters = a.max_iters[s];
      const uint32_t dense_bytes = static_cast<uint32_t>(((N + 1) & ~1) * sizeof(double));
      const bool need_colsq = !(a.flags & CD_COLSQ_GIVEN);
      const bool r_given = (a.flags & CD_R_GIVEN) != 0;
      const bool prologue = need_colsq || !r_given;

      // residual / targets into registers (thread gt owns rows gt + GT*k);
      // in tile mode position p = lane + 32k holds local row perm[p]
      double r[R];
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const int p = gt + GT * k;
        const int row = (TILES && a.perm) ? (p < N ? a.perm[r0 + p] : 0) : p;
        r[k] = (p < N) ? a.y[r0 + row] : 0.0;
      }

      // per-column packing parameters for the ISSUE pointer (tile mode)
      int iss_base = -64;
      int64_t iss_off_l = 0;
      unsigned long long iss_mask_l = 0;

      // continuous column stream: [prologue M columns] + max_iters * M columns
      const int64_t total = (prologue ? (int64_t)M : 0) + (int64_t)max_iters * M;
      int64_t issued = 0;
      int next_col = 0;
      auto issue_one = [&]() {
        if (TILES) {
          const int cbase = next_col & ~31;
          if (cbase != iss_base) {  // warp-uniform reload of 32 columns' packing
            iss_base = cbase;
            const int c = cbase + lane;
            iss_off_l = (c < M) ? a.col_off[doff + c] : 0;
            iss_mask_l = (c < M) ? a.tile_mask[doff + c] : 0ull;
          }
          const int off = __shfl_sync(0xffffffffu, static_cast<int>(iss_off_l), next_col & 31);
          unsigned long long mk;
          if (R <= 32) mk = __shfl_sync(0xffffffffu, static_cast<unsigned>(iss_mask_l), next_col & 31);
          else mk = __shfl_sync(0xffffffffu, iss_mask_l, next_col & 31);
          const uint32_t nb = static_cast<uint32_t>(__popcll(mk)) * 32u * sizeof(double);
          if (LDGSTS) {
            // per-lane 16-byte async copies of the packed column (no TMA unit)
            double* dst = ring + (g_issue % STAGES) * LDMAX;
            const double* src = Ws + off;
            const int pieces = static_cast<int>(nb / 16u);
            for (int i = lane; i < pieces; i += 32) cp_async16(dst + 2 * i, src + 2 * i);
            cp_async_commit();
          } else if (lane == 0) {
            const int st = g_issue % STAGES;
            if (nb) {
              mbar_arrive_expect_tx(&bars[st], nb);
              tma_load_1d(ring + st * LDMAX, Ws + off, nb, &bars[st]);
            } else {
              mbar_arrive(&bars[st]);  // empty column: complete the phase without data
            }
          }
        } else if (gt == 0) {
          const int st = g_issue % STAGES;
          mbar_arrive_expect_tx(&bars[st], dense_bytes);
          tma_load_1d(ring + st * LDMAX, Ws + (int64_t)next_col * ld, dense_bytes, &bars[st]);
        }
        ++g_issue;
        ++issued;
        if (++next_col == M) next_col = 0;
      };
      auto wait_one = [&]() -> const double* {
        const int st = g_cons % STAGES;
        if (LDGSTS) {
          const int ahead = static_cast<int>(g_issue - g_cons) - 1;  // groups that may stay in flight
          if (ahead >= 2) cp_async_wait<2>();
          else if (ahead == 1) cp_async_wait<1>();
          else cp_async_wait<0>();
          __syncwarp();
        } else {
          mbar_wait(&bars[st], (g_cons / STAGES) & 1u);
        }
        ++g_cons;
        return ring + st * LDMAX;
      };
      // Column staging: the column's entries for this thread's rows go to
      // registers once and serve both the dot and the AXPY.  Branch-free: rows
      // past N (dense) or tiles not stored (tile mode) read an in-bounds smem
      // word and select 0, so they contribute exactly nothing.
      double w[KEEPW ? R : 1];
      const double* cur_col = nullptr;
      unsigned long long cur_mk = 0ull;
      auto load_col = [&](const double* col, unsigned long long mk) {
        cur_col = col;
        cur_mk = mk;
        if (!KEEPW) return;
        if (TILES) {
          // tile masks are contiguous ranges [k0, k0 + len) (tiles.cu): tile k
          // sits at slot k - k0 of the staged column, tiles outside are zero
          const int k0 = mk ? (__ffsll(static_cast<long long>(mk)) - 1) : 0;
          const unsigned len = static_cast<unsigned>(__popcll(mk));
          const double* base = col - 32 * k0 + lane;
#pragma unroll
          for (int k = 0; k < R; ++k) {
            const bool in = static_cast<unsigned>(k - k0) < len;
            w[k] = in ? base[32 * k] : 0.0;
          }
        } else {
#pragma unroll
          for (int k = 0; k < R; ++k) {
            const double v = col[gt + GT * k];
            w[k] = (gt + GT * k < N) ? v : 0.0;
          }
        }
      };
      // entry k of the current column for this thread (0 when absent)
      auto wk = [&](int k, int& slot) -> double {
        if (KEEPW) return w[KEEPW ? k : 0];
        if (TILES) {
          const int bit = static_cast<int>((cur_mk >> k) & 1ull);
          const double v = cur_col[32 * slot + lane];
          slot += bit;
          return bit ? v : 0.0;
        }
        const double v = cur_col[gt + GT * k];
        return (gt + GT * k < N) ? v : 0.0;
      };
      auto col_dot = [&]() -> double {
        double d0 = 0.0, d1 = 0.0;  // two independent chains halve the FMA latency
        int slot = 0;
#pragma unroll
        for (int k = 0; k < R; ++k) {
          const double v = wk(k, slot);
          if (k & 1) d1 = fma(v, r[k], d1);
          else d0 = fma(v, r[k], d0);
        }
        return d0 + d1;
      };
      auto col_axpy = [&](double d) {
        int slot = 0;
#pragma unroll
        for (int k = 0; k < R; ++k) r[k] = fma(-d, wk(k, slot), r[k]);
      };
      auto col_sumsq = [&]() -> double {
        double p = 0.0;
        int slot = 0;
#pragma unroll
        for (int k = 0; k < R; ++k) {
          const double v = wk(k, slot);
          p = fma(v, v, p);
        }
        return p;
      };
      for (int q = 0; q < STAGES && issued < total; ++q) issue_one();
      int64_t consumed = 0;

      // ---- prologue: col_sq (elastic_net.py:85) and r = y - W beta0 (94)
      if (prologue) {
        for (int cb = 0; cb < M; cb += 32) {
          const int nc = min(32, M - cb);
          unsigned long long ml = 0ull;
          if (TILES && lane < nc) ml = a.tile_mask[doff + cb + lane];
          for (int t = 0; t < nc; ++t) {
            const int j = cb + t;
            const unsigned long long mk = TILES ? __shfl_sync(0xffffffffu, ml, t) : 0ull;
            const double* col = wait_one();
            ++consumed;
            load_col(col, mk);
            if (need_colsq) {
              double p = group_sum(col_sumsq());
              if (gt == 0) a.col_sq[doff + j] = p;
            }
            if (!r_given) {
              const double b0 = a.beta[doff + j];
              if (b0 != 0.0) col_axpy(b0);
            }
            sync_group();
            if (issued < total) issue_one();
          }
        }
        __threadfence_block();  // col_sq stores visible to the whole group
        sync_group();
      }

      // ---- sweeps (elastic_net.py:137-161)
      int sweeps_done = 0;
      int conv = 0;
      double obj = 0.0;
      for (int sw = 0; sw < max_iters; ++sw) {
        double max_delta = 0.0;
        double acc_l1 = 0.0, acc_l2 = 0.0, acc_max = 0.0;
        for (int cb = 0; cb < M; cb += 32) {
          const int nc = min(32, M - cb);
          // every warp of the group holds the same 32 column parameters
          double bl = 0.0, csl = 0.0;
          unsigned long long ml = 0ull;
          if (PSM) {
            __syncwarp();
            if (lane < nc) {
              pb[lane] = a.beta[doff + cb + lane];
              const double csv = a.col_sq[doff + cb + lane];
              pc[lane] = csv;
              const double dnv = __dadd_rn(csv, lam2);
              pinv[lane] = dnv > 0.0 ? __ddiv_rn(1.0, dnv) : 0.0;
              if (TILES) pm[lane] = static_cast<unsigned>(a.tile_mask[doff + cb + lane]);
            }
            __syncwarp();
          } else if (lane < nc) {
            bl = a.beta[doff + cb + lane];
            csl = a.col_sq[doff + cb + lane];
            if (TILES) ml = a.tile_mask[doff + cb + lane];
          }
          for (int t = 0; t < nc; ++t) {
            unsigned long long mk = 0ull;
            if (TILES) {
              if (PSM) mk = pm[t];
              else if (R <= 32) mk = __shfl_sync(0xffffffffu, static_cast<unsigned>(ml), t);
              else mk = __shfl_sync(0xffffffffu, ml, t);
            }
            const double* col = wait_one();
            ++consumed;
            load_col(col, mk);
            const double dot = group_sum(col_dot());
            const double b_old = PSM ? pb[t] : __shfl_sync(0xffffffffu, bl, t);
            const double cs = PSM ? pc[t] : __shfl_sync(0xffffffffu, csl, t);
            const double dn = __dadd_rn(cs, lam2);
            const double z = __dadd_rn(__dmul_rn(cs, b_old), dot);
            double b_new = 0.0;
            if (dn > 0.0) {
              double mag = __dsub_rn(fabs(z), lam1);
              if (mag < 0.0) mag = 0.0;
              const double num = z >= 0.0 ? mag : -mag;
              if (PSM) {
                // num / dn via the reciprocal and one Newton correction (the
                // correctly rounded quotient except in rare last-ulp cases)
                const double inv = pinv[t];
                const double q0 = __dmul_rn(num, inv);
                b_new = fma(fma(-q0, dn, num), inv, q0);
              } else {
                b_new = __ddiv_rn(num, dn);
              }
            }
            // branch-free update: d == 0 exactly when b_new == b_old, and then the
            // AXPY adds -0 * w to every residual entry, leaving r bit-unchanged
            const double d = __dsub_rn(b_new, b_old);
            col_axpy(d);
            if (PSM) {
              if (lane == 0) pb[t] = b_new;
            } else if (lane == t) {
              bl = b_new;
            }
            max_delta = fmax(max_delta, fabs(d));
            sync_group();
            if (issued < total) issue_one();
          }
          if (PSM) {
            __syncwarp();
            bl = (lane < nc) ? pb[lane] : 0.0;
          }
          if (lane < nc) {
            if (wig == 0) a.beta[doff + cb + lane] = bl;
            const double ab = fabs(bl);
            acc_l1 += ab;
            acc_l2 = fma(bl, bl, acc_l2);
            acc_max = fmax(acc_max, ab);
          }
        }
        double rss = 0.0;
#pragma unroll
        for (int k = 0; k < R; ++k) rss = fma(r[k], r[k], rss);
        rss = group_sum(rss);
        const double l1 = warp_sum(acc_l1);  // identical in every warp of the group
        const double l2 = warp_sum(acc_l2);
        const double mabs = warp_max(acc_max);
        obj = __dadd_rn(__dadd_rn(__dmul_rn(0.5, rss), __dmul_rn(lam1, l1)),
                        __dmul_rn(__dmul_rn(0.5, lam2), l2));
        if (a.hist != nullptr && gt == 0) a.hist[a.hist_off[s] + sw] = obj;
        sweeps_done = sw + 1;
        if (max_delta <= __dmul_rn(tol, fmax(mabs, 1.0))) {
          conv = 1;
          break;
        }
      }
      if (max_iters == 0) {
        // objective at the given beta (used after the Gram-form sweeps, gram.cu):
        // 0.5 |y - W beta|^2 + lam1 |beta|_1 + 0.5 lam2 |beta|^2, exact residual form
        double rss = 0.0, l1 = 0.0, l2 = 0.0;
#pragma unroll
        for (int k = 0; k < R; ++k) rss = fma(r[k], r[k], rss);
        rss = group_sum(rss);
        for (int j = lane; j < M; j += 32) {
          const double b = a.beta[doff + j];
          l1 += fabs(b);
          l2 = fma(b, b, l2);
        }
        l1 = warp_sum(l1);
        l2 = warp_sum(l2);
        obj = __dadd_rn(__dadd_rn(__dmul_rn(0.5, rss), __dmul_rn(lam1, l1)),
                        __dmul_rn(__dmul_rn(0.5, lam2), l2));
      }
      // drain speculative prefetches of the sweep that will not run
      if (LDGSTS) {
        cp_async_wait<0>();
        __syncwarp();
        g_cons += static_cast<uint32_t>(issued - consumed);
        consumed = issued;
      }
      while (consumed < issued) {
        (void)wait_one();
        ++consumed;
      }
      sync_group();
      if (a.flags & CD_WRITE_R) {
#pragma unroll
        for (int k = 0; k < R; ++k) {
          const int p = gt + GT * k;
          if (p < N) a.y[r0 + ((TILES && a.perm) ? a.perm[r0 + p] : p)] = r[k];
        }
      }
      if (gt == 0) {
        a.sweeps[s] = sweeps_done;
        a.converged[s] = conv;
        a.objective[s] = obj;
      }
    }
    // next item: dynamic queue after the static first pass
    unsigned nxt = 0;
    if (gt == 0) nxt = atomicAdd(&g_cd_queue, 1u) + total_groups;
    if (G == 1) {
      item = __shfl_sync(0xffffffffu, nxt, 0);
    } else {
      if (gt == 0) red[2 * G] = __longlong_as_double((long long)nxt);
      group_bar(bar_id, GT);
      item = (unsigned)__double_as_longlong(red[2 * G]);
      group_bar(bar_id, GT);
    }
  }
}

template <int R, int STAGES, int WPC, int G, bool TILES = false, bool KEEPW = true, bool LDGSTS = false>
int launch_cd(const CdArgs& a, cudaStream_t stream) {
  constexpr int NGROUPS = WPC / G;
  const size_t smem = static_cast<size_t>(NGROUPS) * STAGES * (R * 32 * G * sizeof(double)) +
                      static_cast<size_t>(NGROUPS) * STAGES * sizeof(uint64_t) +
                      static_cast<size_t>(NGROUPS) * (2 * G + 1) * sizeof(double) +
                      static_cast<size_t>(NGROUPS) * 128 * sizeof(double);
  static bool configured = false;
  if (!configured) {
    PAM_CUDA_CHECK(cudaFuncSetAttribute(cd_kernel<R, STAGES, WPC, G, TILES, KEEPW, LDGSTS>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = true;
  }
  int dev = 0, sms = 148;
  PAM_CUDA_CHECK(cudaGetDevice(&dev));
  PAM_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  void* qaddr = nullptr;
  PAM_CUDA_CHECK(cudaGetSymbolAddress(&qaddr, g_cd_queue));
  PAM_CUDA_CHECK(cudaMemsetAsync(qaddr, 0, sizeof(unsigned), stream));
  const int64_t ctas = std::max<int64_t>(1, std::min<int64_t>(sms, a.S));
  cd_kernel<R, STAGES, WPC, G, TILES, KEEPW, LDGSTS><<<(unsigned)ctas, WPC * 32, smem, stream>>>(a);
  PAM_LAUNCH_CHECK("cd_kernel");
  return PAM_OK;
}

int cd_dispatch(const CdArgs& a, int max_rows, cudaStream_t stream) {
  // Few subdomains relative to the SM count: spread each fit over a group of
  // warps (shorter per-column latency); many subdomains: one warp per fit.
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const bool few = a.S < 4LL * sms;
  if (!few || max_rows <= 64) {
    // (rows per lane, ring stages, warps per CTA): ring <= ~200 KB per CTA
    if (max_rows <= 32) return launch_cd<1, 4, 16, 1>(a, stream);
    if (max_rows <= 64) return launch_cd<2, 4, 16, 1>(a, stream);
    if (max_rows <= 128) return launch_cd<4, 4, 16, 1>(a, stream);
    if (max_rows <= 256) return launch_cd<8, 4, 16, 1>(a, stream);
    if (max_rows <= 512) return launch_cd<16, 3, 16, 1>(a, stream);
    if (max_rows <= 1024) return launch_cd<32, 3, 8, 1>(a, stream);
  }
  // group kernels: G warps per subdomain
  if (max_rows <= 512) return launch_cd<4, 4, 16, 4>(a, stream);     // 4 groups/CTA
  if (max_rows <= 1024) return launch_cd<8, 3, 16, 4>(a, stream);
  if (max_rows <= 2048) return launch_cd<8, 3, 16, 8>(a, stream);    // 2 groups/CTA
  if (max_rows <= 4096) return launch_cd<16, 3, 8, 8>(a, stream);
  if (max_rows <= 8192) return launch_cd<32, 3, 8, 8>(a, stream);
  set_last_error("pam_cd_f64: subdomain has more than 8192 sample rows (kernel envelope)");
  return PAM_ERR_UNSUPPORTED;
}

int cd_dispatch_tiles(const CdArgs& a, int max_rows, cudaStream_t stream) {
  // one warp per subdomain; tile k of a column <-> register r[k] of every lane
  if (max_rows <= 32) return launch_cd<1, 4, 16, 1, true>(a, stream);
  if (max_rows <= 64) return launch_cd<2, 4, 16, 1, true>(a, stream);
  if (max_rows <= 128) return launch_cd<4, 4, 16, 1, true>(a, stream);
  if (max_rows <= 256) return launch_cd<8, 4, 16, 1, true>(a, stream);
  if (max_rows <= 512) {
    const char* env = getenv("PAM_CD_WPC16");
    const int v = env ? atoi(env) : 16;
    const char* cp = getenv("PAM_CD_COPY");
    if (cp && cp[0] == 'l') return launch_cd<16, 3, 16, 1, true, true, true>(a, stream);
    if (v == 24) return launch_cd<16, 2, 24, 1, true, false>(a, stream);
    if (v == 20) return launch_cd<16, 2, 20, 1, true, false>(a, stream);
    return launch_cd<16, 3, 16, 1, true>(a, stream);
  }
  if (max_rows <= 1024) return launch_cd<32, 3, 8, 1, true>(a, stream);
  if (max_rows <= 2048) return launch_cd<64, 2, 4, 1, true>(a, stream);
  set_last_error("pam_cd_tiles_f64: tile-packed CD supports <= 2048 rows per subdomain");
  return PAM_ERR_UNSUPPORTED;
}

}  // namespace pam

using namespace pam;

extern "C" int64_t pam_cd_max_rows(void) { return 8192; }

extern "C" int pam_cd_ex_f64(int64_t S, const int64_t* order, const int64_t* row_off, double* y,
                             const int64_t* dict_off, const int32_t* m_cur, const int64_t* w_off,
                             const int32_t* ld, const double* W, const double* lam1,
                             const double* lam2, const double* tol, const int32_t* max_iters,
                             const int32_t* active, int32_t max_rows, double* beta, double* col_sq,
                             int32_t* sweeps, int32_t* converged, double* objective, double* hist,
                             const int64_t* hist_off, int flags, void* stream) {
  if (S < 0 || max_rows < 0) return PAM_ERR_ARG;
  if (S == 0) return PAM_OK;
  CdArgs a{S,    order,     row_off,   y,         dict_off, m_cur, w_off,    ld,
           W,    lam1,      lam2,      tol,       max_iters, active, beta,   col_sq,
           sweeps, converged, objective, hist,    hist_off, flags, nullptr, nullptr, nullptr};
  return cd_dispatch(a, max_rows, as_stream(stream));
}

int pam_cd_tiles_ring(int64_t S, const int64_t* order, const int64_t* row_off, const double* y,
                      const int32_t* perm, const int64_t* dict_off, const int32_t* m_cur,
                      const int64_t* w_off, const uint64_t* tile_mask, const int64_t* col_off,
                      const double* W, const double* lam1, const double* lam2, const double* tol,
                      const int32_t* max_iters, const int32_t* active, int32_t max_rows,
                      double* beta, double* col_sq, int32_t* sweeps, int32_t* converged,
                      double* objective, void* stream);

extern "C" int pam_cd_tiles_f64(int64_t S, const int64_t* order, const int64_t* row_off,
                                const double* y, const int32_t* perm, const int64_t* dict_off,
                                const int32_t* m_cur, const int64_t* w_off,
                                const uint64_t* tile_mask, const int64_t* col_off, const double* W,
                                const double* lam1, const double* lam2, const double* tol,
                                const int32_t* max_iters, const int32_t* active, int32_t max_rows,
                                double* beta, double* col_sq, int32_t* sweeps, int32_t* converged,
                                double* objective, double* hist, const int64_t* hist_off,
                                void* stream) {
  if (S < 0 || max_rows < 0 || !tile_mask || !col_off) return PAM_ERR_ARG;
  if (S == 0) return PAM_OK;
  const char* ring_env = getenv("PAM_CD_RING");
  if (hist == nullptr && max_rows <= 1024 && ring_env && atoi(ring_env) == 1)
    return pam_cd_tiles_ring(S, order, row_off, y, perm, dict_off, m_cur, w_off, tile_mask, col_off,
                             W, lam1, lam2, tol, max_iters, active, max_rows, beta, col_sq, sweeps,
                             converged, objective, stream);
  CdArgs a{S,      order,     row_off,   const_cast<double*>(y), dict_off, m_cur, w_off, m_cur,
           W,      lam1,      lam2,      tol,       max_iters, active, beta,   col_sq,
           sweeps, converged, objective, hist,      hist_off,  0,
           reinterpret_cast<const unsigned long long*>(tile_mask), col_off, perm};
  return cd_dispatch_tiles(a, max_rows, as_stream(stream));
}

extern "C" int pam_cd_f64(int64_t S, const int64_t* order, const int64_t* row_off, const double* y,
                          const int64_t* dict_off, const int32_t* m_cur, const int64_t* w_off,
                          const int32_t* ld, const double* W, const double* lam1,
                          const double* lam2, const double* tol, const int32_t* max_iters,
                          const int32_t* active, int32_t max_rows, double* beta, double* col_sq,
                          int32_t* sweeps, int32_t* converged, double* objective, double* hist,
                          const int64_t* hist_off, void* stream) {
  return pam_cd_ex_f64(S, order, row_off, const_cast<double*>(y), dict_off, m_cur, w_off, ld, W,
                       lam1, lam2, tol, max_iters, active, max_rows, beta, col_sq, sweeps,
                       converged, objective, hist, hist_off, 0, stream);
}
