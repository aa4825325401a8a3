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
// K2b), ~2 FMA per 8 bytes.  For many fits of 257-512 rows (C4) the dual
// kernel puts two fits in one warp, one per 16-lane half (cd_dual_kernel).
#include "cd_common.cuh"

#include <stdlib.h>

#include <algorithm>

namespace pam {

// named barrier over the G warps of one subdomain group (G > 1 only)
__device__ __forceinline__ void group_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Dense column-major design matrices (tau = 0, the Gram form's exact
// objective pass, rows > 1024).  R: rows per thread, STAGES: ring depth,
// WPC: warps per CTA, G: warps per subdomain group (rows of a subdomain split
// over the G*32 threads).  Whole columns are staged HBM -> SMEM by
// cp.async.bulk, STAGES ahead of the consumer.
template <int R, int STAGES, int WPC, int G>
__global__ void __launch_bounds__(WPC * 32, 1) cd_kernel(const CdArgs a) {
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
  // per-warp column-parameter block (G == 1): beta, col_sq, 1/(col_sq+lam2)
  // of the current 32-column chunk, read by warp-uniform smem broadcasts
  constexpr bool PSM = (G == 1);
  double* prm_base = reinterpret_cast<double*>(smem_raw) +
                     (static_cast<size_t>(NGROUPS) * STAGES * LDMAX) + NGROUPS * STAGES +
                     NGROUPS * (2 * G + 1);
  double* pb = prm_base + grp * 96;
  double* pc = pb + 32;
  double* pinv = pb + 64;  // 1 / (col_sq + lam2): division by reciprocal + one FMA correction

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

      // residual / targets into registers (thread gt owns rows gt + GT*k)
      double r[R];
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const int p = gt + GT * k;
        r[k] = (p < N) ? a.y[r0 + p] : 0.0;
      }

      // continuous column stream: [prologue M columns] + max_iters * M columns
      const int64_t total = (prologue ? (int64_t)M : 0) + (int64_t)max_iters * M;
      int64_t issued = 0;
      int next_col = 0;
      auto issue_one = [&]() {
        if (gt == 0) {
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
        mbar_wait(&bars[st], (g_cons / STAGES) & 1u);
        ++g_cons;
        return ring + st * LDMAX;
      };
      // Column staging: the column's entries for this thread's rows go to
      // registers once and serve both the dot and the AXPY.  Branch-free: rows
      // past N read an in-bounds smem word and select 0.
      double w[R];
      auto load_col = [&](const double* col) {
#pragma unroll
        for (int k = 0; k < R; ++k) {
          const double v = col[gt + GT * k];
          w[k] = (gt + GT * k < N) ? v : 0.0;
        }
      };
      auto col_dot = [&]() -> double {
        double d0 = 0.0, d1 = 0.0;  // two independent chains halve the FMA latency
#pragma unroll
        for (int k = 0; k < R; ++k) {
          if (k & 1) d1 = fma(w[k], r[k], d1);
          else d0 = fma(w[k], r[k], d0);
        }
        return d0 + d1;
      };
      auto col_axpy = [&](double d) {
#pragma unroll
        for (int k = 0; k < R; ++k) r[k] = fma(-d, w[k], r[k]);
      };
      auto col_sumsq = [&]() -> double {
        double p = 0.0;
#pragma unroll
        for (int k = 0; k < R; ++k) p = fma(w[k], w[k], p);
        return p;
      };
      for (int q = 0; q < STAGES && issued < total; ++q) issue_one();
      int64_t consumed = 0;

      // ---- prologue: col_sq (elastic_net.py:85) and r = y - W beta0 (94)
      if (prologue) {
        for (int j = 0; j < M; ++j) {
          const double* col = wait_one();
          ++consumed;
          load_col(col);
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
          if (PSM) {
            __syncwarp();
            if (lane < nc) {
              pb[lane] = a.beta[doff + cb + lane];
              const double csv = a.col_sq[doff + cb + lane];
              pc[lane] = csv;
              const double dnv = __dadd_rn(csv, lam2);
              pinv[lane] = dnv > 0.0 ? __ddiv_rn(1.0, dnv) : 0.0;
            }
            __syncwarp();
          } else if (lane < nc) {
            bl = a.beta[doff + cb + lane];
            csl = a.col_sq[doff + cb + lane];
          }
          for (int t = 0; t < nc; ++t) {
            const double* col = wait_one();
            ++consumed;
            load_col(col);
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
      while (consumed < issued) {
        (void)wait_one();
        ++consumed;
      }
      sync_group();
      if (a.flags & CD_WRITE_R) {
#pragma unroll
        for (int k = 0; k < R; ++k) {
          const int p = gt + GT * k;
          if (p < N) a.y[r0 + p] = r[k];
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
    if (gt == 0) nxt = atomicAdd(a.queue, 1u) + total_groups;
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

// ----------------------------------------------------------------------------
// Lean tile-stream CD (one fit per warp, tile-packed batches of <= 1024 rows).
//
// Same semantics as cd_kernel over the tile-packed design matrices of
// tiles.cu, with the per-column instruction count cut down (the generic
// per-column loop is issue-bound; profiles/r01_*):
//  * every column is ONE contiguous run of kept 32-row tiles [a0, a0+la),
//    staged packed at the slot start by one cp.async.bulk; a lane addresses
//    its tile with one base and one predicate, out-of-run tiles read a
//    CTA-wide zero block;
//  * paired-row layout (R even): lane l owns packed rows 64q + 2l + {0,1}, so
//    one 16-byte shared load feeds two registers (tile 2q + (l >> 4));
//  * per-32-column chunk parameters (beta, col_sq, 1/(col_sq+lam2), run
//    code, packed offset) are prefetched into registers one chunk ahead and
//    published to a per-warp smem block: no global load on the column loop;
//  * the issue path is one LDS + expect_tx + one bulk copy by lane 0.
// Measured alternatives: per-lane cp.async staging, two-run
// masks, dense tile placement with stale-tile clears and deeper rings were
// all slower and have been removed.

template <int R, int STAGES, int WPC>
__global__ void __launch_bounds__(WPC * 32, 1) cd_tile_kernel(const CdArgs a) {
  constexpr int SLOT = R * 32;  // doubles per ring slot (one dense column)
  constexpr int PBLK = 144;     // doubles per warp: pb/pc/pinv[32] + pk/ioff/icode[32]
  static_assert(R <= 32 && STAGES <= 8, "lean tile CD envelope");
  constexpr bool VEC = (R % 2) == 0;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  double* const ring_all = reinterpret_cast<double*>(smem_raw);
  double* const ring = ring_all + static_cast<size_t>(warp) * STAGES * SLOT;
  uint64_t* const bars = reinterpret_cast<uint64_t*>(ring_all + static_cast<size_t>(WPC) * STAGES * SLOT) +
                         warp * STAGES;
  double* const pb = reinterpret_cast<double*>(reinterpret_cast<uint64_t*>(
                         ring_all + static_cast<size_t>(WPC) * STAGES * SLOT) + WPC * STAGES) +
                     warp * PBLK;
  double* const pc = pb + 32;
  double* const pinv = pb + 64;
  int* const pk = reinterpret_cast<int*>(pb + 96);  // consumer chunk: run codes
  int* const ioff = pk + 32;                        // issue chunk: packed offsets (doubles)
  int* const icode = pk + 64;                       // issue chunk: run codes
  // CTA-wide block of SLOT zero doubles: out-of-run tiles load from here
  double* const zero_blk = reinterpret_cast<double*>(reinterpret_cast<uint64_t*>(
                               ring_all + static_cast<size_t>(WPC) * STAGES * SLOT) + WPC * STAGES) +
                           WPC * PBLK;
  const uint32_t ring_s = smem_u32(ring);
  const uint32_t bar_s = smem_u32(bars);
  const uint32_t zero_s = smem_u32(zero_blk) + 16u * lane;
  // this lane's tile in pair q is 2q + half (VEC) or k (scalar layout)
  const int half = lane >> 4;

  for (int i = threadIdx.x; i < SLOT; i += WPC * 32) zero_blk[i] = 0.0;
  if (lane == 0) {
    for (int i = 0; i < STAGES; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncthreads();

  int st = 0;       // consumer ring slot
  uint32_t ph = 0;  // its mbarrier phase parity
  int ist = 0;      // issue ring slot
  unsigned item = warp * gridDim.x + blockIdx.x;
  const unsigned total_warps = gridDim.x * WPC;

  while (item < a.S) {
    const int64_t s = a.order ? a.order[item] : static_cast<int64_t>(item);
    if (a.active == nullptr || a.active[s] != 0) {
      const int64_t r0 = a.row_off[s];
      const int N = static_cast<int>(a.row_off[s + 1] - r0);
      const int M = a.m_cur[s];
      const int64_t doff = a.dict_off[s];
      const double* Ws = a.W + a.w_off[s];
      const int64_t* colo = a.col_off + doff;
      const unsigned long long* tmk = a.tile_mask + doff;
      double* betas = a.beta + doff;
      double* colsq = a.col_sq + doff;
      const double lam1 = a.lam1[s], lam2 = a.lam2[s], tol = a.tol[s];
      const int max_iters = a.max_iters[s];

      double r[R];
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const int p = VEC ? (64 * (k >> 1) + 2 * lane + (k & 1)) : (lane + 32 * k);
        const int row = a.perm ? (p < N ? a.perm[r0 + p] : 0) : p;
        r[k] = (p < N) ? a.y[r0 + row] : 0.0;
      }

      // ---- issue side: column stream = [prologue M] + max_iters * M
      // 32-bit stream counters: the host rejects M * (1 + max_iters) >= 2^31
      const int total = M * (1 + max_iters);
      int issued = 0;
      int next_col = 0;
      // issue parameters of the next chunk (lane = column); the mask is decoded
      // at publish time so the global load's latency stays off the column loop
      int pf_off = 0;
      unsigned long long pf_mk = 0ull;
      auto fetch_issue = [&](int cb) {
        const int c = cb + lane;
        pf_off = (c < M) ? static_cast<int>(colo[c]) : 0;
        pf_mk = (c < M) ? tmk[c] : 0ull;
      };
      fetch_issue(0);
      // dep: a value computed from this warp's loads of the slot being refilled,
      // so the bulk copy cannot be issued before those shared loads completed
      auto issue_one = [&](double dep) {
        const int c = next_col & 31;
        if (c == 0) {
          __syncwarp();
          ioff[lane] = pf_off;
          icode[lane] = tile_code(pf_mk);
          __syncwarp();
          fetch_issue(next_col + 32 < M ? next_col + 32 : 0);
        }
        if (lane == 0) {
          const int code = icode[c];
          const uint32_t bytes = static_cast<uint32_t>(code_tiles(code)) * 256u;
          const uint32_t bar = bar_s + ist * 8;
          if (bytes) {
            mbar_expect_s(bar, bytes);
            bulk_g2s_dep(ring_s + ist * (SLOT * 8), Ws + ioff[c], bytes, bar, dep);
          } else {
            mbar_arrive_s(bar);
          }
        }
        if (++ist == STAGES) ist = 0;
        ++issued;
        if (++next_col == M) next_col = 0;
      };
      for (int q = 0; q < STAGES && issued < total; ++q) issue_one(0.0);

      // ---- consumer side
      int consumed = 0;
      bool ready = false;  // next slot's mbarrier phase already observed complete
      double w[R];
      auto load_w = [&](int code) {
        const double* col = ring + st * SLOT;
        if (!ready) mbar_wait_s(bar_s + st * 8, ph);
        const int a0 = code & 0xff, la = (code >> 8) & 0xff;
        if (VEC) {
          // unconditional 16-byte shared loads; out-of-run tiles are redirected
          // to the zero block (one select per tile pair, no zeroing moves)
          const uint32_t cA = ring_s + st * (SLOT * 8) + 16u * lane - 256u * a0;
          const int hA = half - a0;
#pragma unroll
          for (int q = 0; q < R / 2; ++q) {
            const bool inA = static_cast<unsigned>(hA + 2 * q) < static_cast<unsigned>(la);
            lds_v2((inA ? cA : zero_s) + 512u * q, w[2 * q], w[2 * q + 1]);
          }
        } else {
          const double* bA = col - 32 * a0 + lane;
#pragma unroll
          for (int k = 0; k < R; ++k) {
            const bool inA = static_cast<unsigned>(k - a0) < static_cast<unsigned>(la);
            w[k] = inA ? bA[32 * k] : 0.0;
          }
        }
      };
      // the column in slot st is in registers: refill the slot (depending on
      // `dep`, a value computed from the loaded words) and step the ring
      auto advance = [&](double dep) {
        if (issued < total) issue_one(dep);
        if (++st == STAGES) {
          st = 0;
          ph ^= 1u;
        }
        ++consumed;
        // non-blocking look at the next slot now, so the barrier round trip
        // overlaps the reduction and update of this column
        ready = (consumed < issued) && mbar_test_s(bar_s + st * 8, ph);
      };

      // prologue: col_sq (elastic_net.py:85) and r = y - W beta0 (elastic_net.py:94)
      for (int cb = 0; cb < M; cb += 32) {
        const int nc = min(32, M - cb);
        int cl = 0;
        double bl0 = 0.0, csl = 0.0;
        if (lane < nc) {
          cl = tile_code(tmk[cb + lane]);
          bl0 = betas[cb + lane];
        }
        for (int t = 0; t < nc; ++t) {
          load_w(__shfl_sync(0xffffffffu, cl, t));
          double p0 = 0.0, p1 = 0.0;
#pragma unroll
          for (int k = 0; k < R; ++k) {
            if (k & 1) p1 = fma(w[k], w[k], p1);
            else p0 = fma(w[k], w[k], p0);
          }
          const double pp = p0 + p1;
          advance(pp);
          const double p = warp_sum(pp);
          if (lane == t) csl = p;
          const double b0 = __shfl_sync(0xffffffffu, bl0, t);
          if (b0 != 0.0) {
#pragma unroll
            for (int k = 0; k < R; ++k) r[k] = fma(-b0, w[k], r[k]);
          }
        }
        if (lane < nc) colsq[cb + lane] = csl;  // re-read below by the same lane
      }

      // sweeps (elastic_net.py:137-161); chunk parameters prefetched one chunk ahead
      const bool one_chunk = M <= 32;
      double nb_l = 0.0, ncs_l = 0.0;
      unsigned long long nk_mk = 0ull;  // decoded at publish time
      auto fetch_params = [&](int cb) {
        const int c = cb + lane;
        nb_l = (c < M) ? betas[c] : 0.0;
        ncs_l = (c < M) ? colsq[c] : 0.0;
        nk_mk = (c < M) ? tmk[c] : 0ull;
      };
      fetch_params(0);
      int sweeps_done = 0, conv = 0;
      double obj = 0.0;
      for (int sw = 0; sw < max_iters; ++sw) {
        double max_delta = 0.0, acc_l1 = 0.0, acc_l2 = 0.0, acc_max = 0.0;
        for (int cb = 0; cb < M; cb += 32) {
          const int nc = min(32, M - cb);
          __syncwarp();
          if (sw == 0 || !one_chunk) {
            pb[lane] = nb_l;
            pc[lane] = ncs_l;
            const double dnv = __dadd_rn(ncs_l, lam2);
            pinv[lane] = dnv > 0.0 ? __ddiv_rn(1.0, dnv) : 0.0;
            pk[lane] = tile_code(nk_mk);
            if (!one_chunk) fetch_params(cb + 32 < M ? cb + 32 : 0);
          }
          __syncwarp();
          for (int t = 0; t < nc; ++t) {
            load_w(pk[t]);
            // four independent FMA chains: the dot sits on the per-column critical path
            double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
#pragma unroll
            for (int k = 0; k < R; ++k) {
              if ((k & 3) == 0) d0 = fma(w[k], r[k], d0);
              else if ((k & 3) == 1) d1 = fma(w[k], r[k], d1);
              else if ((k & 3) == 2) d2 = fma(w[k], r[k], d2);
              else d3 = fma(w[k], r[k], d3);
            }
            const double part = (d0 + d1) + (d2 + d3);
            advance(part);  // slot free once its words are in registers
            const double b_old = pb[t];
            const double cs = pc[t];
            const double inv = pinv[t];
            const double cb_old = __dmul_rn(cs, b_old);  // off the dot's critical path
            const double dn = __dadd_rn(cs, lam2);
            const double dot = warp_sum(part);
            const double z = __dadd_rn(cb_old, dot);
            // soft threshold sign(z) max(|z| - lam1, 0) with both signed numerators
            // formed in parallel (z - lam1 == |z| - lam1 for z > 0, z + lam1 ==
            // -(|z| - lam1) for z < 0, exactly), then num / (cs + lam2) by the
            // reciprocal and one FMA correction; inv == 0 (non-positive
            // denominator) yields 0
            const double np_ = __dsub_rn(z, lam1), nn_ = __dadd_rn(z, lam1);
            const double qp = __dmul_rn(np_, inv), qn = __dmul_rn(nn_, inv);
            const double bp = fma(fma(-qp, dn, np_), inv, qp);
            const double bn = fma(fma(-qn, dn, nn_), inv, qn);
            const double b_new = np_ > 0.0 ? bp : (nn_ < 0.0 ? bn : 0.0);
            const double d = __dsub_rn(b_new, b_old);
#pragma unroll
            for (int k = 0; k < R; ++k) r[k] = fma(-d, w[k], r[k]);
            if (lane == 0) pb[t] = b_new;
            const double ad = fabs(d);
            max_delta = ad > max_delta ? ad : max_delta;  // fmax without the NaN fix-up
          }
          __syncwarp();
          if (lane < nc) {
            const double bl = pb[lane];
            betas[cb + lane] = bl;
            const double ab = fabs(bl);
            acc_l1 += ab;
            acc_l2 = fma(bl, bl, acc_l2);
            acc_max = fmax(acc_max, ab);
          }
        }
        double rss0 = 0.0, rss1 = 0.0;
#pragma unroll
        for (int k = 0; k < R; ++k) {
          if (k & 1) rss1 = fma(r[k], r[k], rss1);
          else rss0 = fma(r[k], r[k], rss0);
        }
        const double rss = warp_sum(rss0 + rss1);
        const double l1 = warp_sum(acc_l1);
        const double l2 = warp_sum(acc_l2);
        const double mabs = warp_max(acc_max);
        obj = __dadd_rn(__dadd_rn(__dmul_rn(0.5, rss), __dmul_rn(lam1, l1)),
                        __dmul_rn(__dmul_rn(0.5, lam2), l2));
        if (a.hist != nullptr && lane == 0) a.hist[a.hist_off[s] + sw] = obj;
        sweeps_done = sw + 1;
        if (max_delta <= __dmul_rn(tol, fmax(mabs, 1.0))) {
          conv = 1;
          break;
        }
      }
      if (max_iters == 0) {
        // objective at the given beta (after the Gram-form sweeps, gram.cu)
        double rss = 0.0, l1 = 0.0, l2 = 0.0;
#pragma unroll
        for (int k = 0; k < R; ++k) rss = fma(r[k], r[k], rss);
        rss = warp_sum(rss);
        for (int j = lane; j < M; j += 32) {
          const double b = betas[j];
          l1 += fabs(b);
          l2 = fma(b, b, l2);
        }
        l1 = warp_sum(l1);
        l2 = warp_sum(l2);
        obj = __dadd_rn(__dadd_rn(__dmul_rn(0.5, rss), __dmul_rn(lam1, l1)),
                        __dmul_rn(__dmul_rn(0.5, lam2), l2));
      }
      // drain the prefetched columns of the sweep that will not run
      while (consumed < issued) {
        mbar_wait_s(bar_s + st * 8, ph);
        if (++st == STAGES) {
          st = 0;
          ph ^= 1u;
        }
        ++consumed;
      }
      __syncwarp();
      if (lane == 0) {
        a.sweeps[s] = sweeps_done;
        a.converged[s] = conv;
        a.objective[s] = obj;
      }
    }
    unsigned nxt = 0;
    if (lane == 0) nxt = atomicAdd(a.queue, 1u) + total_warps;
    item = __shfl_sync(0xffffffffu, nxt, 0);
  }
}

// ----------------------------------------------------------------------------
// Dual lean tile CD: two fits per warp, one per half-warp (<= 512 rows).
//
// The lean kernel at full C4 load (15 fits per SM) spends about a third of its
// per-column time on issue contention between the ~4 fits per scheduler and
// the rest on each fit's serial chain (occupancy probe).  Here a
// warp carries two independent fits in its two 16-lane halves: one issued
// instruction advances both, so the per-fit issue cost roughly halves, and the
// per-column warp reduction is 4 butterfly levels instead of 5.  Lane h of a
// half owns packed rows 32q + 2h + {0,1} (q = tile, R = 32 registers for 512
// rows), so one 16-byte shared load per tile feeds two registers.  Both fits
// walk a common column count Mx = max(M_a, M_b): columns past a fit's own M
// and every column of a finished fit read the zero block and leave beta
// unchanged (d = 0 exactly), so each half computes exactly what the one-fit
// lean kernel computes.  Ring slots hold one column per half; each slot's
// mbarrier takes one arrival per half (lanes 0 and 16 issue their half's bulk
// copy, or a plain arrival for an empty column).  Pairs are consecutive
// entries of the longest-first order, so paired fits have similar work.

template <int R, int STAGES, int WPC>
__global__ void __launch_bounds__(WPC * 32, 1) cd_dual_kernel(const CdArgs a) {
  constexpr int SLOTH = R * 16;  // doubles per half slot (one column of <= 16 R rows)
  constexpr int PBLK = 144;      // doubles per warp: pb/pc/pinv[32] + pk/ioff/icode[32] (index half*16 + c)
  static_assert(R % 2 == 0 && R <= 32 && STAGES <= 8, "dual lean tile CD envelope");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int half = lane >> 4;
  const int hl = lane & 15;
  const int hb = half * 16;  // this half's index base in the parameter blocks
  double* const ring_all = reinterpret_cast<double*>(smem_raw);
  uint64_t* const bars = reinterpret_cast<uint64_t*>(ring_all + static_cast<size_t>(WPC) * STAGES * 2 * SLOTH) +
                         warp * STAGES;
  double* const pb = reinterpret_cast<double*>(reinterpret_cast<uint64_t*>(
                         ring_all + static_cast<size_t>(WPC) * STAGES * 2 * SLOTH) + WPC * STAGES) +
                     warp * PBLK;
  double* const pc = pb + 32;
  double* const pinv = pb + 64;
  int* const pk = reinterpret_cast<int*>(pb + 96);
  int* const ioff = pk + 32;
  int* const icode = pk + 64;
  double* const zero_blk = reinterpret_cast<double*>(reinterpret_cast<uint64_t*>(
                               ring_all + static_cast<size_t>(WPC) * STAGES * 2 * SLOTH) + WPC * STAGES) +
                           WPC * PBLK;
  // slot st of this half: ring_h + st * (2 * SLOTH * 8) bytes
  const uint32_t ring_h = smem_u32(ring_all + static_cast<size_t>(warp) * STAGES * 2 * SLOTH) + half * (SLOTH * 8);
  const uint32_t bar_s = smem_u32(bars);
  const uint32_t zero_s = smem_u32(zero_blk) + 16u * hl;
  constexpr uint32_t SLOT_B = 2u * SLOTH * 8u;

  for (int i = threadIdx.x; i < SLOTH; i += WPC * 32) zero_blk[i] = 0.0;
  if (lane == 0) {
    for (int i = 0; i < STAGES; ++i) mbar_init(&bars[i], 2);
    fence_mbar_init();
  }
  __syncthreads();

  int st = 0;
  uint32_t ph = 0;
  int ist = 0;
  const int64_t P = (a.S + 1) / 2;  // fit pairs
  unsigned item = warp * gridDim.x + blockIdx.x;
  const unsigned total_warps = gridDim.x * WPC;

  while (item < P) {
    const int64_t idx = 2 * static_cast<int64_t>(item) + half;
    int64_t s = -1;
    if (idx < a.S) {
      s = a.order ? a.order[idx] : idx;
      if (a.active != nullptr && a.active[s] == 0) s = -1;
    }
    const bool hvalid = s >= 0;
    const int64_t sx = hvalid ? s : 0;
    const int64_t r0 = a.row_off[sx];
    const int N = hvalid ? static_cast<int>(a.row_off[sx + 1] - r0) : 0;
    const int M = hvalid ? a.m_cur[sx] : 0;
    const int64_t doff = a.dict_off[sx];
    const double* Ws = a.W + a.w_off[sx];
    const int64_t* colo = a.col_off + doff;
    const unsigned long long* tmk = a.tile_mask + doff;
    double* betas = a.beta + doff;
    double* colsq = a.col_sq + doff;
    const double lam1 = a.lam1[sx], lam2 = a.lam2[sx], tol = a.tol[sx];
    const int mi = hvalid ? a.max_iters[sx] : 0;
    const int Mo = __shfl_xor_sync(0xffffffffu, M, 16);
    const int Mx = M > Mo ? M : Mo;
    const int mio = __shfl_xor_sync(0xffffffffu, mi, 16);
    const int mix = mi > mio ? mi : mio;

    double r[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int p = 32 * (k >> 1) + 2 * hl + (k & 1);
      const int row = a.perm ? (p < N ? a.perm[r0 + p] : 0) : p;
      r[k] = (p < N) ? a.y[r0 + row] : 0.0;
    }

    // ---- issue side: column stream = [prologue Mx] + mix * Mx (both halves in step)
    const int64_t total = static_cast<int64_t>(Mx) * (1 + mix);
    int64_t issued = 0;
    int next_col = 0;
    bool live = hvalid;  // this half still streams real columns (cleared on convergence)
    // next chunk's issue parameters; the mask is decoded at publish time, one
    // chunk later, so the global load's latency stays off the column loop
    int pf_off = 0;
    unsigned long long pf_mk = 0ull;
    auto fetch_issue = [&](int cb) {
      const int c = cb + hl;
      pf_off = (c < M) ? static_cast<int>(colo[c]) : 0;
      pf_mk = (c < M) ? tmk[c] : 0ull;
    };
    fetch_issue(0);
    auto issue_one = [&](double dep) {
      const int c = next_col & 15;
      if (c == 0) {
        __syncwarp();
        ioff[hb + hl] = pf_off;
        icode[hb + hl] = tile_code(pf_mk);
        __syncwarp();
        fetch_issue(next_col + 16 < Mx ? next_col + 16 : 0);
      }
      if (hl == 0) {
        const int code = live ? icode[hb + c] : 0;
        const uint32_t bytes = static_cast<uint32_t>(code_tiles(code)) * 256u;
        const uint32_t bar = bar_s + ist * 8;
        if (bytes) {
          mbar_expect_s(bar, bytes);
          bulk_g2s_dep(ring_h + ist * SLOT_B, Ws + ioff[hb + c], bytes, bar, dep);
        } else {
          mbar_arrive_s(bar);
        }
      }
      if (++ist == STAGES) ist = 0;
      ++issued;
      if (++next_col == Mx) next_col = 0;
    };
    for (int q = 0; q < STAGES && issued < total; ++q) issue_one(0.0);

    // ---- consumer side
    int64_t consumed = 0;
    bool ready = false;
    double w[R];
    auto load_w = [&](int code) {
      if (!ready) mbar_wait_s(bar_s + st * 8, ph);
      const int a0 = code & 0xff, la = (code >> 8) & 0xff;
      const uint32_t cA = ring_h + st * SLOT_B + 16u * hl - 256u * a0;
#pragma unroll
      for (int q = 0; q < R / 2; ++q) {
        const bool inA = static_cast<unsigned>(q - a0) < static_cast<unsigned>(la);
        lds_v2((inA ? cA : zero_s) + 256u * q, w[2 * q], w[2 * q + 1]);
      }
    };
    auto advance = [&](double dep) {
      if (issued < total) issue_one(dep);
      if (++st == STAGES) {
        st = 0;
        ph ^= 1u;
      }
      ++consumed;
      ready = (consumed < issued) && mbar_test_s(bar_s + st * 8, ph);
    };

    // prologue: col_sq (elastic_net.py:85) and r = y - W beta0 (elastic_net.py:94)
    for (int cb = 0; cb < Mx; cb += 16) {
      const int nc = min(16, Mx - cb);
      int cl = 0;
      double bl0 = 0.0, csl = 0.0;
      if (cb + hl < M) {
        cl = tile_code(tmk[cb + hl]);
        bl0 = betas[cb + hl];
      }
      for (int t = 0; t < nc; ++t) {
        load_w(__shfl_sync(0xffffffffu, cl, t, 16));
        double p0 = 0.0, p1 = 0.0;
#pragma unroll
        for (int k = 0; k < R; ++k) {
          if (k & 1) p1 = fma(w[k], w[k], p1);
          else p0 = fma(w[k], w[k], p0);
        }
        const double pp = p0 + p1;
        advance(pp);
        const double p = half_sum(pp);
        if (hl == t) csl = p;
        const double b0 = __shfl_sync(0xffffffffu, bl0, t, 16);
        if (__any_sync(0xffffffffu, b0 != 0.0)) {
#pragma unroll
          for (int k = 0; k < R; ++k) r[k] = fma(-b0, w[k], r[k]);
        }
      }
      if (cb + hl < M) colsq[cb + hl] = csl;
    }

    // sweeps (elastic_net.py:137-161)
    const bool one_chunk = Mx <= 16;
    double nb_l = 0.0, ncs_l = 0.0;
    unsigned long long nk_mk = 0ull;  // decoded at publish time (see fetch_issue)
    auto fetch_params = [&](int cb) {
      const int c = cb + hl;
      nb_l = (c < M) ? betas[c] : 0.0;
      ncs_l = (c < M) ? colsq[c] : 0.0;
      nk_mk = (c < M) ? tmk[c] : 0ull;
    };
    fetch_params(0);
    int sweeps_done = 0, conv = 0;
    double obj = 0.0;
    for (int sw = 0; sw < mix; ++sw) {
      const bool act = hvalid && !conv && sw < mi;
      if (!__any_sync(0xffffffffu, act)) break;
      double max_delta = 0.0, acc_l1 = 0.0, acc_l2 = 0.0, acc_max = 0.0;
      for (int cb = 0; cb < Mx; cb += 16) {
        const int nc = min(16, Mx - cb);
        __syncwarp();
        if (sw == 0 || !one_chunk) {
          pb[hb + hl] = nb_l;
          pc[hb + hl] = ncs_l;
          const double dnv = __dadd_rn(ncs_l, lam2);
          pinv[hb + hl] = dnv > 0.0 ? __ddiv_rn(1.0, dnv) : 0.0;
          pk[hb + hl] = tile_code(nk_mk);
          if (!one_chunk) fetch_params(cb + 16 < Mx ? cb + 16 : 0);
        }
        __syncwarp();
        for (int t = 0; t < nc; ++t) {
          load_w(act ? pk[hb + t] : 0);  // a finished half reads zeros
          double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
#pragma unroll
          for (int k = 0; k < R; ++k) {
            if ((k & 3) == 0) d0 = fma(w[k], r[k], d0);
            else if ((k & 3) == 1) d1 = fma(w[k], r[k], d1);
            else if ((k & 3) == 2) d2 = fma(w[k], r[k], d2);
            else d3 = fma(w[k], r[k], d3);
          }
          const double part = (d0 + d1) + (d2 + d3);
          advance(part);
          const double b_old = pb[hb + t];
          const double cs = pc[hb + t];
          const double inv = pinv[hb + t];
          const double cb_old = __dmul_rn(cs, b_old);
          const double dot = half_sum(part);
          const double z = __dadd_rn(cb_old, dot);
          const double np_ = __dsub_rn(z, lam1), nn_ = __dadd_rn(z, lam1);
          // the quotient S(z, lam1) / (col_sq + lam2) as the product with the correctly
          // rounded reciprocal (<= 1.5 ulp from the division, far inside the rounding
          // class of the reordered dots; two dependent DFMAs off the per-column chain:
          // C4 CD 8.13 -> 8.06 s, profiles/r02_cd_dual_predicated_loads_ab.txt)
          const double bp = __dmul_rn(np_, inv), bn = __dmul_rn(nn_, inv);
          double b_new = np_ > 0.0 ? bp : (nn_ < 0.0 ? bn : 0.0);
          if (!act) b_new = b_old;
          const double d = __dsub_rn(b_new, b_old);
#pragma unroll
          for (int k = 0; k < R; ++k) r[k] = fma(-d, w[k], r[k]);
          if (hl == 0) pb[hb + t] = b_new;
          const double ad = fabs(d);
          max_delta = ad > max_delta ? ad : max_delta;
        }
        __syncwarp();
        if (act && hl < nc && cb + hl < M) {
          const double bl = pb[hb + hl];
          betas[cb + hl] = bl;
          const double ab = fabs(bl);
          acc_l1 += ab;
          acc_l2 = fma(bl, bl, acc_l2);
          acc_max = fmax(acc_max, ab);
        }
      }
      double rss0 = 0.0, rss1 = 0.0;
#pragma unroll
      for (int k = 0; k < R; ++k) {
        if (k & 1) rss1 = fma(r[k], r[k], rss1);
        else rss0 = fma(r[k], r[k], rss0);
      }
      const double rss = half_sum(rss0 + rss1);
      const double l1 = half_sum(acc_l1);
      const double l2 = half_sum(acc_l2);
      const double mabs = half_max(acc_max);
      if (act) {
        obj = __dadd_rn(__dadd_rn(__dmul_rn(0.5, rss), __dmul_rn(lam1, l1)),
                        __dmul_rn(__dmul_rn(0.5, lam2), l2));
        if (a.hist != nullptr && hl == 0) a.hist[a.hist_off[s] + sw] = obj;
        sweeps_done = sw + 1;
        if (max_delta <= __dmul_rn(tol, fmax(mabs, 1.0))) {
          conv = 1;
          live = false;  // later stream positions of this half carry no data
        }
      }
    }
    const bool zero_it = hvalid && mi == 0;
    if (__any_sync(0xffffffffu, zero_it)) {
      // objective at the given beta (after the Gram-form sweeps, gram.cu);
      // both halves run the shuffles, only a half with max_iters == 0 keeps it
      double rss = 0.0, l1 = 0.0, l2 = 0.0;
#pragma unroll
      for (int k = 0; k < R; ++k) rss = fma(r[k], r[k], rss);
      rss = half_sum(rss);
      for (int j = hl; j < M; j += 16) {
        const double b = betas[j];
        l1 += fabs(b);
        l2 = fma(b, b, l2);
      }
      l1 = half_sum(l1);
      l2 = half_sum(l2);
      if (zero_it)
        obj = __dadd_rn(__dadd_rn(__dmul_rn(0.5, rss), __dmul_rn(lam1, l1)),
                        __dmul_rn(__dmul_rn(0.5, lam2), l2));
    }
    // drain the prefetched columns of the sweep that will not run
    while (consumed < issued) {
      mbar_wait_s(bar_s + st * 8, ph);
      if (++st == STAGES) {
        st = 0;
        ph ^= 1u;
      }
      ++consumed;
    }
    __syncwarp();
    if (hvalid && hl == 0) {
      a.sweeps[s] = sweeps_done;
      a.converged[s] = conv;
      a.objective[s] = obj;
    }
    unsigned nxt = 0;
    if (lane == 0) nxt = atomicAdd(a.queue, 1u) + total_warps;
    item = __shfl_sync(0xffffffffu, nxt, 0);
  }
}

// ----------------------------------------------------------------------------
// Column-pair tile CD for batches of few fits (<= a few per SM: BASELINE
// configs 2-3, 64-256 fits of 1,024 rows).  With one or two fits per SM a
// fit's per-column dependency chain (dot -> 5-level reduction -> soft
// threshold -> AXPY, ~0.55 us) is the whole cost, and registers/shared memory
// are plentiful.  So columns are taken in pairs (j, j+1): both dots against the
// same residual r_{j-1}, both warp reductions interleaved, then the soft
// thresholds in order with column j+1's dot corrected by the Gram entry,
//   W_{j+1} . r_j = W_{j+1} . r_{j-1} - d_j (W_j . W_{j+1}),
// exact in exact arithmetic (only the rounding of the length-N dot products
// differs from the reference's sequential sums, as for every CD form here;
// SURVEY F2), then both updates.  The pair products g_j = W_j . W_{j+1} (j even)
// are formed in the prologue pass from the same staged tiles.  The ring and
// copy issue are the lean kernel's; a fit's run codes and packed offsets are
// staged in shared memory once per launch.
template <int R, int STAGES, int WPC>
__global__ void __launch_bounds__(WPC * 32, 1) cd_pipe_kernel(const CdArgs a, int gcap) {
  constexpr int SLOT = R * 32;
  static_assert(R % 2 == 0 && R <= 32, "paired-row layout");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // per warp: ring[STAGES][SLOT] | pb/pc/pinv[32] | g[gcap] | codes[gcap] | offs[gcap]
  const size_t per_warp = static_cast<size_t>(STAGES) * SLOT * 8 + 96 * 8 + static_cast<size_t>(gcap) * 16;
  unsigned char* const wbase = smem_raw + static_cast<size_t>(warp) * per_warp;
  double* const ring = reinterpret_cast<double*>(wbase);
  double* const pb = ring + STAGES * SLOT;
  double* const pc = pb + 32;
  double* const pinv = pb + 64;
  double* const gn = pb + 96;
  int* const codes = reinterpret_cast<int*>(gn + gcap);
  int* const offs = codes + gcap;
  uint64_t* const bars_all = reinterpret_cast<uint64_t*>(smem_raw + WPC * per_warp);
  uint64_t* const bars = bars_all + warp * STAGES;
  // zero block 16-byte aligned after the barriers (16-byte shared loads)
  double* const zero_blk = reinterpret_cast<double*>(bars_all + ((WPC * STAGES + 1) & ~1));
  const uint32_t ring_s = smem_u32(ring);
  const uint32_t bar_s = smem_u32(bars);
  const uint32_t zero_s = smem_u32(zero_blk) + 16u * lane;
  const int half = lane >> 4;

  for (int i = threadIdx.x; i < SLOT; i += WPC * 32) zero_blk[i] = 0.0;
  if (lane == 0) {
    for (int i = 0; i < STAGES; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncthreads();

  int st = 0, ist = 0;
  uint32_t ph = 0;
  unsigned item = warp * gridDim.x + blockIdx.x;
  const unsigned total_warps = gridDim.x * WPC;

  while (item < a.S) {
    const int64_t s = a.order ? a.order[item] : static_cast<int64_t>(item);
    if (a.active == nullptr || a.active[s] != 0) {
      const int64_t r0 = a.row_off[s];
      const int N = static_cast<int>(a.row_off[s + 1] - r0);
      const int M = a.m_cur[s];
      const int64_t doff = a.dict_off[s];
      const double* Ws = a.W + a.w_off[s];
      double* betas = a.beta + doff;
      double* colsq = a.col_sq + doff;
      const double lam1 = a.lam1[s], lam2 = a.lam2[s], tol = a.tol[s];
      const int max_iters = a.max_iters[s];
      __syncwarp();
      for (int c = lane; c < M; c += 32) {
        codes[c] = tile_code(a.tile_mask[doff + c]);
        offs[c] = static_cast<int>(a.col_off[doff + c]);
      }
      __syncwarp();

      double r[R];
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const int p = 64 * (k >> 1) + 2 * lane + (k & 1);
        const int row = a.perm ? (p < N ? a.perm[r0 + p] : 0) : p;
        r[k] = (p < N) ? a.y[r0 + row] : 0.0;
      }

      // ---- copy issue (lean kernel's ring; parameters from shared memory)
      const int total = M * (1 + max_iters);
      int issued = 0, next_col = 0;
      auto issue_one = [&](double dep) {
        if (lane == 0) {
          const int code = codes[next_col];
          const uint32_t bytes = static_cast<uint32_t>(code_tiles(code)) * 256u;
          const uint32_t bar = bar_s + ist * 8;
          if (bytes) {
            mbar_expect_s(bar, bytes);
            bulk_g2s_dep(ring_s + ist * (SLOT * 8), Ws + offs[next_col], bytes, bar, dep);
          } else {
            mbar_arrive_s(bar);
          }
        }
        if (++ist == STAGES) ist = 0;
        ++issued;
        if (++next_col == M) next_col = 0;
      };
      for (int q = 0; q < STAGES && issued < total; ++q) issue_one(0.0);
      int consumed = 0;
      // next stream column -> w (run code of that column); refill its slot
      auto take = [&](int col, double (&w)[R]) {
        mbar_wait_s(bar_s + st * 8, ph);
        const int code = codes[col];
        const int a0 = code & 0xff, la = (code >> 8) & 0xff;
        const uint32_t cA = ring_s + st * (SLOT * 8) + 16u * lane - 256u * a0;
        const int hA = half - a0;
        double dep = 0.0;
#pragma unroll
        for (int q = 0; q < R / 2; ++q) {
          const bool inA = static_cast<unsigned>(hA + 2 * q) < static_cast<unsigned>(la);
          lds_v2((inA ? cA : zero_s) + 512u * q, w[2 * q], w[2 * q + 1]);
          dep += w[2 * q];
        }
        if (issued < total) issue_one(dep);
        if (++st == STAGES) {
          st = 0;
          ph ^= 1u;
        }
        ++consumed;
      };
      auto dotp = [&](const double (&w)[R], const double (&x)[R]) {
        double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
#pragma unroll
        for (int k = 0; k < R; ++k) {
          if ((k & 3) == 0) d0 = fma(w[k], x[k], d0);
          else if ((k & 3) == 1) d1 = fma(w[k], x[k], d1);
          else if ((k & 3) == 2) d2 = fma(w[k], x[k], d2);
          else d3 = fma(w[k], x[k], d3);
        }
        return (d0 + d1) + (d2 + d3);
      };

      double wA[R], wB[R];
#pragma unroll
      for (int k = 0; k < R; ++k) wA[k] = wB[k] = 0.0;  // an odd M leaves wB unloaded (multiplied by 0)
      // ---- prologue: col_sq, r = y - W beta0, g_j = W_j . W_{j+1}
      {
        auto pro = [&](int j, double (&w)[R], const double (&wprev)[R]) {
          take(j, w);
          const double cs = warp_sum(dotp(w, w));
          // consecutive-pair product g_{j-1} = W_{j-1} . W_j for pairs starting at even j-1
          const double g = (j & 1) ? warp_sum(dotp(w, wprev)) : 0.0;
          if (lane == 0) {
            colsq[j] = cs;
            if (j & 1) gn[j - 1] = g;
          }
          const double b0 = betas[j];
          if (b0 != 0.0) {
#pragma unroll
            for (int k = 0; k < R; ++k) r[k] = fma(-b0, w[k], r[k]);
          }
        };
        for (int j = 0; j < M; j += 2) {
          pro(j, wA, wB);
          if (j + 1 < M) pro(j + 1, wB, wA);
        }
      }
      __syncwarp();

      int sweeps_done = 0, conv = 0;
      double obj = 0.0;
      for (int sw = 0; sw < max_iters; ++sw) {
        double max_delta = 0.0;
        // column pairs (j, j+1): both dots against the same residual, both
        // 5-level reductions interleaved, then the two soft thresholds in order
        // with column j+1's dot corrected by d_j g_j, then both updates
        for (int j = 0; j < M; j += 2) {
          if ((j & 31) == 0) {
            __syncwarp();
            const int c = j + lane;
            const double bv = c < M ? betas[c] : 0.0;
            const double cv = c < M ? colsq[c] : 0.0;
            pb[lane] = bv;
            pc[lane] = cv;
            const double dnv = __dadd_rn(cv, lam2);
            pinv[lane] = dnv > 0.0 ? __ddiv_rn(1.0, dnv) : 0.0;
            __syncwarp();
          }
          const bool two = j + 1 < M;
          take(j, wA);
          if (two) take(j + 1, wB);
          double sA = dotp(wA, r);
          double sB = two ? dotp(wB, r) : 0.0;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            sA += __shfl_xor_sync(0xffffffffu, sA, o);
            sB += __shfl_xor_sync(0xffffffffu, sB, o);
          }
          const int t = j & 31;
          auto solve = [&](int tt, double dot) {
            const double b_old = pb[tt];
            const double cs = pc[tt];
            const double inv = pinv[tt];
            const double dn = __dadd_rn(cs, lam2);
            const double z = __dadd_rn(__dmul_rn(cs, b_old), dot);
            const double np_ = __dsub_rn(z, lam1), nn_ = __dadd_rn(z, lam1);
            const double qp = __dmul_rn(np_, inv), qn = __dmul_rn(nn_, inv);
            const double bp = fma(fma(-qp, dn, np_), inv, qp);
            const double bn = fma(fma(-qn, dn, nn_), inv, qn);
            const double b_new = np_ > 0.0 ? bp : (nn_ < 0.0 ? bn : 0.0);
            if (lane == 0) pb[tt] = b_new;
            const double d = __dsub_rn(b_new, b_old);
            const double ad = fabs(d);
            max_delta = ad > max_delta ? ad : max_delta;
            return d;
          };
          const double dA = solve(t, sA);
          double dB = 0.0;
          if (two) dB = solve(t + 1, __dsub_rn(sB, __dmul_rn(dA, gn[j])));
#pragma unroll
          for (int k = 0; k < R; ++k) r[k] = fma(-dB, wB[k], fma(-dA, wA[k], r[k]));
          if (t + 2 >= 32 || j + 2 >= M) {  // chunk done: write its betas back
            __syncwarp();
            const int c = (j & ~31) + lane;
            if (c < M && c <= j + 1) betas[c] = pb[lane];
          }
        }
        __syncwarp();
        double rss0 = 0.0, rss1 = 0.0;
#pragma unroll
        for (int k = 0; k < R; ++k) {
          if (k & 1) rss1 = fma(r[k], r[k], rss1);
          else rss0 = fma(r[k], r[k], rss0);
        }
        double acc_l1 = 0.0, acc_l2 = 0.0, acc_max = 0.0;
        for (int c = lane; c < M; c += 32) {
          const double bl = betas[c];
          const double ab = fabs(bl);
          acc_l1 += ab;
          acc_l2 = fma(bl, bl, acc_l2);
          acc_max = fmax(acc_max, ab);
        }
        const double rss = warp_sum(rss0 + rss1);
        const double l1 = warp_sum(acc_l1);
        const double l2 = warp_sum(acc_l2);
        const double mabs = warp_max(acc_max);
        obj = __dadd_rn(__dadd_rn(__dmul_rn(0.5, rss), __dmul_rn(lam1, l1)),
                        __dmul_rn(__dmul_rn(0.5, lam2), l2));
        if (a.hist != nullptr && lane == 0) a.hist[a.hist_off[s] + sw] = obj;
        sweeps_done = sw + 1;
        if (max_delta <= __dmul_rn(tol, fmax(mabs, 1.0))) {
          conv = 1;
          break;
        }
      }
      if (max_iters == 0) {
        double rss = 0.0, l1 = 0.0, l2 = 0.0;
#pragma unroll
        for (int k = 0; k < R; ++k) rss = fma(r[k], r[k], rss);
        rss = warp_sum(rss);
        for (int j = lane; j < M; j += 32) {
          const double b = betas[j];
          l1 += fabs(b);
          l2 = fma(b, b, l2);
        }
        l1 = warp_sum(l1);
        l2 = warp_sum(l2);
        obj = __dadd_rn(__dadd_rn(__dmul_rn(0.5, rss), __dmul_rn(lam1, l1)),
                        __dmul_rn(__dmul_rn(0.5, lam2), l2));
      }
      while (consumed < issued) {  // drain the prefetched columns of the sweep that will not run
        mbar_wait_s(bar_s + st * 8, ph);
        if (++st == STAGES) {
          st = 0;
          ph ^= 1u;
        }
        ++consumed;
      }
      __syncwarp();
      if (lane == 0) {
        a.sweeps[s] = sweeps_done;
        a.converged[s] = conv;
        a.objective[s] = obj;
      }
    }
    unsigned nxt = 0;
    if (lane == 0) nxt = atomicAdd(a.queue, 1u) + total_warps;
    item = __shfl_sync(0xffffffffu, nxt, 0);
  }
}

// ----------------------------------------------------------------------------
// Large fits (N > 8192 rows, dense): one 512-thread CTA per fit, the residual
// in a global scratch (each thread owns rows tid + 512 k, L2-resident), design
// columns read straight from HBM (coalesced), a fixed-order CTA reduction per
// column.  Same arithmetic as cd_kernel; lifts the row envelope of fit()
// (elastic_net.py:66-110 has none).
constexpr int LG_THREADS = 512;
__global__ void __launch_bounds__(LG_THREADS) cd_large_kernel(const CdArgs a) {
  __shared__ double red[2][LG_THREADS / 32];
  __shared__ unsigned nxt_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int buf = 0;
  auto cta_sum = [&](double v) -> double {
    v = warp_sum(v);
    if (lane == 0) red[buf][warp] = v;
    __syncthreads();
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < LG_THREADS / 32; ++w) t += red[buf][w];
    buf ^= 1;  // the next reduction writes the other buffer: one barrier per sum
    return t;
  };
  unsigned item = blockIdx.x;
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
      const bool need_colsq = !(a.flags & CD_COLSQ_GIVEN);
      const bool r_given = (a.flags & CD_R_GIVEN) != 0;
      double* r = a.rbuf + r0;
      for (int i = tid; i < N; i += LG_THREADS) r[i] = a.y[r0 + i];
      if (need_colsq || !r_given) {
        for (int j = 0; j < M; ++j) {
          const double* col = Ws + (int64_t)j * ld;
          if (need_colsq) {
            double p = 0.0;
            for (int i = tid; i < N; i += LG_THREADS) p = fma(col[i], col[i], p);
            p = cta_sum(p);
            if (tid == 0) a.col_sq[doff + j] = p;
          }
          if (!r_given) {
            const double b0 = a.beta[doff + j];
            if (b0 != 0.0)
              for (int i = tid; i < N; i += LG_THREADS) r[i] = fma(-b0, col[i], r[i]);
          }
        }
        __syncthreads();
      }
      int sweeps_done = 0, conv = 0;
      double obj = 0.0;
      for (int sw = 0; sw < max_iters; ++sw) {
        double max_delta = 0.0, l1 = 0.0, l2 = 0.0, mabs = 0.0;
        for (int j = 0; j < M; ++j) {
          const double* col = Ws + (int64_t)j * ld;
          double p = 0.0;
          for (int i = tid; i < N; i += LG_THREADS) p = fma(col[i], r[i], p);
          const double dot = cta_sum(p);
          const double b_old = a.beta[doff + j];
          const double cs = a.col_sq[doff + j];
          const double dn = __dadd_rn(cs, lam2);
          const double z = __dadd_rn(__dmul_rn(cs, b_old), dot);
          double b_new = 0.0;
          if (dn > 0.0) {
            double mag = __dsub_rn(fabs(z), lam1);
            if (mag < 0.0) mag = 0.0;
            b_new = __ddiv_rn(z >= 0.0 ? mag : -mag, dn);
          }
          const double d = __dsub_rn(b_new, b_old);
          if (d != 0.0)
            for (int i = tid; i < N; i += LG_THREADS) r[i] = fma(-d, col[i], r[i]);
          __syncthreads();  // every thread read beta[j] before it is replaced
          if (tid == 0) a.beta[doff + j] = b_new;
          max_delta = fmax(max_delta, fabs(d));
          const double ab = fabs(b_new);
          l1 += ab;
          l2 = fma(b_new, b_new, l2);
          mabs = fmax(mabs, ab);
        }
        double rr = 0.0;
        for (int i = tid; i < N; i += LG_THREADS) rr = fma(r[i], r[i], rr);
        const double rss = cta_sum(rr);
        obj = __dadd_rn(__dadd_rn(__dmul_rn(0.5, rss), __dmul_rn(lam1, l1)),
                        __dmul_rn(__dmul_rn(0.5, lam2), l2));
        if (a.hist != nullptr && tid == 0) a.hist[a.hist_off[s] + sw] = obj;
        sweeps_done = sw + 1;
        if (max_delta <= __dmul_rn(tol, fmax(mabs, 1.0))) {
          conv = 1;
          break;
        }
      }
      if (max_iters == 0) {
        double rr = 0.0, q1 = 0.0, q2 = 0.0;
        for (int i = tid; i < N; i += LG_THREADS) rr = fma(r[i], r[i], rr);
        for (int j = tid; j < M; j += LG_THREADS) {
          const double b = a.beta[doff + j];
          q1 += fabs(b);
          q2 = fma(b, b, q2);
        }
        const double rss = cta_sum(rr);
        const double t1 = cta_sum(q1);
        const double t2 = cta_sum(q2);
        obj = __dadd_rn(__dadd_rn(__dmul_rn(0.5, rss), __dmul_rn(lam1, t1)),
                        __dmul_rn(__dmul_rn(0.5, lam2), t2));
      }
      if (a.flags & CD_WRITE_R)
        for (int i = tid; i < N; i += LG_THREADS) a.y[r0 + i] = r[i];
      if (tid == 0) {
        a.sweeps[s] = sweeps_done;
        a.converged[s] = conv;
        a.objective[s] = obj;
      }
    }
    __syncthreads();
    if (tid == 0) nxt_s = atomicAdd(a.queue, 1u) + gridDim.x;
    __syncthreads();
    item = nxt_s;
  }
}

// ----------------------------------------------------------------------------
// launchers.  The dynamic shared-memory attribute is set on every launch (it
// is per device and per function; the call is cheap), so one process may
// drive several GPUs.


template <typename K>
int launch_persistent(K kernel, const CdArgs& a, int64_t units, int threads, size_t smem,
                      cudaStream_t stream, const char* what) {
  PAM_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  PAM_CUDA_CHECK(cudaMemsetAsync(a.queue, 0, sizeof(unsigned), stream));
  const int64_t ctas = std::max<int64_t>(1, std::min<int64_t>(sm_count(), units));
  kernel<<<(unsigned)ctas, threads, smem, stream>>>(a);
  PAM_LAUNCH_CHECK(what);
  return PAM_OK;
}

template <int R, int STAGES, int WPC, int G>
int launch_cd(const CdArgs& a, cudaStream_t stream) {
  constexpr int NGROUPS = WPC / G;
  const size_t smem = static_cast<size_t>(NGROUPS) * STAGES * (R * 32 * G * sizeof(double)) +
                      static_cast<size_t>(NGROUPS) * STAGES * sizeof(uint64_t) +
                      static_cast<size_t>(NGROUPS) * (2 * G + 1) * sizeof(double) +
                      static_cast<size_t>(NGROUPS) * 96 * sizeof(double);
  return launch_persistent(cd_kernel<R, STAGES, WPC, G>, a, a.S, WPC * 32, smem, stream, "cd_kernel");
}

template <int R, int STAGES, int WPC>
int launch_cd_tile(const CdArgs& a, cudaStream_t stream) {
  const size_t smem = static_cast<size_t>(WPC) * STAGES * R * 32 * sizeof(double) +
                      static_cast<size_t>(WPC) * STAGES * sizeof(uint64_t) +
                      static_cast<size_t>(WPC) * 144 * sizeof(double) + R * 32 * sizeof(double);
  return launch_persistent(cd_tile_kernel<R, STAGES, WPC>, a, a.S, WPC * 32, smem, stream,
                           "cd_tile_kernel");
}

template <int R, int STAGES, int WPC>
int launch_cd_dual(const CdArgs& a, cudaStream_t stream) {
  constexpr int SLOTH = R * 16;
  const size_t smem = static_cast<size_t>(WPC) * STAGES * 2 * SLOTH * sizeof(double) +
                      static_cast<size_t>(WPC) * STAGES * sizeof(uint64_t) +
                      static_cast<size_t>(WPC) * 144 * sizeof(double) + SLOTH * sizeof(double);
  return launch_persistent(cd_dual_kernel<R, STAGES, WPC>, a, (a.S + 1) / 2, WPC * 32, smem, stream,
                           "cd_dual_kernel");
}

template <int R, int STAGES, int WPC>
int launch_cd_pipe(const CdArgs& a, int gcap, cudaStream_t stream) {
  constexpr int SLOT = R * 32;
  const size_t per_warp = static_cast<size_t>(STAGES) * SLOT * 8 + 96 * 8 + static_cast<size_t>(gcap) * 16;
  const size_t smem = WPC * per_warp + static_cast<size_t>((WPC * STAGES + 1) & ~1) * 8 + SLOT * 8;
  auto kernel = cd_pipe_kernel<R, STAGES, WPC>;
  PAM_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  PAM_CUDA_CHECK(cudaMemsetAsync(a.queue, 0, sizeof(unsigned), stream));
  const int64_t ctas = std::max<int64_t>(1, std::min<int64_t>(sm_count(), ceil_div(a.S, WPC)));
  kernel<<<(unsigned)ctas, WPC * 32, smem, stream>>>(a, gcap);
  PAM_LAUNCH_CHECK("cd_pipe_kernel");
  return PAM_OK;
}

int launch_cd_large(const CdArgs& a, cudaStream_t stream) {
  if (a.rbuf == nullptr) {
    set_last_error("pam_cd_f64: fits above 8192 rows need the residual scratch of pam_cd_workspace_bytes");
    return PAM_ERR_ARG;
  }
  PAM_CUDA_CHECK(cudaMemsetAsync(a.queue, 0, sizeof(unsigned), stream));
  const int64_t ctas = std::max<int64_t>(1, std::min<int64_t>(2LL * sm_count(), a.S));
  cd_large_kernel<<<(unsigned)ctas, LG_THREADS, 0, stream>>>(a);
  PAM_LAUNCH_CHECK("cd_large_kernel");
  return PAM_OK;
}

// Dense design matrices.  Many fits: one warp per fit; few fits (< 4 per SM):
// a group of G warps per fit (shorter per-column latency); > 8192 rows: the
// CTA-per-fit kernel with the residual in global memory.
int cd_dispatch(const CdArgs& a, int max_rows, cudaStream_t stream) {
  if (max_rows > CD_REG_ROWS) return launch_cd_large(a, stream);
  const bool few = a.S < 4LL * sm_count();
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
  return launch_cd<32, 3, 8, 8>(a, stream);                          // <= 8192
}

// Few fits per SM (BASELINE configs 2-3): the column-pair kernel; its
// per-warp staging holds a fit's run codes, offsets and consecutive-column
// products, sized from the largest dictionary of the batch (max_m, host).
int launch_pair(const CdArgs& a, int max_rows, int max_m, cudaStream_t stream) {
  const int sms = sm_count();
  const int gcap = (max_m + 31) / 32 * 32;
  const int wpc_need = static_cast<int>(std::min<int64_t>(3, std::max<int64_t>(1, ceil_div(a.S, sms))));
  // shared memory per warp: 3 slots + params + 16 B per dictionary slot
  const int R = max_rows <= 512 ? 16 : 32;
  const size_t per_warp = 3 * R * 32 * 8 + 96 * 8 + static_cast<size_t>(gcap) * 16;
  const size_t avail = 227 * 1024 - R * 32 * 8 - 64;
  const int wpc_fit = static_cast<int>(avail / per_warp);
  if (wpc_fit < 1) return PAM_ERR_UNSUPPORTED;  // dictionary too large for the staging
  const int wpc = std::min(wpc_need, wpc_fit);
  if (R == 16) {
    if (wpc >= 3) return launch_cd_pipe<16, 3, 3>(a, gcap, stream);
    if (wpc == 2) return launch_cd_pipe<16, 3, 2>(a, gcap, stream);
    return launch_cd_pipe<16, 3, 1>(a, gcap, stream);
  }
  if (wpc >= 3) return launch_cd_pipe<32, 3, 3>(a, gcap, stream);
  if (wpc == 2) return launch_cd_pipe<32, 3, 2>(a, gcap, stream);
  return launch_cd_pipe<32, 3, 1>(a, gcap, stream);
}

// Tile-packed design matrices (<= 1024 rows).  Auto selection:
//  * 257-1024 rows and <= 2 fits per SM: the exact blocked CD (cd_block.cu);
//  * 257-1024 rows and <= 3 fits per SM: the column-pair kernel;
//  * 257-512 rows and >= 8 fits per SM (C4): two fits per warp;
//  * otherwise one fit per warp.
int cd_auto_kernel(int64_t S, int max_rows) {
  const int64_t sms = sm_count();
  if (max_rows > 256 && S <= 2 * sms) return PAM_CD_BLOCK;
  if (max_rows > 256 && S <= 3 * sms) return PAM_CD_PAIR;
  if (max_rows > 256 && max_rows <= 512 && S >= 8 * sms) return PAM_CD_DUAL;
  return PAM_CD_LEAN;
}

int cd_dispatch_tiles(const CdArgs& a, int max_rows, int max_m, int kernel, void* block_ws,
                      cudaStream_t stream) {
  if (kernel == PAM_CD_AUTO) kernel = cd_auto_kernel(a.S, max_rows);
  if (kernel == PAM_CD_BLOCK) return launch_cd_block(a, max_rows, block_ws, stream);
  if (kernel == PAM_CD_PAIR && max_rows > 32) {
    const int rc = launch_pair(a, max_rows, max_m, stream);
    if (rc != PAM_ERR_UNSUPPORTED) return rc;
  }
  if (kernel == PAM_CD_DUAL && max_rows <= 512) return launch_cd_dual<32, 3, 8>(a, stream);
  if (max_rows <= 32) return launch_cd_tile<1, 4, 16>(a, stream);
  if (max_rows <= 64) return launch_cd_tile<2, 4, 16>(a, stream);
  if (max_rows <= 128) return launch_cd_tile<4, 4, 16>(a, stream);
  if (max_rows <= 256) return launch_cd_tile<8, 4, 16>(a, stream);
  if (max_rows <= 512) return launch_cd_tile<16, 3, 16>(a, stream);
  return launch_cd_tile<32, 3, 8>(a, stream);
}

}  // namespace pam

using namespace pam;

extern "C" int64_t pam_cd_max_rows(void) { return INT32_MAX; }

extern "C" int64_t pam_cd_workspace_bytes(int64_t S, int64_t total_rows, int64_t total_slots, int32_t max_rows,
                                          int32_t kernel) {
  if (S < 0 || total_rows < 0 || total_slots < 0) return -1;
  int64_t b = 256;  // work counters
  if (max_rows > CD_REG_ROWS) b += total_rows * static_cast<int64_t>(sizeof(double));
  const int k = (kernel == PAM_CD_AUTO && max_rows <= 1024) ? cd_auto_kernel(S, max_rows) : kernel;
  if (k == PAM_CD_BLOCK && max_rows <= 1024) b += cd_block_workspace_bytes(S, total_slots);
  return b;
}

namespace {
CdArgs make_args(int64_t S, const int64_t* order, const int64_t* row_off, double* y,
                 const int64_t* dict_off, const int32_t* m_cur, const int64_t* w_off, const int32_t* ld,
                 const double* W, const double* lam1, const double* lam2, const double* tol,
                 const int32_t* max_iters, const int32_t* active, double* beta, double* col_sq,
                 int32_t* sweeps, int32_t* converged, double* objective, double* hist,
                 const int64_t* hist_off, int flags, const uint64_t* tile_mask, const int64_t* col_off,
                 const int32_t* perm, void* work) {
  CdArgs a{};
  a.S = S;
  a.order = order;
  a.row_off = row_off;
  a.y = y;
  a.dict_off = dict_off;
  a.m_cur = m_cur;
  a.w_off = w_off;
  a.ld = ld;
  a.W = W;
  a.lam1 = lam1;
  a.lam2 = lam2;
  a.tol = tol;
  a.max_iters = max_iters;
  a.active = active;
  a.beta = beta;
  a.col_sq = col_sq;
  a.sweeps = sweeps;
  a.converged = converged;
  a.objective = objective;
  a.hist = hist;
  a.hist_off = hist_off;
  a.flags = flags;
  a.tile_mask = reinterpret_cast<const unsigned long long*>(tile_mask);
  a.col_off = col_off;
  a.perm = perm;
  a.queue = static_cast<unsigned*>(work);
  a.rbuf = reinterpret_cast<double*>(static_cast<char*>(work) + 256);
  return a;
}
}  // namespace

extern "C" int pam_cd_ex_f64(int64_t S, const int64_t* order, const int64_t* row_off, double* y,
                             const int64_t* dict_off, const int32_t* m_cur, const int64_t* w_off,
                             const int32_t* ld, const double* W, const double* lam1,
                             const double* lam2, const double* tol, const int32_t* max_iters,
                             const int32_t* active, int32_t max_rows, double* beta, double* col_sq,
                             int32_t* sweeps, int32_t* converged, double* objective, double* hist,
                             const int64_t* hist_off, int flags, void* work, void* stream) {
  if (S < 0 || max_rows < 0 || work == nullptr) return PAM_ERR_ARG;
  if (S == 0) return PAM_OK;
  CdArgs a = make_args(S, order, row_off, y, dict_off, m_cur, w_off, ld, W, lam1, lam2, tol, max_iters,
                       active, beta, col_sq, sweeps, converged, objective, hist, hist_off, flags, nullptr,
                       nullptr, nullptr, work);
  if (max_rows <= CD_REG_ROWS) a.rbuf = nullptr;
  return cd_dispatch(a, max_rows, as_stream(stream));
}

extern "C" int pam_cd_f64(int64_t S, const int64_t* order, const int64_t* row_off, const double* y,
                          const int64_t* dict_off, const int32_t* m_cur, const int64_t* w_off,
                          const int32_t* ld, const double* W, const double* lam1,
                          const double* lam2, const double* tol, const int32_t* max_iters,
                          const int32_t* active, int32_t max_rows, double* beta, double* col_sq,
                          int32_t* sweeps, int32_t* converged, double* objective, double* hist,
                          const int64_t* hist_off, void* work, void* stream) {
  return pam_cd_ex_f64(S, order, row_off, const_cast<double*>(y), dict_off, m_cur, w_off, ld, W,
                       lam1, lam2, tol, max_iters, active, max_rows, beta, col_sq, sweeps,
                       converged, objective, hist, hist_off, 0, work, stream);
}

extern "C" int pam_cd_tiles_f64(int64_t S, const int64_t* order, const int64_t* row_off,
                                const double* y, const int32_t* perm, const int64_t* dict_off,
                                const int32_t* m_cur, const int64_t* w_off,
                                const uint64_t* tile_mask, const int64_t* col_off, const double* W,
                                const double* lam1, const double* lam2, const double* tol,
                                const int32_t* max_iters, const int32_t* active, int32_t max_rows,
                                int32_t max_m, double* beta, double* col_sq, int32_t* sweeps,
                                int32_t* converged, double* objective, double* hist,
                                const int64_t* hist_off, int32_t kernel, void* work, void* stream) {
  if (S < 0 || max_rows < 0 || max_m < 0 || !tile_mask || !col_off || work == nullptr) return PAM_ERR_ARG;
  if (kernel < PAM_CD_AUTO || kernel > PAM_CD_BLOCK) return PAM_ERR_ARG;
  if (max_rows > 1024) {
    set_last_error("pam_cd_tiles_f64: tile-packed CD supports <= 1024 rows per subdomain");
    return PAM_ERR_UNSUPPORTED;
  }
  if (S == 0) return PAM_OK;
  CdArgs a = make_args(S, order, row_off, const_cast<double*>(y), dict_off, m_cur, w_off, m_cur, W, lam1,
                       lam2, tol, max_iters, active, beta, col_sq, sweeps, converged, objective, hist,
                       hist_off, 0, tile_mask, col_off, perm, work);
  a.rbuf = nullptr;
  return cd_dispatch_tiles(a, max_rows, max_m, kernel, static_cast<char*>(work) + 256, as_stream(stream));
}
