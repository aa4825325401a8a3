// cd_block.cu — exact blocked cyclic CD for batches of FEW fits (<= 2 per SM,
// BASELINE configs 2-3 and the paper's Table-2 run: 1-256 fits of 1,024 rows,
// up to 2,860 columns), software-pipelined with a dedicated solver warp.
//
// Reference loop (elastic_net.py:114-161): for j = 0..M-1 in order,
//   z_j = col_sq_j beta_j + W_j . r,  b = S(z_j, lam1) / (col_sq_j + lam2),
//   r -= (b - beta_j) W_j.
// With one or two fits per SM the per-column chain of the one-warp kernels
// (dot -> warp reduction -> soft threshold -> AXPY, ~0.55 us per column,
// profiles/r01_ncu_cd_pair_c2_raw.csv: FP64 pipe 4 %, DRAM 0.05 of peak) IS
// the runtime.  Columns are therefore taken in blocks (<= 16 columns whose
// packed tiles fit a shared-memory slot) and a CTA per fit works on three blocks
// at once:
//
//   workers (8 warps), step t:  r -= W_{t-1} d_{t-1};  zpart_{t+1} = W_{t+1}^T r
//   solver  (1 warp),  step t:  z_t = sum zpart_t - G[t, t-1] d_{t-1};  in-block
//                               cyclic updates of block t -> d_t
//   stream  (1 warp),  step t:  block t+2's column parameters and per-worker column
//                               lists; the bulk copy of block t+3 after the barrier
//
// zpart_{t+1} is formed against the residual BEFORE block t's updates; the
// missing term is exactly -G[t+1, t] d_t (G = W^T W restricted to the two
// blocks), accumulated by the solver inside step t's update loop -- the same
// identity as the in-block corrections, now across the block boundary, so the
// update sequence is still the reference's cyclic order j = 0..M-1, sweep
// after sweep (elastic_net.py:137-161); only the rounding of the inner
// products (and of the quotient, see the solver loop) differs, ~1e-12, the
// SURVEY F2 class.  The stream of blocks is continuous across sweeps (block 0
// of sweep k+1 follows block nblk-1 of sweep k, with G[0, nblk-1]).  The
// diagonal and the previous-block Gram blocks are computed once per round in
// the prologue pass and streamed with the block.  One CTA barrier per step.
//
// Round-2 session-4 structure (profiles/r02_cd_block_ab_s4.txt: C2 4.08 -> 3.0 s,
// C3 12.4 -> 8.8 s, Table-2 6.0 -> 4.35 s):
//  * workers are ROW parallel in both phases: a thread keeps its 4 residual rows
//    in registers, so the dots need no residual mirror in shared memory (the
//    block's tiles are the only shared-memory traffic, read once for the dots
//    and once for the AXPY; the column-parallel dots re-read the residual and
//    were shared-memory-bandwidth bound) and no barrier between AXPY and dots;
//    a warp's 16 partial sums go through a halving butterfly;
//  * the stream warp builds, per worker warp, the list of the block's columns
//    whose tile run meets that warp's rows: dots and AXPY visit only those;
//  * the solver's serial chain per column is one FMA, the shift by lam1, one
//    multiply by 1 / (col_sq + lam2) and the sign selects (the next column's value
//    is broadcast two steps early and corrected through G[k][k-1], G[k][k-2]);
//  * the solver warp has issue scheduler 0 to itself (warp placement below);
//  * block / sweep indices are carried incrementally (no division by nblk).
#include "cd_common.cuh"

#include <algorithm>
#include <cstdio>

namespace pam {

namespace bp {

#ifdef PAM_BLK_PROF
#define PROF_DECL long long pf_t[8] = {0, 0, 0, 0, 0, 0, 0, 0}; long long pf_c = 0;
#define PROF_START pf_c = clock64();
#define PROF_LAP(i) { const long long pf_n = clock64(); pf_t[i] += pf_n - pf_c; pf_c = pf_n; }
#else
#define PROF_DECL
#define PROF_START
#define PROF_LAP(i)
#endif

constexpr int STAGES = 4;       // blocks t-1 (AXPY), t (solve), t+1 (dots), t+2 (in flight)
constexpr int NWK = 8;          // worker warps (16 measured 30 % slower: per-column overhead scales with warps)
// Warp roles.  Warp w issues on scheduler w % 4: the solver (warp 0) keeps scheduler
// 0 to itself -- its ~60-instruction serial stream per column gets every issue
// slot -- sharing it only with the stream warp (4, a few instructions per step) and
// an idle warp (8); the worker warps are the ones with w % 4 != 0.
constexpr int NWARPS = NWK + (NWK - 1) / 3 + 1;  // NWK = 8: warps 0..10
constexpr int NT = NWARPS * 32;
constexpr int DT = 4 * 32;  // the stream warp's issuing thread
constexpr int RPT = 1024 / (NWK * 32);  // residual rows per worker thread (= tiles per worker warp)
static_assert(RPT == 4 && NWK == 8, "worker row ownership and the fixed 8-warp sums assume 8 worker warps of 4 rows per thread");
constexpr int LCAP = 16;            // entries per worker warp's column list (= GMAX)
constexpr int64_t WS_PER_SLOT = 576;  // 32 B descriptor + 2 x 33 Gram doubles (+ padding) per slot
constexpr int64_t WS_PER_FIT = 96;

struct Blk {  // per block of a fit, in the workspace
  int j0, nb, gd, go;  // first column, columns, diagonal / previous-block Gram offsets (doubles)
  int woff, wlen, nbp, pad;  // packed W offset / length (doubles), columns of the previous block
};

__device__ __forceinline__ int even_up(int x) { return (x + 1) & ~1; }
__device__ __forceinline__ int col_pack(int rel, int code) { return rel | ((code & 0xff) << 16) | ((code >> 8) << 24); }

template <int SLOT_WD, int GMAX, int MINB>
__global__ void __launch_bounds__(NT, MINB) cd_block_kernel(const CdArgs a, unsigned char* const ws) {
  constexpr int GD = GMAX * GMAX;
  constexpr int SLOT_D = SLOT_WD + 2 * GD;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* const slots = reinterpret_cast<double*>(smem_raw);
  double* const zpart = slots + STAGES * SLOT_D;  // [2][NWK][16] block dots per worker warp (element parity)
  double* const zraw = zpart + 2 * NWK * 16;      // [64] staging (beta0 of a prologue block)
  double* const dfull = zraw + 64;              // [2][32] block steps by column (element parity)
  double* const red = dfull + 64;               // [64] reductions (sweep-parity double-buffered)
  double* const sprm = red + 64;                // [20][4] solver: {beta, 1/denom, G[k][k-1], G[k][k-2]} of column k
  int* const par = reinterpret_cast<int*>(sprm + 80);  // [4][32] packed column parameters (element & 3)
  int* const enb = par + 128;                         // [4] columns of element (e & 3)
  int* const lcp = enb + 4;                           // [4][NWK][LCAP] per worker warp: the element's columns whose run meets its rows
  int* const lcnt = lcp + 4 * NWK * LCAP;             // [4][NWK] entries of each list
  int* const ctl = lcnt + 4 * NWK;  // [10]: nblk, next item, stop flags [2] (step parity), sweeps done, converged
  uint64_t* const bars = reinterpret_cast<uint64_t*>(ctl + 10);  // 8-byte aligned
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool solver = warp == 0;
  const int ww = warp - 1 - (warp >> 2);  // worker index of a worker warp
  const bool worker = (warp & 3) != 0 && ww < NWK;
  const bool streamer = warp == 4;  // descriptor / parameter pipeline and the bulk copies
  const uint32_t slots_s = smem_u32(slots);
  const uint32_t bars_s = smem_u32(bars);

  if (tid == 0) {
    for (int i = 0; i < STAGES; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncthreads();

  uint32_t ebase = 0;  // ring elements consumed by earlier fits / passes (all threads)
  unsigned item = blockIdx.x;

  auto cta_bar = [&]() { __syncthreads(); };

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
      unsigned char* const wsf = ws + doff * WS_PER_SLOT + s * WS_PER_FIT;
      Blk* blk = reinterpret_cast<Blk*>(wsf);
      double* Gf = reinterpret_cast<double*>(wsf + sizeof(Blk) * (M + 1));
      double* invs = Gf + 32 * static_cast<int64_t>(M);  // 1 / (col_sq + lam2) by column (Gram blocks take <= 32 doubles per column)
      const double lam1 = a.lam1[s], lam2 = a.lam2[s], tol = a.tol[s];
      const int max_iters = a.max_iters[s];

      // ---- block boundaries (warp 0): <= GMAX columns whose packed tiles fit a slot
      if (warp == 0) {
        int nb = 0, j0 = 0, gpos = 0, acc = 0, nbp = 0;
        auto close = [&](int j1) {
          const int n = j1 - j0;
          if (lane == 0) {
            Blk bk;
            bk.j0 = j0;
            bk.nb = n;
            bk.woff = static_cast<int>(colo[j0]);
            bk.wlen = acc;
            bk.nbp = nbp;  // fixed up for block 0 below
            bk.gd = gpos;
            bk.go = gpos + even_up(n * n);
            bk.pad = 0;
            blk[nb] = bk;
          }
          gpos += even_up(n * n) + even_up(n * GMAX);  // previous block has <= GMAX columns
          nbp = n;
          ++nb;
          j0 = j1;
          acc = 0;
        };
        for (int cb = 0; cb < M; cb += 32) {
          const int c = cb + lane;
          const int wl = (c < M) ? 32 * __popcll(tmk[c]) : 0;
          const int cnt = min(32, M - cb);
          for (int t = 0; t < cnt; ++t) {
            const int j = cb + t;
            const int w = __shfl_sync(0xffffffffu, wl, t);
            if (j > j0 && (acc + w > SLOT_WD || j - j0 == GMAX)) close(j);
            acc += w;
          }
        }
        close(M);
        __syncwarp();
        if (lane == 0) {
          blk[0].nbp = blk[nb - 1].nb;  // block 0 follows the last block of the previous sweep
          ctl[0] = nb;
        }
      }
      // residual rows of a worker thread (position order, perm -> local row): worker warp w
      // owns positions [32 RPT w, 32 RPT (w + 1)); lane l the pairs 64 v + 2 l + {0, 1}, so a
      // warp's 16-byte tile loads are contiguous in shared memory (no bank conflicts)
      double r[RPT];
#pragma unroll
      for (int k = 0; k < RPT; ++k) r[k] = 0.0;
      if (worker) {
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
          const int p = 32 * RPT * ww + 64 * (k >> 1) + 2 * lane + (k & 1);
          const int row = a.perm ? (p < N ? a.perm[r0 + p] : 0) : p;
          r[k] = (p < N) ? a.y[r0 + row] : 0.0;
        }
      }
      cta_bar();
      const int nblk = ctl[0];

      // ---- the ring: element e (counted from the pass start) = one block's packed
      //      W + its Gram blocks; thread 32 issues, every thread waits each element
      //      once, in order (`seen`), so no wait ever lags a slot by two phases
#ifdef PAM_BLK_PROF_TMA
      long long tma_cyc = 0, tma_bytes = 0;
#endif
      Blk ibk;  // stream thread: descriptor of its next issue (loaded one issue ahead)
      auto iload = [&](int b) {
        if (tid == DT) ibk = blk[b];
      };
      auto issue = [&](uint32_t e, bool with_g, int b_next) {
        if (tid == DT) {
          const Blk bk = ibk;
          const int st = (ebase + e) % STAGES;
          const uint32_t wbytes = static_cast<uint32_t>(bk.wlen) * 8u;
          const uint32_t gbytes = with_g ? static_cast<uint32_t>(even_up(bk.nb * bk.nb)) * 8u : 0u;
          const uint32_t obytes = with_g ? static_cast<uint32_t>(even_up(bk.nb * bk.nbp)) * 8u : 0u;
          const uint32_t bar = bars_s + st * 8;
          mbar_expect_s(bar, wbytes + gbytes + obytes);
          bulk_g2s(slots_s + st * (SLOT_D * 8), Ws + bk.woff, wbytes, bar);
          if (gbytes) bulk_g2s(slots_s + (st * SLOT_D + SLOT_WD) * 8, Gf + bk.gd, gbytes, bar);
          if (obytes) bulk_g2s(slots_s + (st * SLOT_D + SLOT_WD + GD) * 8, Gf + bk.go, obytes, bar);
#ifdef PAM_BLK_PROF_TMA
          {
            const long long c0 = clock64();
            while (!mbar_test_s(bar, ((ebase + e) / STAGES) & 1u)) {
            }
            tma_cyc += clock64() - c0;
            tma_bytes += wbytes + gbytes + obytes;
          }
#endif
        }
        iload(b_next);
      };
      auto slot_of = [&](uint32_t e) -> const double* { return slots + ((ebase + e) % STAGES) * SLOT_D; };
      uint32_t seen = 0;
      // one lane polls, the warp follows through __syncwarp (a warp-wide try_wait on
      // one barrier word from nine warps at once measured ~700 cycles per step)
      auto wait_next = [&]() {
        if (lane == 0) mbar_wait_s(bars_s + ((ebase + seen) % STAGES) * 8, ((ebase + seen) / STAGES) & 1u);
        __syncwarp();
        ++seen;
      };
      // packed column parameters of block b: registers (one warp, lane c <-> column
      // j0 + c), published into buffer k of par / enb later
      int pf_par = 0, pf_nb = 0;
      auto pfetch = [&](int b) {
        const Blk bk = blk[b];
        pf_nb = bk.nb;
        pf_par = (lane < bk.nb) ? col_pack(static_cast<int>(colo[bk.j0 + lane]) - bk.woff,
                                           tile_code(tmk[bk.j0 + lane]))
                                : 0;
      };
      // warp NWK's register pipeline: descriptor (two publishes ahead), then the raw
      // column offset / tile mask (one publish ahead), packed only at publish time
      Blk pd;
      int rw_nb = 0, rw_woff = 0;
      long long rw_off = 0;
      unsigned long long rw_mk = 0ull;
      auto pfetch_d = [&](const Blk& bk) {
        rw_nb = bk.nb;
        rw_woff = bk.woff;
        rw_off = (lane < bk.nb) ? colo[bk.j0 + lane] : 0;
        rw_mk = (lane < bk.nb) ? tmk[bk.j0 + lane] : 0ull;
      };
      auto pack_raw = [&]() {
        pf_nb = rw_nb;
        pf_par = (lane < rw_nb) ? col_pack(static_cast<int>(rw_off) - rw_woff, tile_code(rw_mk)) : 0;
      };
      // publish element buffer k: the packed parameters by column, and per worker warp w
      // the list of the columns whose tile run meets w's rows (tiles RPT w .. RPT w +
      // RPT - 1), in column order; a list entry is offset | column << 13 | a0 << 17 | la << 22
      auto publish = [&](int k) {
        par[32 * k + lane] = pf_par;
        if (lane == 0) enb[k] = pf_nb;
        const int a0 = (pf_par >> 16) & 0xff, la = (pf_par >> 24) & 0xff;
        const bool on = lane < pf_nb && la > 0;
        const int wlo = a0 / RPT, whi = (a0 + la - 1) / RPT;
        const int entry = (pf_par & 0x1fff) | (lane << 13) | (a0 << 17) | (la << 22);
        const unsigned lt = (1u << lane) - 1u;
#pragma unroll
        for (int w = 0; w < NWK; ++w) {
          const bool mine = on && wlo <= w && w <= whi;
          const unsigned m = __ballot_sync(0xffffffffu, mine);
          if (mine) lcp[(k * NWK + w) * LCAP + __popc(m & lt)] = entry;
          if (lane == 0) lcnt[k * NWK + w] = __popc(m);
        }
      };
      // workers: rows -= sum d_j W_j over the columns j of this warp's list (entries
      // lst[0..cnt), steps dv[] by column), four columns per pass (all loads of a pass in
      // flight before its FMAs; a tile outside the column's run, or an entry past cnt,
      // contributes an exact zero), in column order
      auto axpy_cols = [&](const double* Wb, const double* dv, const int* lst, int cnt) {
        const int tile0 = RPT * ww + (lane >> 4);  // tile of pair v: tile0 + 2 v
        const int sub = (2 * lane) & 31;
        const double2 zz = make_double2(0.0, 0.0);
        for (int k = 0; k < cnt; k += 4) {
          double d[4];
          double2 w[4][RPT / 2];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const bool ok = k + u < cnt;
            const int cp = lst[ok ? k + u : k];
            const int o = cp & 0x1fff, j = (cp >> 13) & 15, a0 = (cp >> 17) & 31, la = cp >> 22;
#pragma unroll
            for (int v = 0; v < RPT / 2; ++v) {
              const int tr = tile0 + 2 * v - a0;
              const bool in = ok && static_cast<unsigned>(tr) < static_cast<unsigned>(la);
              w[u][v] = in ? *reinterpret_cast<const double2*>(Wb + o + 32 * tr + sub) : zz;
            }
            d[u] = dv[j];
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
#pragma unroll
            for (int v = 0; v < RPT / 2; ++v) {
              r[2 * v] = fma(-d[u], w[u][v].x, r[2 * v]);
              r[2 * v + 1] = fma(-d[u], w[u][v].y, r[2 * v + 1]);
            }
          }
        }
      };
      // a warp's squared norm of packed column cp -> every lane (prologue col_sq)
      auto col_sq_dot = [&](const double* Wb, int cp) -> double {
        const int o = cp & 0xffff, la = cp >> 24;
        const double2* w2 = reinterpret_cast<const double2*>(Wb + o);
        const int n2 = 16 * la;  // double2 elements of the run
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int i = lane;
        for (; i + 32 < n2; i += 64) {
          const double2 wa = w2[i], wb = w2[i + 32];
          s0 = fma(wa.x, wa.x, s0);
          s1 = fma(wa.y, wa.y, s1);
          s2 = fma(wb.x, wb.x, s2);
          s3 = fma(wb.y, wb.y, s3);
        }
        if (i < n2) {
          const double2 wa = w2[i];
          s0 = fma(wa.x, wa.x, s0);
          s1 = fma(wa.y, wa.y, s1);
        }
        return warp_sum((s0 + s1) + (s2 + s3));
      };
      // workers: the dots of a block's columns against the residual, ROW parallel: each
      // thread multiplies its own rows (registers) with the entries of those rows in
      // the columns of its warp's list (the columns whose run meets the warp's rows),
      // the warp adds its 32 lanes' partial sums by a halving butterfly (16 -> 8 ->
      // 4 -> 2 -> 1 values per lane, or 8 -> .. for lists of <= 8 columns) and the
      // lanes holding a total store it to the column's entry of zp[16] (zero for the
      // columns not on the list); the solver adds the worker warps' parts in warp
      // order.  No residual mirror in shared memory: per block the shared-memory
      // traffic is the block's tiles, once for the dots and once for the AXPY.
      auto block_dots = [&](const double* Wb, const int* lst, int cnt, double* zp) {
        const int tile0 = RPT * ww + (lane >> 4);  // tile of pair v: tile0 + 2 v
        const int sub = (2 * lane) & 31;
        const double2 zz = make_double2(0.0, 0.0);
        double p[16];
        if (lane < 16) zp[lane] = 0.0;
#pragma unroll
        for (int j0 = 0; j0 < 16; j0 += 4) {
          if (j0 < cnt) {
            double2 w[4][RPT / 2];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const bool ok = j0 + u < cnt;
              const int cp = lst[ok ? j0 + u : j0];
              const int o = cp & 0x1fff, a0 = (cp >> 17) & 31, la = cp >> 22;
#pragma unroll
              for (int v = 0; v < RPT / 2; ++v) {
                const int tr = tile0 + 2 * v - a0;
                const bool in = ok && static_cast<unsigned>(tr) < static_cast<unsigned>(la);
                w[u][v] = in ? *reinterpret_cast<const double2*>(Wb + o + 32 * tr + sub) : zz;
              }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
              for (int v = 0; v < RPT / 2; ++v) {
                acc0 = fma(w[u][v].x, r[2 * v], acc0);
                acc1 = fma(w[u][v].y, r[2 * v + 1], acc1);
              }
              p[j0 + u] = acc0 + acc1;
            }
          } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) p[j0 + u] = 0.0;
          }
        }
        __syncwarp();  // the zeroed zp is ordered before the totals below
        int pos;       // list position of the total this lane ends up holding
        double tot;
        if (cnt > 8) {
#pragma unroll
          for (int lvl = 0; lvl < 4; ++lvl) {
            const int half = 8 >> lvl;  // values kept after this level
            const int bit = 16 >> lvl;  // lane bit of this level
            const bool hi = (lane & bit) != 0;
#pragma unroll
            for (int i = 0; i < half; ++i) {
              const double keep = hi ? p[i + half] : p[i];
              const double send = hi ? p[i] : p[i + half];
              p[i] = keep + __shfl_xor_sync(0xffffffffu, send, bit);
            }
          }
          tot = p[0] + __shfl_xor_sync(0xffffffffu, p[0], 1);
          pos = lane >> 1;
        } else {
#pragma unroll
          for (int lvl = 0; lvl < 3; ++lvl) {
            const int half = 4 >> lvl;
            const int bit = 16 >> lvl;
            const bool hi = (lane & bit) != 0;
#pragma unroll
            for (int i = 0; i < half; ++i) {
              const double keep = hi ? p[i + half] : p[i];
              const double send = hi ? p[i] : p[i + half];
              p[i] = keep + __shfl_xor_sync(0xffffffffu, send, bit);
            }
          }
          double t2 = p[0] + __shfl_xor_sync(0xffffffffu, p[0], 2);
          tot = t2 + __shfl_xor_sync(0xffffffffu, t2, 1);
          pos = lane >> 2;
        }
        const bool holder = (cnt > 8) ? (lane & 1) == 0 : (lane & 3) == 0;
        if (holder && pos < cnt) zp[(lst[pos] >> 13) & 15] = tot;
      };
      // ---- prologue pass: col_sq (elastic_net.py:85), r = y - W beta0 (94), and the
      //      diagonal and previous-block Gram blocks; elements 0..nblk-1, then block 0
      //      once more for G[0, nblk-1] (block 0 follows block nblk-1 across sweeps)
      {
        const uint32_t np_el = static_cast<uint32_t>(nblk) + 1;
        auto pblock = [&](uint32_t e) -> int { return e < static_cast<uint32_t>(nblk) ? static_cast<int>(e) : 0; };
        uint32_t q = 0;
        iload(0);
        for (; q < min(static_cast<uint32_t>(STAGES - 1), np_el); ++q) issue(q, false, pblock(q + 1 < np_el ? q + 1 : q));
        for (uint32_t e = 0; e < np_el; ++e) {
          const bool wrap = e == static_cast<uint32_t>(nblk);
          const int b = pblock(e);
          const Blk bk = blk[b];
          const int nb = bk.nb;
          if (warp == 1) {
            pfetch(b);
            publish(e & 3);
          }
          if (!wrap && tid < nb) zraw[tid] = betas[bk.j0 + tid];  // beta0 of the block
          wait_next();
          cta_bar();
          const double* Wb = slot_of(e);
          const int* pk = par + 32 * (e & 3);
          if (!wrap) {
            for (int j = warp; j < nb; j += NWARPS) {
              const double cs = col_sq_dot(Wb, pk[j]);
              if (lane == 0) {
                colsq[bk.j0 + j] = cs;
                const double dn = __dadd_rn(cs, lam2);
                invs[bk.j0 + j] = dn > 0.0 ? __ddiv_rn(1.0, dn) : 0.0;
              }
            }
          }
          // Gram blocks: diagonal G[c][k] (not for the wrap element) and previous-block
          // G[c][i] = W_c . W_i (c in this block, i in the previous one), stored with c
          // fastest: diagonal at [k * nb + c], previous-block at [i * nb + c]
          const int gd_n = wrap ? 0 : nb * nb;
          const int nbp = (e == 0) ? 0 : bk.nbp;
          const double* Wp = (e == 0) ? Wb : slot_of(e - 1);
          const int* pkp = par + 32 * ((e - 1) & 3);
          for (int pi = tid; pi < gd_n + nb * nbp; pi += NT) {
            const bool diag = pi < gd_n;
            const int q2 = diag ? pi : pi - gd_n;
            const int c = q2 % nb, k = q2 / nb;
            const int cpc = pk[c];
            const int cpk = diag ? pk[k] : pkp[k];
            const double* Wk = diag ? Wb : Wp;
            const int oc = cpc & 0xffff, ac = (cpc >> 16) & 0xff, lc = cpc >> 24;
            const int ok = cpk & 0xffff, ak = (cpk >> 16) & 0xff, lk = cpk >> 24;
            const int t0 = max(ac, ak), t1 = min(ac + lc, ak + lk);
            double g = 0.0;
            for (int tt = t0; tt < t1; ++tt) {
              const double* pc = Wb + oc + 32 * (tt - ac);
              const double* pq = Wk + ok + 32 * (tt - ak);
#pragma unroll 8
              for (int i = 0; i < 32; ++i) g = fma(pc[i], pq[i], g);
            }
            Gf[(diag ? bk.gd : bk.go) + k * nb + c] = g;
          }
          if (!wrap && worker) {  // r -= W_b beta0_b
            const int li = static_cast<int>(e & 3) * NWK + ww;
            axpy_cols(Wb, zraw, lcp + li * LCAP, lcnt[li]);
          }
          asm volatile("fence.proxy.async.global;" ::: "memory");  // the sweeps re-read G by TMA
          cta_bar();  // slot e-1 free
          if (q < np_el) {
            issue(q, false, pblock(q + 1 < np_el ? q + 1 : q));
            ++q;
          }
        }
        ebase += np_el;
      }

      // ---- sweeps: one continuous stream of blocks, element t = block t % nblk of
      //      sweep t / nblk.  Step t: solver -> block t; workers -> AXPY of t-1, dots of t+1.
      //      Block and sweep indices are carried incrementally (bcur, swc, qb): a
      //      division by the run-time nblk costs ~40 instructions on every warp.
      const uint32_t total = static_cast<uint32_t>(nblk) * static_cast<uint32_t>(max_iters);
      auto modn = [&](int x) -> int {
        while (x >= nblk) x -= nblk;
        return x;
      };
      seen = 0;
      uint32_t q = 0;
      int qb = 0;  // q % nblk
      iload(0);
      for (; q < min(static_cast<uint32_t>(STAGES - 1), total); ++q) {
        const int qn = modn(qb + 1);
        issue(q, true, qn);
        qb = qn;
      }
      if (streamer) {
        if (total > 0) {
          pfetch(0);
          publish(0);
        }
        if (total > 1) {
          pfetch(modn(1));
          publish(1);
        }
        if (total > 2) {
          pfetch(modn(2));          // published at step 0
          pfetch_d(blk[modn(3)]);   // packed at step 0, published at step 1
          pd = blk[modn(4)];        // columns loaded at step 0
        }
      }
      if (tid < 64) dfull[tid] = 0.0;
      if (tid < 2) ctl[2 + tid] = 0;  // stop flags (step parity)
      if (tid == 0) ctl[4] = ctl[5] = 0;  // sweeps done, converged
      cta_bar();
      if (worker && total > 0) {  // pre-step: dots of element 0 against the prologue residual
        wait_next();
        block_dots(slot_of(0), lcp + ww * LCAP, lcnt[ww], zpart + ww * 16);
      }
      cta_bar();

      // solver state: lane c <-> column c of the current block; descriptors and the
      // next block's beta / col_sq are register-pipelined (no global load on the chain)
      double bc = 0.0, csc = 0.0;
      double nbx = 0.0, ncs = 0.0, ninv = 0.0;  // beta / col_sq / 1 / (col_sq + lam2) of element t+1
      Blk sd_cur, sd_n1, sd_n2;     // descriptors of elements t, t+1, t+2
      auto sprefetch = [&](const Blk& bk) {
        nbx = (lane < bk.nb) ? betas[bk.j0 + lane] : 0.0;
        ncs = (lane < bk.nb) ? colsq[bk.j0 + lane] : 0.0;
        ninv = (lane < bk.nb) ? invs[bk.j0 + lane] : 0.0;  // 1 / (col_sq + lam2), from the prologue
      };
      if (solver && total > 0) {
        sd_n1 = blk[0];
        sd_n2 = blk[modn(1)];
        sprefetch(sd_n1);
      }
      double max_delta = 0.0, acc_l1 = 0.0, acc_l2 = 0.0, acc_max = 0.0;  // solver, per sweep
      double corr = 0.0;  // solver: G[t, t-1] d_{t-1} of this lane's column (accumulated during step t-1)
      double invc = 0.0;                // 1 / (col_sq + lam2) of this block's column
      double g1n = 0.0, g2n = 0.0;      // next block's G[c][c-1], G[c][c-2] (read from its slot a step early)
      bool first_blk = true;
      int st_j = -1;      // deferred coefficient store: index (or -1) and value
      double st_b = 0.0;
      int bcur = 0, swc = 0;  // t % nblk, t / nblk
      PROF_DECL
      for (uint32_t t = 0; total > 0; ++t) {
        const bool stopped = ctl[2 + ((t + 1) & 1)] != 0;  // set by the solver at step t-1
        const bool sweep_closed = t > 0 && bcur == 0;      // step t-1 was the last block of sweep swc - 1
        PROF_START
        if (solver) {
          if (!stopped) {
            if (st_j >= 0) betas[st_j] = st_b;  // previous block's coefficients (deferred)
            st_j = -1;
            sd_cur = sd_n1;
            sd_n1 = sd_n2;
            const Blk& bk = sd_cur;
            const int nb = bk.nb;
            if (nblk > 1 || t == 0) {
              bc = nbx;
              csc = ncs;
              invc = ninv;
            }
            if (nblk > 1 && t + 1 < total) sprefetch(sd_n1);  // its betas were written by this lane
            if (t + 2 < total) sd_n2 = blk[modn(bcur + 2)];
            PROF_LAP(0)
            if (seen <= t) wait_next();
            PROF_LAP(1)
            const double* Wb = slot_of(t);
            const double* Gd = Wb + SLOT_WD;
            // the next block's previous-block Gram block G[t+1, t] (its slot landed a
            // step ago): the term -G[t+1, t] d_t of the next step's dots is accumulated
            // inside this step's update loop, off the serial chain
            const bool has_next = t + 1 < total;
            if (has_next && seen <= t + 1) wait_next();
            const double* Go1 = slot_of(t + 1) + SLOT_WD + GD;
            const int nb1 = has_next ? sd_n1.nb : 0;
            // z = (zraw - G[t, t-1] d_{t-1}) + col_sq beta; lane c <-> column c
            double zsum = 0.0;
            if (lane < nb) {
              const double* zb = zpart + (t & 1) * NWK * 16 + lane;
              double zw[NWK];
#pragma unroll
              for (int w = 0; w < NWK; ++w) zw[w] = zb[16 * w];
              zsum = ((zw[0] + zw[1]) + (zw[2] + zw[3])) + ((zw[4] + zw[5]) + (zw[6] + zw[7]));  // fixed tree over the worker warps
            }
            const double zdot = (lane < nb) ? __dsub_rn(zsum, corr) : 0.0;
            double zc = __dadd_rn(__dmul_rn(csc, bc), zdot);
            // per-column constants, broadcast-read inside the loop (columns >= nb:
            // zeros, so a padded step is exactly d = 0): beta, 1 / (col_sq + lam2) and the
            // two sub-diagonal Gram entries G[k][k-1], G[k][k-2] (loaded a step early
            // from this block's slot, except for the first block)
            {
              const bool on = lane < nb;
              double g1 = g1n, g2 = g2n;
              if (first_blk) {
                g1 = (on && lane > 0) ? Gd[(lane - 1) * nb + lane] : 0.0;
                g2 = (on && lane > 1) ? Gd[(lane - 2) * nb + lane] : 0.0;
                first_blk = false;
              }
              if (lane < 20) {
                double2* sp = reinterpret_cast<double2*>(sprm + 4 * lane);
                sp[0] = make_double2(on ? bc : 0.0, on ? invc : 0.0);
                sp[1] = make_double2(g1, g2);
              }
            }
            __syncwarp();
            PROF_LAP(2)
            // the block's cyclic updates (elastic_net.py:137-156).  Lane c carries
            // zc = col_sq_c beta_c + W_c . r with the block's earlier steps applied.
            // Column k's value is broadcast TWO steps early (steps <= k-3 applied) and
            // the terms of steps k-2 and k-1 are applied to the broadcast copy:
            //   z_k = [zpre_k - d_{k-2} G[k][k-2] + beta_{k-1} G[k][k-1]] - b_{k-1} G[k][k-1]
            // with b_{k-1} the NEW coefficient of column k-1, so the bracket is ready
            // before b_{k-1} and the serial chain per column is one FMA, the shift by
            // lam1, one multiply by 1 / (col_sq + lam2) and the sign selects.  (The
            // quotient is the product with the correctly rounded reciprocal: <= 1.5 ulp
            // from the reference's division, far inside the rounding class of the
            // reordered inner products.)  Four columns per straight-line group.
            double dc = 0.0;
            double zq = __shfl_sync(0xffffffffu, zc, 0);    // bracket of column k
            double zp1 = __shfl_sync(0xffffffffu, zc, 1);   // broadcast copy of column k+1 (steps <= k-2)
            double bprev = 0.0, dprev = 0.0;
            double cr0 = 0.0, cr1 = 0.0;
            const double* gcp = Gd + lane;    // G[lane][k] at gcp[k * nb]
            const double* gop = Go1 + lane;   // G[t+1 column lane][t column k] at gop[k * nb1]
            const bool lane_on = lane < nb, lane_on1 = lane < nb1;
            for (int k0 = 0; k0 < nb; k0 += 4) {
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int k = k0 + u;
                const double2 p0 = *reinterpret_cast<const double2*>(sprm + 4 * k);        // beta_k, inv_k
                const double2 p1 = *reinterpret_cast<const double2*>(sprm + 4 * k + 2);    // G[k][k-1], G[k][k-2]
                const double2 q1 = *reinterpret_cast<const double2*>(sprm + 4 * k + 6);    // G[k+1][k], G[k+1][k-1]
                const bool kin = k < nb;
                const double gcol = (kin && lane_on) ? gcp[k * nb] : 0.0;
                const double gnx = (kin && lane_on1) ? gop[k * nb1] : 0.0;
                // bracket of column k+1 from the copy taken one step ago (steps <= k-2
                // applied): step k-1's term and column k's OLD coefficient times G[k+1][k]
                const double zq_n = fma(p0.x, q1.x, fma(-dprev, q1.y, zp1));
                const double zp2 = __shfl_sync(0xffffffffu, zc, (k + 2) & 31);  // steps <= k-1 applied
                // serial chain
                const double z = fma(-bprev, p1.x, zq);
                const double np_ = __dsub_rn(z, lam1), nn_ = __dadd_rn(z, lam1);
                const double qp = __dmul_rn(np_, p0.y), qn = __dmul_rn(nn_, p0.y);
                const double b_new = np_ > 0.0 ? qp : (nn_ < 0.0 ? qn : 0.0);
                // off the chain
                const double d = __dsub_rn(b_new, p0.x);
                zc = fma(-d, gcol, zc);
                if (u & 1) cr1 = fma(d, gnx, cr1);
                else cr0 = fma(d, gnx, cr0);
                if (lane == k) {
                  bc = b_new;
                  dc = d;
                }
                const double ad = fabs(d);
                max_delta = ad > max_delta ? ad : max_delta;
                bprev = b_new;
                dprev = d;
                zq = zq_n;
                zp1 = zp2;
              }
            }
            corr = cr0 + cr1;
            // next block: its sub-diagonal Gram entries and column parameters (slot t+1 is
            // resident, parameters published two steps ago) -- off the next step's chain
            if (has_next) {
              const double* Gd1 = slot_of(t + 1) + SLOT_WD;
              const bool on1 = lane < nb1;
              g1n = (on1 && lane > 0) ? Gd1[(lane - 1) * nb1 + lane] : 0.0;
              g2n = (on1 && lane > 1) ? Gd1[(lane - 2) * nb1 + lane] : 0.0;
            }
            PROF_LAP(3)
            // steps by column for the workers' AXPY (their per-warp column lists were built
            // by the stream warp when it published the block)
            dfull[32 * (t & 1) + lane] = (lane < nb) ? dc : 0.0;
            // the block's coefficients go to global memory at the top of the NEXT step:
            // a store issued right before the CTA barrier holds every warp at the barrier
            // until it is performed (~700 cycles per step, 40 % of all stall samples)
            st_j = (lane < nb) ? bk.j0 + lane : -1;
            st_b = bc;
            if (lane < nb) {
              const double ab = fabs(bc);
              acc_l1 += ab;
              acc_l2 = fma(bc, bc, acc_l2);
              acc_max = fmax(acc_max, ab);
            }
            int stop = 0;
            if (bcur == nblk - 1) {  // sweep complete: the reference's stop rule (elastic_net.py:158)
              const double l1 = warp_sum(acc_l1), l2 = warp_sum(acc_l2), mabs = warp_max(acc_max);
              const double md = warp_max(max_delta);
              const int sw = swc;
              const bool cv = md <= __dmul_rn(tol, fmax(mabs, 1.0));
              if (lane == 0) {
                red[8 + 2 * (sw & 1)] = l1;
                red[9 + 2 * (sw & 1)] = l2;
                ctl[4] = sw + 1;
                if (cv) ctl[5] = 1;
              }
              stop = (cv || sw + 1 == max_iters) ? 1 : 0;
              max_delta = acc_l1 = acc_l2 = acc_max = 0.0;
            }
            if (lane == 0) ctl[2 + (t & 1)] = stop;
            PROF_LAP(4)
          } else if (lane == 0) {
            ctl[2 + (t & 1)] = 1;
          }
        } else if (worker) {
          // workers: r -= W_{t-1} d_{t-1}, then (unless stopped) the dots of t+1
          if (t > 0) {
            const uint32_t e = t - 1;
            const int li = static_cast<int>(e & 3) * NWK + ww;
            axpy_cols(slot_of(e), dfull + 32 * (e & 1), lcp + li * LCAP, lcnt[li]);
          }
          PROF_LAP(0)
          PROF_LAP(1)
          if (!stopped && t + 1 < total) {
            const uint32_t e = t + 1;
            wait_next();
            PROF_LAP(4)
            const int li = static_cast<int>(e & 3) * NWK + ww;
            block_dots(slot_of(e), lcp + li * LCAP, lcnt[li], zpart + ((e & 1) * NWK + ww) * 16);
          }
          PROF_LAP(3)
          if (sweep_closed) {
            // the AXPY above completed sweep swc - 1: its residual sum of squares
            const int sw = swc - 1;
            double rr = 0.0;
#pragma unroll
            for (int k = 0; k < RPT; ++k) rr = fma(r[k], r[k], rr);
            rr = warp_sum(rr);
            if (lane == 0) red[32 + 16 * (sw & 1) + ww] = rr;
          }
        }
        else if (streamer && !stopped && t + 2 < total) {
          // stream warp: the parameter pipeline (global loads; nothing else waits on them)
          publish((t + 2) & 3);                             // packed at step t-1
          pack_raw();                                       // element t+3 (raw loads of step t-1)
          if (t + 4 < total) pfetch_d(pd);                  // element t+4's columns (descriptor of step t-1)
          if (t + 5 < total) pd = blk[modn(bcur + 5)];      // element t+5's descriptor
        }
        PROF_LAP(5)
        cta_bar();  // end of step t
        PROF_LAP(6)
        if (sweep_closed && tid == DT) {
          const int sw = swc - 1;
          double rss = 0.0;
#pragma unroll
          for (int w = 0; w < NWK; ++w) rss += red[32 + 16 * (sw & 1) + w];
          const double obj = __dadd_rn(__dadd_rn(__dmul_rn(0.5, rss), __dmul_rn(lam1, red[8 + 2 * (sw & 1)])),
                                       __dmul_rn(__dmul_rn(0.5, lam2), red[9 + 2 * (sw & 1)]));
          if (a.hist != nullptr) a.hist[a.hist_off[s] + sw] = obj;
          red[12] = obj;
        }
        if (stopped) break;  // this was the drain step (the final AXPY)
        if (q < total && ctl[2 + (t & 1)] == 0) {  // refill the slot of element t-1
          const int qn = modn(qb + 1);
          issue(q, true, qn);
          qb = qn;
          ++q;
        }
        if (++bcur == nblk) {
          bcur = 0;
          ++swc;
        }
        PROF_LAP(7)
      }
      if (solver && st_j >= 0) betas[st_j] = st_b;  // the last block's coefficients
#ifdef PAM_BLK_PROF_TMA
      if (blockIdx.x == 0 && tid == DT) printf("tma fit %d: %lld cycles for %lld bytes, %u issues\n", (int)s, tma_cyc, tma_bytes, q);
#endif
#ifdef PAM_BLK_PROF
      if (blockIdx.x == 0 && lane == 0 && (warp == 0 || warp == 1 || warp == 5 || warp == 4))
        printf("blkprof fit %d warp %d nblk %d M %d: %lld %lld %lld %lld %lld %lld %lld %lld\n", (int)s, warp, nblk, M, pf_t[0], pf_t[1], pf_t[2], pf_t[3], pf_t[4], pf_t[5], pf_t[6], pf_t[7]);
#endif
      if (max_iters == 0) {
        // objective at the given beta (prologue residual)
        double rr = 0.0, q1 = 0.0, q2 = 0.0;
        if (worker) {
#pragma unroll
          for (int k = 0; k < RPT; ++k) rr = fma(r[k], r[k], rr);
        }
        for (int j = tid; j < M; j += NT) {
          const double bj = betas[j];
          q1 += fabs(bj);
          q2 = fma(bj, bj, q2);
        }
        rr = warp_sum(rr);
        q1 = warp_sum(q1);
        q2 = warp_sum(q2);
        if (lane == 0) {
          red[warp] = rr;
          red[20 + warp] = q1;
          red[40 + warp] = q2;
        }
        cta_bar();
        if (tid == 32) {
          double rss = 0.0, t1 = 0.0, t2 = 0.0;
          for (int w = 0; w < NWARPS; ++w) {
            rss += red[w];
            t1 += red[20 + w];
            t2 += red[40 + w];
          }
          red[12] = __dadd_rn(__dadd_rn(__dmul_rn(0.5, rss), __dmul_rn(lam1, t1)), __dmul_rn(__dmul_rn(0.5, lam2), t2));
        }
      }
      // observe every element issued beyond the stop (at most STAGES - 1 behind)
      if (!solver && !worker) seen = q;  // stream / idle warps never waited in the sweeps; phases derive from ebase + seen
      while (seen < q) wait_next();
      cta_bar();
      if (tid == 32) {
        a.sweeps[s] = max_iters == 0 ? 0 : ctl[4];
        a.converged[s] = max_iters == 0 ? 0 : ctl[5];
        a.objective[s] = red[12];
      }
      ebase += q;
    }
    cta_bar();
    if (tid == 0) ctl[1] = static_cast<int>(atomicAdd(a.queue, 1u) + gridDim.x);
    cta_bar();
    item = static_cast<unsigned>(ctl[1]);
  }
}

}  // namespace bp

int64_t cd_block_workspace_bytes(int64_t S, int64_t total_slots) {
  return total_slots * bp::WS_PER_SLOT + S * bp::WS_PER_FIT;
}

template <int SLOT_WD, int GMAX, int MINB>
int launch_block_pipe_cfg(const CdArgs& a, void* block_ws, cudaStream_t stream) {
  using namespace bp;
  const size_t smem = static_cast<size_t>(STAGES) * (SLOT_WD + 2 * GMAX * GMAX) * 8 + (2 * NWK * 16 + 64 * 3 + 80) * 8 +
                      (128 + 4 + 4 * NWK * LCAP + 4 * NWK + 10) * 4 + 8 * STAGES + 16;
  auto kernel = cd_block_kernel<SLOT_WD, GMAX, MINB>;
  PAM_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  PAM_CUDA_CHECK(cudaMemsetAsync(a.queue, 0, sizeof(unsigned), stream));
  const int64_t ctas = std::max<int64_t>(1, std::min<int64_t>(static_cast<int64_t>(MINB) * sm_count(), a.S));
  kernel<<<(unsigned)ctas, NT, smem, stream>>>(a, static_cast<unsigned char*>(block_ws));
  PAM_LAUNCH_CHECK("cd_block_kernel");
  return PAM_OK;
}

// One CTA per SM (544 threads; C3's 256 fits run in two waves, which measured
// faster than two CTAs per SM with half the slot), 4 x (44 KB W + 2 x 2 KB Gram)
// slots, blocks of up to 16 columns (a BASELINE C2/C3 column is ~5 KB of tiles,
// so the W slot decides the block size in round 0).
int launch_cd_block(const CdArgs& a, int max_rows, void* block_ws, cudaStream_t stream) {
  if (max_rows > 1024 || block_ws == nullptr) return PAM_ERR_UNSUPPORTED;
  return launch_block_pipe_cfg<5632, 16, 1>(a, block_ws, stream);
}

}  // namespace pam
