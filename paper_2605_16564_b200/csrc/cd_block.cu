// cd_block.cu — exact blocked cyclic CD for batches of FEW fits (<= 3 per SM,
// BASELINE configs 2-3: 64-256 fits of 1,024 rows, up to 2,860 columns).
//
// Reference loop (elastic_net.py:114-161): for j = 0..M-1 in order,
//   z_j = col_sq_j beta_j + W_j . r,  b = S(z_j, lam1) / (col_sq_j + lam2),
//   r -= (b - beta_j) W_j.
// With one or two fits per SM the per-column chain (dot -> warp reduction ->
// soft threshold -> AXPY) of the one-warp kernels IS the runtime (~0.55 us per
// column, profiles/r01_ncu_cd_pair_c2_raw.csv: FP64 pipe 4 %, DRAM 0.05 of
// peak).  This kernel reorganises the same cyclic sweep exactly:
//
//   columns are taken in blocks B = [j0, j1) (<= 32 columns whose packed tiles
//   fit one shared-memory slot);
//   1. all dots W_B^T r of the block at once (independent, row-parallel over
//      the CTA's 8 warps, then a 31-shuffle transposed reduction per warp and a
//      fixed-order cross-warp sum);
//   2. the cyclic updates inside the block, in order, with the in-block
//      corrections  W_k . r_{after j} = W_k . r - sum_{i<=j} d_i G[k][i]  from the
//      block's diagonal Gram block G = W_B^T W_B (computed once per round in the
//      prologue pass, stored in the workspace, streamed with the block);
//   3. one AXPY r -= W_B d_B for the whole block (columns with d = 0 skipped:
//      exactly the reference's "no update when b_new == b_old").
// Only the rounding of the length-N inner products differs from the
// reference's sequential sums (the SURVEY F2 class, ~1e-12 in beta); every
// decision (order, soft threshold, division, stop rule) is the reference's.
// The serial chain per column shrinks to one shuffle + the soft threshold +
// one FMA (~80 cycles) instead of a 5-level reduction and a ring round trip,
// and the streaming of W is spread over 8 warps with 26 KB bulk copies.
//
// Layout: one CTA (8 warps) per fit, persistent CTAs pulling fits from the
// queue (2 CTAs per SM).  Warp w owns the 32-row tiles t = w + 8k (k < 4) of
// the tile-packed design matrix (tiles.cu), lane l row l of each tile, so the
// residual lives in 4 registers per thread and every in-run test is
// warp-uniform (a branch, not a select).  Ring: 3 slots of [packed W of the
// block | its diagonal Gram block], one cp.async.bulk each, issued by thread
// 0 two blocks ahead; a slot is refilled after the barrier of the next block,
// which every warp reaches only after finishing the previous block.
#include "cd_common.cuh"

#include <algorithm>

namespace pam {

constexpr int BK_STAGES = 3;
constexpr int BK_NW = 8;          // warps per fit
// Workspace per fit s at byte dict_off[s] * 288 + 32 s: (nblk + 1) <= M + 1 block
// descriptors int4 (first column, Gram offset, W offset, W doubles), then the
// diagonal Gram blocks (nb x nb row-major, each padded to an even count:
// sum <= 33 M + 1 doubles), i.e. <= 288 bytes per dictionary slot + 32.
constexpr int64_t BK_WS_PER_SLOT = 288;
constexpr int64_t BK_WS_PER_FIT = 32;

__device__ __forceinline__ int even_up(int x) { return (x + 1) & ~1; }

// packed per-column parameter: relative offset (doubles, < 2^16) | a0 << 16 | la << 24
__device__ __forceinline__ int col_pack(int rel, int code) { return rel | ((code & 0xff) << 16) | ((code >> 8) << 24); }

// The in-block cyclic updates (elastic_net.py:137-156 for j = j0..j1-1), run
// by one warp with every lane computing the same chain: the block's dots live
// in registers z[0..NS), the step for column k reads z[k] directly (no
// shuffle on the serial path), and only z[k+1]'s correction d_k G[k+1][k] is
// on the chain; the other corrections and the smem broadcast loads of G,
// beta, col_sq and 1/(col_sq + lam2) are independent of it.  NS >= nb is a
// compile-time bound (8/16/24/32), so z stays in registers.
template <int NS>
__device__ __forceinline__ double block_solve(int nb, const double* zd, double* bsm, double* bsm2,
                                              const double* csm, const double* ism, const double* G,
                                              double* dd, double lam1, double lam2, int lane, double max_delta) {
  double z[NS];
#pragma unroll
  for (int j = 0; j < NS; ++j) z[j] = (j < nb) ? zd[j] : 0.0;
#pragma unroll
  for (int k = 0; k < NS; ++k) {
    if (k < nb) {
      const double b_old = bsm[k];
      const double cs = csm[k];
      const double inv = ism[k];
      const double dn = __dadd_rn(cs, lam2);
      const double zz = __dadd_rn(__dmul_rn(cs, b_old), z[k]);
      const double np_ = __dsub_rn(zz, lam1), nn_ = __dadd_rn(zz, lam1);
      const double qp = __dmul_rn(np_, inv), qn = __dmul_rn(nn_, inv);
      const double bp = fma(fma(-qp, dn, np_), inv, qp);
      const double bn = fma(fma(-qn, dn, nn_), inv, qn);
      const double b_new = np_ > 0.0 ? bp : (nn_ < 0.0 ? bn : 0.0);
      const double d = __dsub_rn(b_new, b_old);
#pragma unroll
      for (int j = k + 1; j < NS; ++j)
        if (j < nb) z[j] = fma(-d, G[j * nb + k], z[j]);
      if (lane == 0) {
        bsm[k] = b_new;
        if (bsm2) bsm2[k] = b_new;
        dd[k] = d;
      }
      const double ad = fabs(d);
      max_delta = ad > max_delta ? ad : max_delta;
    }
  }
  return max_delta;
}

// Per block, three phases separated by CTA barriers:
//   D  dots: warp w takes columns j = w, w + NW, ... of the block; a column is
//      one contiguous run of 32 la doubles in the slot, dotted against the
//      residual mirror rs[32 a0 ..] with 16-byte loads, then a warp sum;
//   S  solve: warp 0, lane c <-> column j0 + c, the cyclic updates in order
//      with the in-block Gram corrections (all other warps meanwhile idle);
//   A  AXPY: thread t owns rows 4t..4t+3 (registers), applies every column
//      with d != 0 whose run covers its tile, then refreshes its rows of rs.
template <int NW, int STAGES, int SLOT_WD, int MINB>
__global__ void __launch_bounds__(NW * 32, MINB) cd_block_kernel(const CdArgs a, unsigned char* const ws) {
  constexpr int NT = NW * 32;
  constexpr int RPT = 1024 / NT;  // residual rows per thread (N <= 1024)
  static_assert(RPT == 4, "row ownership assumes 256 threads");
  constexpr int SLOT_D = SLOT_WD + 1024;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* const slots = reinterpret_cast<double*>(smem_raw);
  double* const rs = slots + STAGES * SLOT_D;  // [1024] residual mirror (position order)
  double* const zd = rs + 1024;                // [32] block dots
  double* const dd = zd + 32;                  // [32] block steps
  double* const pb = dd + 32;                  // [2][32] beta of the block's columns
  double* const pc = pb + 64;                  // [2][32] col_sq
  double* const pi = pc + 64;                  // [2][32] 1 / (col_sq + lam2)
  double* const sred = pi + 64;                // [NW + 8] reductions / broadcast scalars
  int* const par = reinterpret_cast<int*>(sred + NW + 8);  // [2][32] packed column parameters
  int* const ctl = par + 64;                                // [4]: nblk, next item, next-block j0 / nb
  uint64_t* const bars = reinterpret_cast<uint64_t*>(ctl + 4);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t slots_s = smem_u32(slots);
  const uint32_t bars_s = smem_u32(bars);

  if (tid == 0) {
    for (int i = 0; i < STAGES; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncthreads();

  int st = 0;       // consumer slot (all threads)
  uint32_t ph = 0;  // its parity
  int ist = 0;      // producer slot (tracked by all threads, used by thread 0)
  unsigned item = blockIdx.x;

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
      unsigned char* const wsf = ws + doff * BK_WS_PER_SLOT + s * BK_WS_PER_FIT;
      int4* blk = reinterpret_cast<int4*>(wsf);
      double* Gf = reinterpret_cast<double*>(wsf + 16 * (M + 1));
      const double lam1 = a.lam1[s], lam2 = a.lam2[s], tol = a.tol[s];
      const int max_iters = a.max_iters[s];

      // ---- block boundaries: <= 32 columns whose packed tiles fit a slot
      if (warp == 0) {
        int nb = 0, j0 = 0, gpos = 0, acc = 0;
        for (int cb = 0; cb < M; cb += 32) {
          const int c = cb + lane;
          const int wl = (c < M) ? 32 * __popcll(tmk[c]) : 0;
          const int cnt = min(32, M - cb);
          for (int t = 0; t < cnt; ++t) {
            const int j = cb + t;
            const int w = __shfl_sync(0xffffffffu, wl, t);
            if (j > j0 && (acc + w > SLOT_WD || j - j0 == 32)) {  // close [j0, j)
              if (lane == 0) blk[nb] = make_int4(j0, gpos, static_cast<int>(colo[j0]), acc);
              gpos += even_up((j - j0) * (j - j0));
              ++nb;
              j0 = j;
              acc = 0;
            }
            acc += w;
          }
        }
        if (lane == 0) {
          blk[nb] = make_int4(j0, gpos, static_cast<int>(colo[j0]), acc);
          gpos += even_up((M - j0) * (M - j0));
          blk[nb + 1] = make_int4(M, gpos, 0, 0);
          ctl[0] = nb + 1;
        }
      }
      // residual rows 4 tid .. 4 tid + 3 (position order; perm -> local row)
      double r[RPT];
#pragma unroll
      for (int k = 0; k < RPT; ++k) {
        const int p = RPT * tid + k;
        const int row = a.perm ? (p < N ? a.perm[r0 + p] : 0) : p;
        r[k] = (p < N) ? a.y[r0 + row] : 0.0;
        rs[p] = r[k];
      }
      __syncthreads();
      const int nblk = ctl[0];

      // thread 0 keeps the descriptor of its next issue in registers (loaded one
      // issue ahead, so the global load is off the barrier-to-barrier path)
      int4 ibk = make_int4(0, 0, 0, 0);
      int inx = 0;
      auto iload = [&](int b) {
        if (tid == 0) {
          ibk = blk[b];
          inx = blk[b + 1].x;
        }
      };
      auto issue = [&](int b, bool with_g, int b_next) {
        if (tid == 0) {
          const int4 bk = ibk;
          const int nbk = inx - bk.x;
          const uint32_t wbytes = static_cast<uint32_t>(bk.w) * 8u;
          const uint32_t gbytes = with_g ? static_cast<uint32_t>(even_up(nbk * nbk)) * 8u : 0u;
          const uint32_t bar = bars_s + ist * 8;
          mbar_expect_s(bar, wbytes + gbytes);
          bulk_g2s(slots_s + ist * (SLOT_D * 8), Ws + bk.z, wbytes, bar);
          if (gbytes) bulk_g2s(slots_s + (ist * SLOT_D + SLOT_WD) * 8, Gf + bk.y, gbytes, bar);
          (void)b;
        }
        iload(b_next);
        if (++ist == STAGES) ist = 0;
      };
      auto wait_slot = [&]() -> const double* {
        mbar_wait_s(bars_s + st * 8, ph);
        const double* p = slots + st * SLOT_D;
        if (++st == STAGES) {
          st = 0;
          ph ^= 1u;
        }
        return p;
      };
      // parameters of a block (warp `w_load`, lane c <-> column j0 + c): global
      // loads into registers first (prefetch), published to the smem buffer later
      int pf_ctl = 0, pf_par = 0;
      double pf_b = 0.0, pf_cs = 0.0;
      auto prefetch_params = [&](int b, int w_load) {
        if (warp == w_load) {
          const int4 bk = blk[b];
          const int nbk = blk[b + 1].x - bk.x;
          pf_ctl = bk.x | (nbk << 24);  // j0 < 2^24, nb <= 32
          if (lane < nbk) {
            const int j = bk.x + lane;
            pf_par = col_pack(static_cast<int>(colo[j]) - bk.z, tile_code(tmk[j]));
            pf_b = betas[j];
            pf_cs = colsq[j];
          }
        }
      };
      auto publish_params = [&](int pbuf, int w_load, bool with_beta) {
        if (warp == w_load) {
          if (lane == 0) ctl[2 + pbuf] = pf_ctl;
          par[32 * pbuf + lane] = pf_par;
          if (with_beta) pb[32 * pbuf + lane] = pf_b;
          pc[32 * pbuf + lane] = pf_cs;
          const double dn = __dadd_rn(pf_cs, lam2);
          pi[32 * pbuf + lane] = dn > 0.0 ? __ddiv_rn(1.0, dn) : 0.0;
        }
      };
      auto load_params = [&](int b, int pbuf, int w_load) {
        prefetch_params(b, w_load);
        publish_params(pbuf, w_load, true);
      };
      // phase A: rows of this thread -= sum_j d_j W_j (columns with d == 0 skipped)
      auto axpy = [&](const double* Wb, const double* dsrc, int pbuf, int nb) {
        const int tile = (RPT * tid) >> 5;
        const int sub = (RPT * tid) & 31;
        for (int j = 0; j < nb; ++j) {
          const double dj = dsrc[j];
          if (dj == 0.0) continue;
          const int cp = par[32 * pbuf + j];
          const int o = cp & 0xffff, a0 = (cp >> 16) & 0xff, la = cp >> 24;
          if (static_cast<unsigned>(tile - a0) < static_cast<unsigned>(la)) {
            const double2* w2 = reinterpret_cast<const double2*>(Wb + o + 32 * (tile - a0) + sub);
            const double2 u = w2[0], v = w2[1];
            r[0] = fma(-dj, u.x, r[0]);
            r[1] = fma(-dj, u.y, r[1]);
            r[2] = fma(-dj, v.x, r[2]);
            r[3] = fma(-dj, v.y, r[3]);
          }
        }
        double2* r2 = reinterpret_cast<double2*>(rs + RPT * tid);
        r2[0] = make_double2(r[0], r[1]);
        r2[1] = make_double2(r[2], r[3]);
      };
      // phase D: warp dot of column j with rs (or with itself: col_sq) -> lane 0
      auto col_dot = [&](const double* Wb, int cp, bool self) -> double {
        const int o = cp & 0xffff, a0 = (cp >> 16) & 0xff, la = cp >> 24;
        const double2* w2 = reinterpret_cast<const double2*>(Wb + o);
        const double2* r2 = reinterpret_cast<const double2*>(rs + 32 * a0);
        double s0 = 0.0, s1 = 0.0;
        for (int i = lane; i < 16 * la; i += 32) {
          const double2 w = w2[i];
          const double2 x = self ? w : r2[i];
          s0 = fma(w.x, x.x, s0);
          s1 = fma(w.y, x.y, s1);
        }
        return warp_sum(s0 + s1);
      };

      // ---- prologue pass: col_sq (elastic_net.py:85), r = y - W beta0 (94),
      //      diagonal Gram blocks (written to the workspace)
      {
        int q = 0;
        iload(0);
        for (; q < min(STAGES - 1, nblk); ++q) issue(q, false, min(q + 1, nblk - 1));
        for (int b = 0; b < nblk; ++b) {
          load_params(b, 0, 0);
          const double* Wb = wait_slot();
          __syncthreads();  // params visible; every warp past the previous block
          if (q < nblk) {
            issue(q, false, min(q + 1, nblk - 1));
            ++q;
          }
          const int j0 = ctl[2] & 0xffffff, nb = ctl[2] >> 24;
          for (int j = warp; j < nb; j += NW) {
            const double cs = col_dot(Wb, par[j], true);
            if (lane == 0) colsq[j0 + j] = cs;
          }
          // diagonal Gram block G[c][k] = W_c . W_k over the intersection of the runs
          const int np = nb * (nb + 1) / 2;
          const int gpos = blk[b].y;
          for (int pi = tid; pi < np; pi += NT) {
            int c = 0, rem = pi;
            while (rem >= nb - c) {
              rem -= nb - c;
              ++c;
            }
            const int k = c + rem;
            const int pcc = par[c], pkk = par[k];
            const int oc = pcc & 0xffff, ac = (pcc >> 16) & 0xff, lc = pcc >> 24;
            const int ok = pkk & 0xffff, ak = (pkk >> 16) & 0xff, lk = pkk >> 24;
            const int t0 = max(ac, ak), t1 = min(ac + lc, ak + lk);
            double g = 0.0;
            for (int t = t0; t < t1; ++t) {
              const double* pcw = Wb + oc + 32 * (t - ac);
              const double* pkw = Wb + ok + 32 * (t - ak);
#pragma unroll 8
              for (int i = 0; i < 32; ++i) g = fma(pcw[i], pkw[i], g);
            }
            Gf[gpos + c * nb + k] = g;
            Gf[gpos + k * nb + c] = g;
          }
          axpy(Wb, pb, 0, nb);  // r -= W beta0 (zero betas skipped)
          // the Gram blocks are read back by the async (TMA) proxy in the sweeps
          asm volatile("fence.proxy.async.global;" ::: "memory");
          __syncthreads();  // slot, params and rs consumed / refreshed
        }
      }

      // ---- sweeps (elastic_net.py:137-161)
      int sweeps_done = 0, conv = 0;
      double obj = 0.0;
      const int total = nblk * max_iters;
      int q = 0;
      iload(0);
      for (; q < min(STAGES - 1, total); ++q) issue(q % nblk, true, (q + 1) % nblk);
      if (total > 0) load_params(0, 0, 0);
      int pbuf = 0;
      for (int sw = 0; sw < max_iters; ++sw) {
        double max_delta = 0.0, acc_l1 = 0.0, acc_l2 = 0.0, acc_max = 0.0;  // warp 0
        for (int b = 0; b < nblk; ++b) {
          const double* Wb = wait_slot();
          __syncthreads();  // B1: params of b and rs visible; every warp past block b-1
          if (q < total) {
            issue(q % nblk, true, (q + 1) % nblk);
            ++q;
          }
          const int j0 = ctl[2 + pbuf] & 0xffffff, nb = ctl[2 + pbuf] >> 24;
          // the next block's parameters: its columns are not written by this block
          // (one block: warp 0 keeps both beta buffers current instead)
          prefetch_params(b + 1 < nblk ? b + 1 : 0, NW - 1);
          // D: all dots of the block
          for (int j = warp; j < nb; j += NW) {
            const double z = col_dot(Wb, par[32 * pbuf + j], false);
            if (lane == 0) zd[j] = z;
          }
          __syncthreads();  // B2: dots visible
          // S: cyclic updates inside the block (warp 0)
          if (warp == 0) {
            const double* Gb = Wb + SLOT_WD;
            double* bsm = pb + 32 * pbuf;
            // one-block dictionary: the next "block" is this one, keep its betas current
            double* bsm2 = (nblk == 1) ? pb + 32 * (pbuf ^ 1) : nullptr;
            const double* csm = pc + 32 * pbuf;
            const double* ism = pi + 32 * pbuf;
            if (nb <= 8) max_delta = block_solve<8>(nb, zd, bsm, bsm2, csm, ism, Gb, dd, lam1, lam2, lane, max_delta);
            else if (nb <= 16) max_delta = block_solve<16>(nb, zd, bsm, bsm2, csm, ism, Gb, dd, lam1, lam2, lane, max_delta);
            else if (nb <= 24) max_delta = block_solve<24>(nb, zd, bsm, bsm2, csm, ism, Gb, dd, lam1, lam2, lane, max_delta);
            else max_delta = block_solve<32>(nb, zd, bsm, bsm2, csm, ism, Gb, dd, lam1, lam2, lane, max_delta);
            __syncwarp();
            if (lane < nb) {
              const double bc = bsm[lane];
              betas[j0 + lane] = bc;
              const double ab = fabs(bc);
              acc_l1 += ab;
              acc_l2 = fma(bc, bc, acc_l2);
              acc_max = fmax(acc_max, ab);
            }
          }
          __syncthreads();  // B3: steps visible; betas of this block written
          // A: r -= W_B d_B; publish the next block's parameters
          publish_params(pbuf ^ 1, NW - 1, nblk > 1);
          axpy(Wb, dd, pbuf, nb);
          pbuf ^= 1;
        }
        // objective after the sweep; every thread reaches the same decision
        double rr = 0.0;
#pragma unroll
        for (int k = 0; k < RPT; ++k) rr = fma(r[k], r[k], rr);
        rr = warp_sum(rr);
        if (lane == 0) sred[warp] = rr;
        if (warp == 0) {
          const double l1 = warp_sum(acc_l1), l2 = warp_sum(acc_l2), mabs = warp_max(acc_max);
          if (lane == 0) {
            sred[NW] = l1;
            sred[NW + 1] = l2;
            sred[NW + 2] = mabs;
            sred[NW + 3] = max_delta;
          }
        }
        __syncthreads();
        double rss = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) rss += sred[w];
        const double l1 = sred[NW], l2 = sred[NW + 1], mabs = sred[NW + 2], md = sred[NW + 3];
        obj = __dadd_rn(__dadd_rn(__dmul_rn(0.5, rss), __dmul_rn(lam1, l1)),
                        __dmul_rn(__dmul_rn(0.5, lam2), l2));
        if (a.hist != nullptr && tid == 0) a.hist[a.hist_off[s] + sw] = obj;
        sweeps_done = sw + 1;
        __syncthreads();  // sred consumed before the next sweep reuses it
        if (md <= __dmul_rn(tol, fmax(mabs, 1.0))) {
          conv = 1;
          break;
        }
      }
      if (max_iters == 0) {
        double rr = 0.0, q1 = 0.0, q2 = 0.0;
#pragma unroll
        for (int k = 0; k < RPT; ++k) rr = fma(r[k], r[k], rr);
        for (int j = tid; j < M; j += NT) {
          const double bj = betas[j];
          q1 += fabs(bj);
          q2 = fma(bj, bj, q2);
        }
        rr = warp_sum(rr);
        q1 = warp_sum(q1);
        q2 = warp_sum(q2);
        if (lane == 0) {
          sred[warp] = rr;
          zd[warp] = q1;
          dd[warp] = q2;
        }
        __syncthreads();
        double rss = 0.0, t1 = 0.0, t2 = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          rss += sred[w];
          t1 += zd[w];
          t2 += dd[w];
        }
        obj = __dadd_rn(__dadd_rn(__dmul_rn(0.5, rss), __dmul_rn(lam1, t1)), __dmul_rn(__dmul_rn(0.5, lam2), t2));
      }
      // drain the copies issued for blocks that will not run
      const int consumed = sweeps_done * nblk;
      for (int c = consumed; c < q; ++c) (void)wait_slot();
      __syncthreads();
      if (tid == 0) {
        a.sweeps[s] = sweeps_done;
        a.converged[s] = conv;
        a.objective[s] = obj;
      }
    }
    __syncthreads();
    if (tid == 0) ctl[1] = static_cast<int>(atomicAdd(a.queue, 1u) + gridDim.x);
    __syncthreads();
    item = static_cast<unsigned>(ctl[1]);
  }
}

int64_t cd_block_workspace_bytes(int64_t S, int64_t total_slots) {
  return total_slots * BK_WS_PER_SLOT + S * BK_WS_PER_FIT;
}

template <int SLOT_WD, int PER_SM>
int launch_block_cfg(const CdArgs& a, void* block_ws, cudaStream_t stream) {
  constexpr int per_sm = PER_SM;
  constexpr int NW = BK_NW, STAGES = BK_STAGES;
  const size_t smem = static_cast<size_t>(STAGES) * (SLOT_WD + 1024) * 8 + (1024 + 32 * 2 + 64 * 3 + NW + 8) * 8 +
                      (64 + 4) * 4 + 8 * STAGES + 16;
  auto kernel = cd_block_kernel<NW, STAGES, SLOT_WD, PER_SM>;
  PAM_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  PAM_CUDA_CHECK(cudaMemsetAsync(a.queue, 0, sizeof(unsigned), stream));
  const int64_t ctas = std::max<int64_t>(1, std::min<int64_t>(static_cast<int64_t>(per_sm) * sm_count(), a.S));
  kernel<<<(unsigned)ctas, NW * 32, smem, stream>>>(a, static_cast<unsigned char*>(block_ws));
  PAM_LAUNCH_CHECK("cd_block_kernel");
  return PAM_OK;
}

// <= 1 fit per SM: one CTA per SM with 3 x 64 KB slots (blocks of up to 32
// columns); more fits: two CTAs per SM with 3 x 24 KB slots.
int launch_cd_block(const CdArgs& a, int max_rows, void* block_ws, cudaStream_t stream) {
  if (max_rows > 1024 || block_ws == nullptr) return PAM_ERR_UNSUPPORTED;
  if (a.S <= sm_count()) return launch_block_cfg<7680, 1>(a, block_ws, stream);
  return launch_block_cfg<3072, 2>(a, block_ws, stream);
}

}  // namespace pam
