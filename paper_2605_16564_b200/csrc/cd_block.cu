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
// packed tiles fit a shared-memory slot): all dots of a block at once
// (column-parallel, one warp per column), the block's cyclic updates in order
// through its diagonal Gram block G_bb (one solver warp, one shuffle + the soft
// threshold + one FMA per column on the serial path), one row-parallel AXPY
// for the block.  The first, unpipelined version of this (round 2) ran the
// three phases back to back and left 8 of 9 warps idle during the solve
// (37 % of stall samples, profiles/r02_ncu_cd_block_c2_lines.txt); here block
// t's solve overlaps block t-1's AXPY and block t+1's dots:
//
//   workers (8 warps), step t:  r -= W_{t-1} d_{t-1};  zraw_{t+1} = W_{t+1}^T r
//   solver  (1 warp),  step t:  z_t = zraw_t - G[t, t-1] d_{t-1};  in-block
//                               cyclic updates of block t -> d_t
//
// zraw_{t+1} is formed against the residual BEFORE block t's updates; the
// missing term is exactly -G[t+1, t] d_t (G = W^T W restricted to the two
// blocks), applied by the solver at the start of step t+1 -- the same
// identity as the in-block corrections, now across the block boundary, so the
// update sequence is still the reference's cyclic order j = 0..M-1, sweep
// after sweep (elastic_net.py:137-161); only the rounding of the inner
// products differs (~1e-12, the SURVEY F2 class).  The stream of blocks is
// continuous across sweeps (block 0 of sweep k+1 follows block nblk-1 of sweep
// k, with G[0, nblk-1]).  The diagonal and the off-diagonal (previous-block)
// Gram blocks are computed once per round in the prologue pass and streamed
// with the block.  One end-of-step CTA barrier per block; the workers add one
// named barrier between their AXPY and their dots.
#include "cd_common.cuh"

#include <algorithm>

namespace pam {

namespace bp {

constexpr int STAGES = 4;       // blocks t-1 (AXPY), t (solve), t+1 (dots), t+2 (in flight)
constexpr int NWK = 8;          // worker warps
constexpr int NT = (NWK + 1) * 32;  // + solver warp 0
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
  double* const rs = slots + STAGES * SLOT_D;  // [1024] residual mirror (position order)
  double* const zraw = rs + 1024;               // [2][32] block dots (element parity)
  double* const dd = zraw + 64;                 // [2][32] block steps, compacted to the nonzero ones
  double* const dfull = dd + 64;                // [2][32] block steps by column (solver)
  double* const red = dfull + 64;               // [32] reductions (sweep-parity double-buffered)
  int* const par = reinterpret_cast<int*>(red + 32);  // [4][32] packed column parameters (element & 3)
  int* const enb = par + 128;                         // [4] columns of element (e & 3)
  int* const nzi = enb + 4;                           // [2][32] columns of the nonzero steps
  int* const enz = nzi + 64;                          // [2] nonzero steps of the element
  int* const ctl = enz + 2;  // [8]: nblk, next item, stop flags [2] (step parity), sweeps done, converged
  uint64_t* const bars = reinterpret_cast<uint64_t*>(ctl + 10);  // 8-byte aligned
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool solver = warp == 0;
  const int wt = tid - 32;  // worker thread index (0..255), rows 4 wt .. 4 wt + 3
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
  auto worker_bar = [&]() { asm volatile("bar.sync 1, %0;" ::"n"(NWK * 32) : "memory"); };

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
      // residual rows 4 wt .. 4 wt + 3 (workers; position order, perm -> local row)
      double r[4] = {0.0, 0.0, 0.0, 0.0};
      if (!solver) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int p = 4 * wt + k;
          const int row = a.perm ? (p < N ? a.perm[r0 + p] : 0) : p;
          r[k] = (p < N) ? a.y[r0 + row] : 0.0;
          rs[p] = r[k];
        }
      }
      cta_bar();
      const int nblk = ctl[0];

      // ---- the ring: element e (counted from the pass start) = one block's packed
      //      W + its Gram blocks; thread 32 issues, every thread waits each element
      //      once, in order (`seen`), so no wait ever lags a slot by two phases
      Blk ibk;  // thread 32: descriptor of its next issue (loaded one issue ahead)
      auto iload = [&](int b) {
        if (tid == 32) ibk = blk[b];
      };
      auto issue = [&](uint32_t e, bool with_g, int b_next) {
        if (tid == 32) {
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
        }
        iload(b_next);
      };
      auto slot_of = [&](uint32_t e) -> const double* { return slots + ((ebase + e) % STAGES) * SLOT_D; };
      uint32_t seen = 0;
      auto wait_next = [&]() {
        mbar_wait_s(bars_s + ((ebase + seen) % STAGES) * 8, ((ebase + seen) / STAGES) & 1u);
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
      auto publish = [&](int k) {
        par[32 * k + lane] = pf_par;
        if (lane == 0) enb[k] = pf_nb;
      };
      // workers: rows -= sum_j d_j W_j over the block in slot Wb (d == 0 skipped)
      auto axpy = [&](const double* Wb, const double* dsrc, const int* pk, int nb) {
        const int tile = (4 * wt) >> 5;
        const int sub = (4 * wt) & 31;
        for (int j = 0; j < nb; ++j) {
          const double dj = dsrc[j];
          if (dj == 0.0) continue;
          const int cp = pk[j];
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
        double2* r2 = reinterpret_cast<double2*>(rs + 4 * wt);
        r2[0] = make_double2(r[0], r[1]);
        r2[1] = make_double2(r[2], r[3]);
      };
      // workers, sweeps: rows -= d_k W_{col k} over the compacted nonzero steps
      auto axpy_nz = [&](const double* Wb, const double* dnz, const int* idx, int cnt, const int* pk) {
        const int tile = (4 * wt) >> 5;
        const int sub = (4 * wt) & 31;
        // two columns per pass: both columns' loads are in flight before the FMAs
        // (a column outside this thread's tile contributes an exact zero step)
        auto term = [&](int k, double& dj, double2& u, double2& v) {
          const int cp = pk[idx[k]];
          const int o = cp & 0xffff, a0 = (cp >> 16) & 0xff, la = cp >> 24;
          const bool in = static_cast<unsigned>(tile - a0) < static_cast<unsigned>(la);
          const double2* w2 = reinterpret_cast<const double2*>(Wb + (in ? o + 32 * (tile - a0) + sub : 0));
          u = w2[0];
          v = w2[1];
          dj = in ? dnz[k] : 0.0;
        };
        int k = 0;
        for (; k + 1 < cnt; k += 2) {
          double da, db;
          double2 ua, va, ub, vb;
          term(k, da, ua, va);
          term(k + 1, db, ub, vb);
          r[0] = fma(-db, ub.x, fma(-da, ua.x, r[0]));
          r[1] = fma(-db, ub.y, fma(-da, ua.y, r[1]));
          r[2] = fma(-db, vb.x, fma(-da, va.x, r[2]));
          r[3] = fma(-db, vb.y, fma(-da, va.y, r[3]));
        }
        if (k < cnt) {
          double da;
          double2 ua, va;
          term(k, da, ua, va);
          r[0] = fma(-da, ua.x, r[0]);
          r[1] = fma(-da, ua.y, r[1]);
          r[2] = fma(-da, va.x, r[2]);
          r[3] = fma(-da, va.y, r[3]);
        }
        double2* r2 = reinterpret_cast<double2*>(rs + 4 * wt);
        r2[0] = make_double2(r[0], r[1]);
        r2[1] = make_double2(r[2], r[3]);
      };
      // a warp's dot of packed column cp with rs (self: with itself) -> every lane
      auto col_dot = [&](const double* Wb, int cp, bool self) -> double {
        const int o = cp & 0xffff, a0 = (cp >> 16) & 0xff, la = cp >> 24;
        const double2* w2 = reinterpret_cast<const double2*>(Wb + o);
        const double2* x2 = reinterpret_cast<const double2*>(rs + 32 * a0);
        const int n2 = 16 * la;  // double2 elements of the run
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int i = lane;
        for (; i + 32 < n2; i += 64) {  // two independent element pairs per lane per pass
          const double2 wa = w2[i], wb = w2[i + 32];
          const double2 xa = self ? wa : x2[i], xb = self ? wb : x2[i + 32];
          s0 = fma(wa.x, xa.x, s0);
          s1 = fma(wa.y, xa.y, s1);
          s2 = fma(wb.x, xb.x, s2);
          s3 = fma(wb.y, xb.y, s3);
        }
        if (i < n2) {
          const double2 wa = w2[i];
          const double2 xa = self ? wa : x2[i];
          s0 = fma(wa.x, xa.x, s0);
          s1 = fma(wa.y, xa.y, s1);
        }
        return warp_sum((s0 + s1) + (s2 + s3));
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
            for (int j = warp; j < nb; j += NWK + 1) {
              const double cs = col_dot(Wb, pk[j], true);
              if (lane == 0) colsq[bk.j0 + j] = cs;
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
          if (!wrap && !solver) axpy(Wb, zraw, pk, nb);  // r -= W_b beta0_b
          asm volatile("fence.proxy.async.global;" ::: "memory");  // the sweeps re-read G by TMA
          cta_bar();  // slot e-1 free, rs current
          if (q < np_el) {
            issue(q, false, pblock(q + 1 < np_el ? q + 1 : q));
            ++q;
          }
        }
        ebase += np_el;
      }

      // ---- sweeps: one continuous stream of blocks, element t = block t % nblk of
      //      sweep t / nblk.  Step t: solver -> block t; workers -> AXPY of t-1, dots of t+1.
      const uint32_t total = static_cast<uint32_t>(nblk) * static_cast<uint32_t>(max_iters);
      seen = 0;
      uint32_t q = 0;
      iload(0);
      for (; q < min(static_cast<uint32_t>(STAGES - 1), total); ++q) issue(q, true, static_cast<int>((q + 1) % nblk));
      if (total > 0 && warp == 1) {
        pfetch(0);
        publish(0);
      }
      if (total > 1 && warp == 2) {
        pfetch(1 % nblk);
        publish(1);
      }
      if (total > 2 && warp == NWK) {
        pfetch(2 % nblk);  // published at step 0
        pfetch_d(blk[3 % nblk]);  // packed at step 0, published at step 1
        pd = blk[4 % nblk];       // columns loaded at step 0
      }
      if (tid < 2) enz[tid] = 0;
      if (tid < 64) dd[tid] = dfull[tid] = 0.0;
      if (tid < 2) ctl[2 + tid] = 0;  // stop flags (step parity)
      if (tid == 0) ctl[4] = ctl[5] = 0;  // sweeps done, converged
      cta_bar();
      if (!solver && total > 0) {  // pre-step: dots of element 0 against the prologue residual
        wait_next();
        const double* Wb = slot_of(0);
        for (int j = warp - 1; j < enb[0]; j += NWK) {
          const double z = col_dot(Wb, par[j], false);
          if (lane == 0) zraw[j] = z;
        }
      }
      cta_bar();

      // solver state: lane c <-> column c of the current block; descriptors and the
      // next block's beta / col_sq are register-pipelined (no global load on the chain)
      double bc = 0.0, csc = 0.0;
      double nbx = 0.0, ncs = 0.0;  // beta / col_sq of element t+1
      Blk sd_cur, sd_n1, sd_n2;     // descriptors of elements t, t+1, t+2
      auto sprefetch = [&](const Blk& bk) {
        nbx = (lane < bk.nb) ? betas[bk.j0 + lane] : 0.0;
        ncs = (lane < bk.nb) ? colsq[bk.j0 + lane] : 0.0;
      };
      if (solver && total > 0) {
        sd_n1 = blk[0];
        sd_n2 = blk[1 % nblk];
        sprefetch(sd_n1);
      }
      double max_delta = 0.0, acc_l1 = 0.0, acc_l2 = 0.0, acc_max = 0.0;  // solver, per sweep
      for (uint32_t t = 0; total > 0; ++t) {
        const bool stopped = ctl[2 + ((t + 1) & 1)] != 0;  // set by the solver at step t-1
        if (solver) {
          if (!stopped) {
            const int b = static_cast<int>(t % nblk);
            sd_cur = sd_n1;
            sd_n1 = sd_n2;
            const Blk& bk = sd_cur;
            const int nb = bk.nb;
            if (nblk > 1 || t == 0) {
              bc = nbx;
              csc = ncs;
            }
            const double dnc = __dadd_rn(csc, lam2);
            const double invc = dnc > 0.0 ? __ddiv_rn(1.0, dnc) : 0.0;
            if (nblk > 1 && t + 1 < total) sprefetch(sd_n1);  // its betas were written by this lane
            if (t + 2 < total) sd_n2 = blk[(t + 2) % nblk];
            wait_next();
            const double* Wb = slot_of(t);
            const double* Gd = Wb + SLOT_WD;
            const double* Go = Wb + SLOT_WD + GD;
            // z = zraw - G[t, t-1] d_{t-1}
            double zdot = (lane < nb) ? zraw[32 * (t & 1) + lane] : 0.0;
            if (t > 0 && lane < nb) {
              const double* dp = dfull + 32 * ((t - 1) & 1);
              const int nbp = bk.nbp;
              double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
              int i = 0;
              for (; i + 4 <= nbp; i += 4) {
                c0 = fma(Go[i * nb + lane], dp[i], c0);
                c1 = fma(Go[(i + 1) * nb + lane], dp[i + 1], c1);
                c2 = fma(Go[(i + 2) * nb + lane], dp[i + 2], c2);
                c3 = fma(Go[(i + 3) * nb + lane], dp[i + 3], c3);
              }
              for (; i < nbp; ++i) c0 = fma(Go[i * nb + lane], dp[i], c0);
              zdot = __dsub_rn(zdot, (c0 + c1) + (c2 + c3));
            }
            // the block's cyclic updates (elastic_net.py:137-156)
            double dc = 0.0;
            for (int k = 0; k < nb; ++k) {
              const double zk = __shfl_sync(0xffffffffu, zdot, k);
              const double b_old = __shfl_sync(0xffffffffu, bc, k);
              const double cs = __shfl_sync(0xffffffffu, csc, k);
              const double inv = __shfl_sync(0xffffffffu, invc, k);
              const double dn = __dadd_rn(cs, lam2);
              const double z = __dadd_rn(__dmul_rn(cs, b_old), zk);
              const double np_ = __dsub_rn(z, lam1), nn_ = __dadd_rn(z, lam1);
              const double qp = __dmul_rn(np_, inv), qn = __dmul_rn(nn_, inv);
              const double bp = fma(fma(-qp, dn, np_), inv, qp);
              const double bn = fma(fma(-qn, dn, nn_), inv, qn);
              const double b_new = np_ > 0.0 ? bp : (nn_ < 0.0 ? bn : 0.0);
              const double d = __dsub_rn(b_new, b_old);
              if (lane == k) {
                bc = b_new;
                dc = d;
              }
              const double gk = (lane < nb) ? Gd[k * nb + lane] : 0.0;  // G symmetric: column k
              zdot = fma(-d, gk, zdot);
              const double ad = fabs(d);
              max_delta = ad > max_delta ? ad : max_delta;
            }
            // steps by column (solver's correction next step) and compacted to the
            // nonzero ones for the workers' AXPY (d == 0 leaves r unchanged)
            dfull[32 * (t & 1) + lane] = (lane < nb) ? dc : 0.0;
            {
              const unsigned nzm = __ballot_sync(0xffffffffu, lane < nb && dc != 0.0);
              if (lane < nb && dc != 0.0) {
                const int pos = __popc(nzm & ((1u << lane) - 1u));
                dd[32 * (t & 1) + pos] = dc;
                nzi[32 * (t & 1) + pos] = lane;
              }
              if (lane == 0) enz[t & 1] = __popc(nzm);
            }
            if (lane < nb) {
              betas[bk.j0 + lane] = bc;
              const double ab = fabs(bc);
              acc_l1 += ab;
              acc_l2 = fma(bc, bc, acc_l2);
              acc_max = fmax(acc_max, ab);
            }
            int stop = 0;
            if (b == nblk - 1) {  // sweep complete: the reference's stop rule (elastic_net.py:158)
              const double l1 = warp_sum(acc_l1), l2 = warp_sum(acc_l2), mabs = warp_max(acc_max);
              const double md = warp_max(max_delta);
              const int sw = static_cast<int>(t / nblk);
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
          } else if (lane == 0) {
            ctl[2 + (t & 1)] = 1;
          }
        } else {
          // workers: r -= W_{t-1} d_{t-1}, then (unless stopped) the dots of t+1
          if (t > 0) {
            const uint32_t e = t - 1;
            axpy_nz(slot_of(e), dd + 32 * (e & 1), nzi + 32 * (e & 1), enz[e & 1], par + 32 * (e & 3));
          }
          if (warp == NWK && !stopped && t + 2 < total) {
            publish((t + 2) & 3);                             // packed at step t-1
            pack_raw();                                       // element t+3 (raw loads of step t-1)
            if (t + 4 < total) pfetch_d(pd);                  // element t+4's columns (descriptor of step t-1)
            if (t + 5 < total) pd = blk[(t + 5) % nblk];      // element t+5's descriptor
          }
          worker_bar();  // rs current, parameters of t+2 published
          if (!stopped && t + 1 < total) {
            const uint32_t e = t + 1;
            wait_next();
            const double* Wb = slot_of(e);
            const int* pk = par + 32 * (e & 3);
            for (int j = warp - 1; j < enb[e & 3]; j += NWK) {
              const double z = col_dot(Wb, pk[j], false);
              if (lane == 0) zraw[32 * (e & 1) + j] = z;
            }
          }
          if (t > 0 && (t - 1) % nblk == static_cast<uint32_t>(nblk - 1)) {
            // the AXPY above completed sweep sw: its residual sum of squares
            const int sw = static_cast<int>((t - 1) / nblk);
            double rr = fma(r[0], r[0], fma(r[1], r[1], fma(r[2], r[2], r[3] * r[3])));
            rr = warp_sum(rr);
            if (lane == 0) red[16 + 8 * (sw & 1) + warp - 1] = rr;
          }
        }
        cta_bar();  // end of step t
        if (t > 0 && (t - 1) % nblk == static_cast<uint32_t>(nblk - 1) && tid == 32) {
          const int sw = static_cast<int>((t - 1) / nblk);
          double rss = 0.0;
#pragma unroll
          for (int w = 0; w < NWK; ++w) rss += red[16 + 8 * (sw & 1) + w];
          const double obj = __dadd_rn(__dadd_rn(__dmul_rn(0.5, rss), __dmul_rn(lam1, red[8 + 2 * (sw & 1)])),
                                       __dmul_rn(__dmul_rn(0.5, lam2), red[9 + 2 * (sw & 1)]));
          if (a.hist != nullptr) a.hist[a.hist_off[s] + sw] = obj;
          red[12] = obj;
        }
        if (stopped) break;  // this was the drain step (the final AXPY)
        if (q < total && ctl[2 + (t & 1)] == 0) {  // refill the slot of element t-1
          issue(q, true, static_cast<int>((q + 1) % nblk));
          ++q;
        }
      }
      if (max_iters == 0) {
        // objective at the given beta (prologue residual)
        double rr = 0.0, q1 = 0.0, q2 = 0.0;
        if (!solver) rr = fma(r[0], r[0], fma(r[1], r[1], fma(r[2], r[2], r[3] * r[3])));
        for (int j = tid; j < M; j += NT) {
          const double bj = betas[j];
          q1 += fabs(bj);
          q2 = fma(bj, bj, q2);
        }
        rr = warp_sum(rr);
        q1 = warp_sum(q1);
        q2 = warp_sum(q2);
        if (lane == 0) {
          zraw[warp] = rr;
          zraw[16 + warp] = q1;
          dd[warp] = q2;
        }
        cta_bar();
        if (tid == 32) {
          double rss = 0.0, t1 = 0.0, t2 = 0.0;
          for (int w = 0; w < NWK + 1; ++w) {
            rss += zraw[w];
            t1 += zraw[16 + w];
            t2 += dd[w];
          }
          red[12] = __dadd_rn(__dadd_rn(__dmul_rn(0.5, rss), __dmul_rn(lam1, t1)), __dmul_rn(__dmul_rn(0.5, lam2), t2));
        }
      }
      // observe every element issued beyond the stop (at most STAGES - 1 behind)
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
  const size_t smem = static_cast<size_t>(STAGES) * (SLOT_WD + 2 * GMAX * GMAX) * 8 + (1024 + 64 * 3 + 32) * 8 +
                      (128 + 4 + 64 + 2 + 10) * 4 + 8 * STAGES + 16;
  auto kernel = cd_block_kernel<SLOT_WD, GMAX, MINB>;
  PAM_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  PAM_CUDA_CHECK(cudaMemsetAsync(a.queue, 0, sizeof(unsigned), stream));
  const int64_t ctas = std::max<int64_t>(1, std::min<int64_t>(static_cast<int64_t>(MINB) * sm_count(), a.S));
  kernel<<<(unsigned)ctas, NT, smem, stream>>>(a, static_cast<unsigned char*>(block_ws));
  PAM_LAUNCH_CHECK("cd_block_kernel");
  return PAM_OK;
}

// <= 2 fits per SM: one CTA per SM (C3's 256 fits in two waves measured
// faster than two CTAs per SM with half the slot), 4 x (44 KB W + 2 x 2 KB
// Gram) slots, blocks of up to 16 columns (a BASELINE C2/C3 column is ~5 KB of
// tiles, so the W slot decides); more fits: two CTAs per SM, 4 x (20 KB + 4 KB).
int launch_cd_block(const CdArgs& a, int max_rows, void* block_ws, cudaStream_t stream) {
  if (max_rows > 1024 || block_ws == nullptr) return PAM_ERR_UNSUPPORTED;
  if (a.S <= 2 * sm_count()) return launch_block_pipe_cfg<5632, 16, 1>(a, block_ws, stream);
  return launch_block_pipe_cfg<2560, 16, 2>(a, block_ws, stream);
}

}  // namespace pam
