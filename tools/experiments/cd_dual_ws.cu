// ARCHIVED EXPERIMENT (not built into libpam_b200.so).  Warp-specialised
// variant of cd_dual_kernel, measured on C4 (one B200, same box A/B):
// CD 10.65 s (nanosleep backoff) / 10.52 s (busy polling) per step vs 8.27 s
// for cd_dual_kernel; bit-identical results (parity tests were green).  The
// single producer warp adds a polling hop between a slot's release and its
// refill and serialises 16 streams' copy issue; with a 3-slot ring (the
// shared-memory limit at 16 fits per SM) that latency reaches the consumers,
// so even the HBM-bound round 0 slowed from 1.89 to 2.35 s.  See DESIGN.md §3.
// To rebuild: add it to build_native.SOURCES and restore launch_cd_dual_ws in
// cd_common.cuh / PAM_CD_DUALWS in cd.cu.
// cd_dual_ws.cu — the two-fits-per-warp tile CD (cd_dual_kernel, cd.cu) with
// WARP SPECIALISATION: 8 consumer warps (16 fits per SM, the C4 load) do only
// the coordinate updates; one producer warp issues every bulk copy of the
// CTA's 16 column streams.
//
// Why (profiles/r01_ncu_cd_dual_round1_raw.csv): in rounds 1-2
// of C4 the dual kernel is bound by each warp's per-column instruction
// stream, and 35 % of its stall samples sat in the divergent refill block
// (lanes 0/16 each issuing their half's copy: branch, expect_tx, bulk copy,
// reconvergence) on every column.  Here a consumer releases a ring slot with
// ONE non-divergent instruction (mbarrier.arrive by all 32 lanes on the
// slot's "empty" barrier) and never issues copies; the producer lanes (lane w
// <-> consumer warp w) poll the empty barriers, read the column's packed
// offset and run code from a per-warp parameter block the consumer publishes
// one 16-column chunk ahead, and issue both halves' copies against the slot's
// "full" barrier (one arrive.expect_tx with the summed bytes).
//
// The arithmetic per fit is exactly cd_dual_kernel's (same loads, same dot
// order, same soft threshold), so the results are bit-identical to it; the
// column stream of a pair is [prologue Mx] + mix * Mx as there.  Handshakes
// (shared memory, volatile + block fences): a consumer publishes each pair's
// descriptor (pair_seq), each chunk's issue parameters (pub_seq) and clears a
// half's `live` flag when it converges (its later columns carry no data); at
// the end of a pair it raises stop_req, the producer answers with the number
// of stream positions it issued (issued_end, stop_ack), and the consumer
// drains the speculative ones.  Stream positions count continuously across
// pairs, so every barrier parity is position / STAGES.
#include "cd_common.cuh"

#include <algorithm>

namespace pam {

constexpr int WS_NCW = 8;  // consumer warps (2 fits each) = warpgroups 0-1
constexpr int WS_THREADS = (WS_NCW + 4) * 32;  // + producer warpgroup (warp 8 works, 9-11 exit)

struct WsCtl {  // per consumer warp, in shared memory
  volatile int pair_seq;   // consumer: descriptor of pair pair_seq is valid
  volatile int pub_seq;    // consumer: issue parameters of chunks <= pub_seq are valid
  volatile int stop_req;   // consumer: pair stop_req is finished
  volatile int stop_ack;   // producer: acknowledged stop_req
  volatile int issued_end; // producer: stream positions issued up to the stop
  volatile int live[2];    // consumer: half still needs data
  volatile int terminal;   // consumer: no more pairs
  volatile int Mx, mix;
  volatile int M[2];
  volatile long long woff[2];  // W offset (doubles) of each half's fit
};

__device__ __forceinline__ void mbar_arrive_dep(uint32_t bar, double dep) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n\t// dep %1" ::"r"(bar), "d"(dep) : "memory");
}

template <int R, int STAGES>
__global__ void __launch_bounds__(WS_THREADS, 1) cd_dual_ws_kernel(const CdArgs a) {
  constexpr int SLOTH = R * 16;  // doubles per half slot
  constexpr int PBLK = 128;      // doubles per consumer warp: pb/pc/pinv[32] + pk[32] (int)
  constexpr uint32_t SLOT_B = 2u * SLOTH * 8u;
  static_assert(R % 2 == 0 && R <= 32 && STAGES <= 8, "dual tile CD envelope");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  double* const ring_all = reinterpret_cast<double*>(smem_raw);
  uint64_t* const full = reinterpret_cast<uint64_t*>(ring_all + static_cast<size_t>(WS_NCW) * STAGES * 2 * SLOTH);
  uint64_t* const empty = full + WS_NCW * STAGES;
  double* const pblk = reinterpret_cast<double*>(empty + WS_NCW * STAGES);
  int* const iprm = reinterpret_cast<int*>(pblk + WS_NCW * PBLK);  // [NCW][2 buffers][off 32 | code 32]
  WsCtl* const ctl = reinterpret_cast<WsCtl*>(iprm + WS_NCW * 2 * 64);
  double* const zero_blk = reinterpret_cast<double*>(ctl + WS_NCW);
  const uint32_t full_s = smem_u32(full), empty_s = smem_u32(empty);

  for (int i = threadIdx.x; i < SLOTH; i += WS_THREADS) zero_blk[i] = 0.0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < WS_NCW * STAGES; ++i) {
      mbar_init(&full[i], 1);    // the producer's arrive(.expect_tx)
      mbar_init(&empty[i], 32);  // every lane of the consumer warp
    }
    fence_mbar_init();
  }
  for (int w = threadIdx.x; w < WS_NCW; w += WS_THREADS) {
    ctl[w].pair_seq = 0;
    ctl[w].pub_seq = -1;
    ctl[w].stop_req = 0;
    ctl[w].stop_ack = 0;
    ctl[w].terminal = 0;
  }
  __syncthreads();

  // register split (launch: 168 per thread): the producer warpgroup gives
  // registers back, the consumer warpgroups take 232 each (8*32*232 + 4*32*40
  // <= 64 K)
  if (warp >= WS_NCW) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    if (warp != WS_NCW) return;
    // ======================= producer: lane w serves consumer warp w
    const int w = lane;
    const bool mine = w < WS_NCW;
    int state = mine ? 0 : 2;  // 0 wait pair, 1 issue, 2 done
    int seen = 0;              // last pair sequence taken
    int gpos = 0;              // stream positions issued (running)
    int lpos = 0, total = 0, Mx = 1, nch = 1, Ms0 = 0, Ms1 = 0;
    long long wo0 = 0, wo1 = 0;
    const uint32_t ring_w = smem_u32(ring_all + static_cast<size_t>(mine ? w : 0) * STAGES * 2 * SLOTH);
    const volatile int* ip = iprm + (mine ? w : 0) * 128;
    WsCtl& c = ctl[mine ? w : 0];
    while (__any_sync(0xffffffffu, state != 2)) {
      bool progress = false;
      if (state == 0) {
        if (c.terminal) {
          state = 2;
        } else if (c.pair_seq > seen) {
          __threadfence_block();
          seen = c.pair_seq;
          Mx = c.Mx;
          nch = (Mx + 15) >> 4;
          total = Mx * (1 + c.mix);
          Ms0 = c.M[0];
          Ms1 = c.M[1];
          wo0 = c.woff[0];
          wo1 = c.woff[1];
          lpos = 0;
          state = 1;
          progress = true;
        }
      } else if (state == 1) {
        if (c.stop_req == seen) {
          c.issued_end = gpos;
          __threadfence_block();
          c.stop_ack = seen;
          state = 0;
          progress = true;
        } else if (lpos < total) {
          const int stg = gpos % STAGES;
          const bool free_slot = gpos < STAGES || mbar_test_s(empty_s + (w * STAGES + stg) * 8,
                                                              static_cast<uint32_t>((gpos / STAGES - 1) & 1));
          const int col = lpos % Mx;
          const int g = (lpos / Mx) * nch + (col >> 4);
          if (free_slot && c.pub_seq >= g) {
            __threadfence_block();
            const volatile int* buf = ip + (g & 1) * 64;
            const int cc = col & 15;
            const int code0 = (c.live[0] && col < Ms0) ? buf[32 + cc] : 0;
            const int code1 = (c.live[1] && col < Ms1) ? buf[32 + 16 + cc] : 0;
            const uint32_t b0 = static_cast<uint32_t>(code_tiles(code0)) * 256u;
            const uint32_t b1 = static_cast<uint32_t>(code_tiles(code1)) * 256u;
            const uint32_t bar = full_s + (w * STAGES + stg) * 8;
            if (b0 + b1) {
              mbar_expect_s(bar, b0 + b1);
              if (b0) bulk_g2s(ring_w + stg * SLOT_B, a.W + wo0 + buf[cc], b0, bar);
              if (b1) bulk_g2s(ring_w + stg * SLOT_B + SLOTH * 8, a.W + wo1 + buf[16 + cc], b1, bar);
            } else {
              mbar_arrive_s(bar);
            }
            ++gpos;
            ++lpos;
            progress = true;
          }
        }
      }
      (void)progress;  // busy polling (a __nanosleep(64) backoff measured 10.65 s CD at C4)
    }
    return;
  }

  // ========================= consumers: two fits per warp (cd_dual_kernel)
  asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");
  const int half = lane >> 4;
  const int hl = lane & 15;
  const int hb = half * 16;
  double* const pb = pblk + warp * PBLK;
  double* const pc = pb + 32;
  double* const pinv = pb + 64;
  int* const pk = reinterpret_cast<int*>(pb + 96);
  int* const ipw = iprm + warp * 128;
  WsCtl& c = ctl[warp];
  const uint32_t ring_h = smem_u32(ring_all + static_cast<size_t>(warp) * STAGES * 2 * SLOTH) + half * (SLOTH * 8);
  const uint32_t fbar = full_s + warp * STAGES * 8, ebar = empty_s + warp * STAGES * 8;
  const uint32_t zero_s = smem_u32(zero_blk) + 16u * hl;

  int gpos = 0;  // stream positions consumed (running across pairs)
  int pair_seq = 0;
  const int64_t P = (a.S + 1) / 2;
  unsigned item = warp * gridDim.x + blockIdx.x;
  const unsigned total_warps = gridDim.x * WS_NCW;

  while (true) {
    if (item >= P) {
      __syncwarp();
      if (lane == 0) c.terminal = 1;
      break;
    }
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
    const int nch = (Mx + 15) >> 4;

    double r[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int p = 32 * (k >> 1) + 2 * hl + (k & 1);
      const int row = a.perm ? (p < N ? a.perm[r0 + p] : 0) : p;
      r[k] = (p < N) ? a.y[r0 + row] : 0.0;
    }

    // issue parameters of chunk g (pass g / nch, columns 16 (g % nch) ..) into
    // buffer g & 1; the global loads are made one chunk ahead (registers)
    int pf_off = 0;
    unsigned long long pf_mk = 0ull;
    auto prefetch_chunk = [&](int g) {
      const int col = 16 * (g % nch) + hl;
      pf_off = (col < M) ? static_cast<int>(colo[col]) : 0;
      pf_mk = (col < M) ? tmk[col] : 0ull;
    };
    auto publish_chunk = [&](int g) {
      volatile int* buf = ipw + (g & 1) * 64;
      buf[hb + hl] = pf_off;
      buf[32 + hb + hl] = tile_code(pf_mk);
      __syncwarp();
      __threadfence_block();
      if (lane == 0) c.pub_seq = g;
      prefetch_chunk(g + 1);
    };
    // pair descriptor for the producer (issue parameters of chunk 0 first)
    prefetch_chunk(0);
    publish_chunk(0);
    if (hl == 0) {
      c.live[half] = hvalid ? 1 : 0;
      c.M[half] = M;
      c.woff[half] = hvalid ? a.w_off[sx] : 0;
    }
    __syncwarp();
    if (lane == 0) {
      c.Mx = Mx;
      c.mix = mix;
      __threadfence_block();
      c.pair_seq = ++pair_seq;
    } else {
      ++pair_seq;
    }
    int chunk_g = 0;  // chunk of the next consumed position

    // ---- consumer side
    bool ready = false;
    double w[R];
    auto load_w = [&](int code) {
      const int st = gpos % STAGES;
      if (!ready) mbar_wait_s(fbar + st * 8, static_cast<uint32_t>((gpos / STAGES) & 1));
      const int a0 = code & 0xff, la = (code >> 8) & 0xff;
      const uint32_t cA = ring_h + st * SLOT_B + 16u * hl - 256u * a0;
#pragma unroll
      for (int q = 0; q < R / 2; ++q) {
        const bool inA = static_cast<unsigned>(q - a0) < static_cast<unsigned>(la);
        lds_v2((inA ? cA : zero_s) + 256u * q, w[2 * q], w[2 * q + 1]);
      }
    };
    // the column of position gpos is in registers: release its slot (every
    // lane arrives, ordered after its loads by `dep`) and look at the next one
    auto advance = [&](double dep) {
      mbar_arrive_dep(ebar + (gpos % STAGES) * 8, dep);
      ++gpos;
      ready = mbar_test_s(fbar + (gpos % STAGES) * 8, static_cast<uint32_t>((gpos / STAGES) & 1));
    };
    // at the first column of each chunk: publish the NEXT chunk's issue parameters
    auto chunk_start = [&]() {
      publish_chunk(chunk_g + 1);
      ++chunk_g;
    };

    // prologue: col_sq (elastic_net.py:85) and r = y - W beta0 (elastic_net.py:94)
    for (int cb = 0; cb < Mx; cb += 16) {
      const int nc = min(16, Mx - cb);
      chunk_start();
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
    unsigned long long nk_mk = 0ull;
    auto fetch_params = [&](int cb) {
      const int col = cb + hl;
      nb_l = (col < M) ? betas[col] : 0.0;
      ncs_l = (col < M) ? colsq[col] : 0.0;
      nk_mk = (col < M) ? tmk[col] : 0ull;
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
        chunk_start();
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
          const double dn = __dadd_rn(cs, lam2);
          const double dot = half_sum(part);
          const double z = __dadd_rn(cb_old, dot);
          const double np_ = __dsub_rn(z, lam1), nn_ = __dadd_rn(z, lam1);
          const double qp = __dmul_rn(np_, inv), qn = __dmul_rn(nn_, inv);
          const double bp = fma(fma(-qp, dn, np_), inv, qp);
          const double bn = fma(fma(-qn, dn, nn_), inv, qn);
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
          if (hl == 0) c.live[half] = 0;  // later stream positions of this half carry no data
        }
      }
    }
    const bool zero_it = hvalid && mi == 0;
    if (__any_sync(0xffffffffu, zero_it)) {
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
    // stop the producer, then drain the positions it issued speculatively
    __syncwarp();
    if (lane == 0) c.stop_req = pair_seq;
    while (c.stop_ack != pair_seq) {
    }
    __threadfence_block();
    const int end = c.issued_end;
    while (gpos < end) {
      mbar_wait_s(fbar + (gpos % STAGES) * 8, static_cast<uint32_t>((gpos / STAGES) & 1));
      mbar_arrive_dep(ebar + (gpos % STAGES) * 8, 0.0);
      ++gpos;
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

int launch_cd_dual_ws(const CdArgs& a, cudaStream_t stream) {
  constexpr int R = 32, STAGES = 3;
  constexpr int SLOTH = R * 16;
  const size_t smem = static_cast<size_t>(WS_NCW) * STAGES * 2 * SLOTH * 8 + 2 * WS_NCW * STAGES * 8 +
                      WS_NCW * 128 * 8 + WS_NCW * 2 * 64 * 4 + WS_NCW * sizeof(WsCtl) + SLOTH * 8;
  auto kernel = cd_dual_ws_kernel<R, STAGES>;
  PAM_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  PAM_CUDA_CHECK(cudaMemsetAsync(a.queue, 0, sizeof(unsigned), stream));
  const int64_t pairs = (a.S + 1) / 2;
  const int64_t ctas = std::max<int64_t>(1, std::min<int64_t>(sm_count(), pairs));
  kernel<<<(unsigned)ctas, WS_THREADS, smem, stream>>>(a);
  PAM_LAUNCH_CHECK("cd_dual_ws_kernel");
  return PAM_OK;
}

}  // namespace pam
