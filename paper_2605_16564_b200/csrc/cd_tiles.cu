// cd_tiles.cu — K2b over tile-packed design matrices with a BYTE ring.
//
// Same coordinate descent as cd.cu (reference elastic_net.py:113-161: cyclic
// order, soft threshold, true division, stop rule, per-sweep objective) over
// the tile-packed columns produced by tiles.cu.  The difference is the
// staging buffer: tile-packed columns have variable size (popcount(mask) x
// 256 B, ~2 KB on average at C4 instead of 4 KB dense), and the kernel is
// bound by the BYTES IN FLIGHT per SM (Little's law against the loaded HBM
// latency, measured: a fixed 3-slot ring reached only 68% of HBM).  So each
// warp owns a byte ring of RB doubles and keeps issuing cp.async.bulk copies
// until the ring or its NB mbarriers are full: ~2x more columns in flight
// for the same shared memory, i.e. the same ~190 KB/SM in flight as the
// dense stream that saturates HBM.
//
// Ring rule (replayed identically by producer and consumer, so the consumer
// never needs the producer's addresses): a column of nd doubles starts at the
// current physical position p unless p + nd > RB, in which case it starts at
// 0 and the RB - p tail is wasted; the producer may issue while the doubles
// held by unreleased columns (plus waste) stay <= RB and fewer than NB
// columns are in flight.  All positions are 32-bit, no modulo arithmetic.
#include "pam_common.cuh"

#include <stdlib.h>

#include <algorithm>

namespace pam {

__device__ unsigned int g_cdt_queue;

struct CdTilesArgs {
  int64_t S;
  const int64_t* order;
  const int64_t* row_off;
  const double* y;
  const int32_t* perm;
  const int64_t* dict_off;
  const int32_t* m_cur;
  const int64_t* w_off;
  const unsigned long long* tile_mask;
  const int64_t* col_off;
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
};

// R: 32-row tiles per column (<= 32); RB: ring doubles per warp; NB: mbarriers per warp
template <int R, int WPC, int RB, int NB>
__global__ void __launch_bounds__(WPC * 32, 1) cd_tiles_kernel(const CdTilesArgs a) {
  static_assert(R <= 32, "32-bit tile masks");
  static_assert(RB >= 32 * R, "a full column must fit the ring");
  static_assert((NB & (NB - 1)) == 0, "NB must be a power of two");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  double* ring = reinterpret_cast<double*>(smem_raw) + static_cast<size_t>(warp) * RB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<double*>(smem_raw) + WPC * RB) +
                   warp * NB;
  if (lane == 0) {
    for (int b = 0; b < NB; ++b) mbar_init(&bars[b], 1);
    fence_mbar_init();
    fence_proxy_async_smem();
  }
  __syncwarp();

  uint32_t seq_issue = 0, seq_cons = 0;  // running column counters (barrier = seq % NB)
  const unsigned total_warps = gridDim.x * WPC;
  unsigned item = warp * gridDim.x + blockIdx.x;

  while (item < a.S) {
    const int64_t s = a.order ? a.order[item] : static_cast<int64_t>(item);
    if (a.active == nullptr || a.active[s] != 0) {
      const int64_t r0 = a.row_off[s];
      const int N = static_cast<int>(a.row_off[s + 1] - r0);
      const int M = a.m_cur[s];
      const int64_t doff = a.dict_off[s];
      const double* Ws = a.W + a.w_off[s];
      const double lam1 = a.lam1[s], lam2 = a.lam2[s], tol = a.tol[s];
      const int max_iters = a.max_iters[s];

      double r[R];
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const int p = lane + 32 * k;
        const int row = a.perm ? (p < N ? a.perm[r0 + p] : 0) : p;
        r[k] = (p < N) ? a.y[r0 + row] : 0.0;
      }

      // producer state (physical ring positions, 32-bit, no modulo)
      const int64_t total = (int64_t)(max_iters + 1) * M;  // prologue pass + sweeps
      int64_t issued = 0;
      int p_col = 0;
      int p_phys = 0;   // physical start of the next column
      int in_use = 0;   // doubles held by unreleased columns, including wrap waste
      int iss_base = -64;
      int iss_off_l = 0;
      unsigned iss_mask_l = 0u;
      // consumer state (replays the placement rule)
      int c_phys = 0;
      int64_t consumed = 0;

      auto try_issue = [&]() {
        while (issued < total && (seq_issue - seq_cons) < (uint32_t)NB) {
          const int cbase = p_col & ~31;
          if (cbase != iss_base) {  // warp-uniform reload of 32 columns' packing
            iss_base = cbase;
            const int c = cbase + lane;
            iss_off_l = (c < M) ? static_cast<int>(a.col_off[doff + c]) : 0;
            iss_mask_l = (c < M) ? static_cast<unsigned>(a.tile_mask[doff + c]) : 0u;
          }
          const unsigned mk = __shfl_sync(0xffffffffu, iss_mask_l, p_col & 31);
          const int nd = 32 * __popc(mk);
          const bool wrap = p_phys + nd > RB;  // (p_phys == RB wraps even with zero waste)
          const int waste = wrap ? RB - p_phys : 0;
          if (in_use + waste + nd > RB) break;  // ring full until the consumer releases
          const int start = wrap ? 0 : p_phys;
          const int off = __shfl_sync(0xffffffffu, iss_off_l, p_col & 31);
          if (lane == 0) {
            uint64_t* bar = &bars[seq_issue & (NB - 1)];
            if (nd) {
              mbar_arrive_expect_tx(bar, static_cast<uint32_t>(nd) * sizeof(double));
              tma_load_1d(ring + start, Ws + off, static_cast<uint32_t>(nd) * sizeof(double), bar);
            } else {
              mbar_arrive(bar);
            }
          }
          p_phys = start + nd;
          in_use += waste + nd;
          ++seq_issue;
          ++issued;
          if (++p_col == M) p_col = 0;
        }
      };
      // consume the next column (mask mk): returns its smem base; release() after use
      int cur_nd = 0, cur_free = 0;
      auto acquire = [&](unsigned mk) -> const double* {
        cur_nd = 32 * __popc(mk);
        const bool wrap = c_phys + cur_nd > RB;
        const int waste = wrap ? RB - c_phys : 0;
        const int start = wrap ? 0 : c_phys;
        cur_free = waste + cur_nd;
        c_phys = start + cur_nd;
        mbar_wait(&bars[seq_cons & (NB - 1)], (seq_cons / NB) & 1u);
        return ring + start;
      };
      auto release = [&]() {
        __syncwarp();
        in_use -= cur_free;
        ++seq_cons;
        ++consumed;
        try_issue();
      };

      double w[R];
      auto load_col = [&](const double* col, unsigned mk) {
        int slot = 0;
#pragma unroll
        for (int g = 0; g < (R + 3) / 4; ++g) {
          const int cnt = (4 * g + 4 <= R) ? 4 : (R - 4 * g);
          const unsigned full = (1u << cnt) - 1u;
          const unsigned nib = (mk >> (4 * g)) & full;
          if (nib == full) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (u < cnt) w[4 * g + u] = col[32 * (slot + u) + lane];
            slot += cnt;
          } else if (nib == 0u) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (u < cnt) w[4 * g + u] = 0.0;
          } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              if (u < cnt) {
                const int bit = static_cast<int>((nib >> u) & 1u);
                const double v = col[32 * min(slot, R - 1) + lane];
                w[4 * g + u] = bit ? v : 0.0;
                slot += bit;
              }
            }
          }
        }
      };

      try_issue();

      // ---- prologue: col_sq (elastic_net.py:85) and r = y - W beta0 (94)
      for (int cb = 0; cb < M; cb += 32) {
        const int nc = min(32, M - cb);
        const unsigned ml = (lane < nc) ? static_cast<unsigned>(a.tile_mask[doff + cb + lane]) : 0u;
        for (int t = 0; t < nc; ++t) {
          const int j = cb + t;
          const unsigned mk = __shfl_sync(0xffffffffu, ml, t);
          const double* col = acquire(mk);
          load_col(col, mk);
          double p = 0.0;
#pragma unroll
          for (int k = 0; k < R; ++k) p = fma(w[k], w[k], p);
          p = warp_sum(p);
          if (lane == 0) a.col_sq[doff + j] = p;
          const double b0 = a.beta[doff + j];
          if (b0 != 0.0) {
#pragma unroll
            for (int k = 0; k < R; ++k) r[k] = fma(-b0, w[k], r[k]);
          }
          release();
        }
      }
      __syncwarp();

      // ---- sweeps (elastic_net.py:137-161)
      int sweeps_done = 0, conv = 0;
      double obj = 0.0;
      for (int sw = 0; sw < max_iters; ++sw) {
        double max_delta = 0.0, acc_l1 = 0.0, acc_l2 = 0.0, acc_max = 0.0;
        for (int cb = 0; cb < M; cb += 32) {
          const int nc = min(32, M - cb);
          double bl = 0.0, csl = 0.0;
          unsigned ml = 0u;
          if (lane < nc) {
            bl = a.beta[doff + cb + lane];
            csl = a.col_sq[doff + cb + lane];
            ml = static_cast<unsigned>(a.tile_mask[doff + cb + lane]);
          }
          for (int t = 0; t < nc; ++t) {
            const unsigned mk = __shfl_sync(0xffffffffu, ml, t);
            const double* col = acquire(mk);
            load_col(col, mk);
            double d0 = 0.0, d1 = 0.0;
#pragma unroll
            for (int k = 0; k < R; ++k) {
              if (k & 1) d1 = fma(w[k], r[k], d1);
              else d0 = fma(w[k], r[k], d0);
            }
            const double dot = warp_sum(d0 + d1);
            const double b_old = __shfl_sync(0xffffffffu, bl, t);
            const double cs = __shfl_sync(0xffffffffu, csl, t);
            const double dn = __dadd_rn(cs, lam2);
            const double z = __dadd_rn(__dmul_rn(cs, b_old), dot);
            double b_new = 0.0;
            if (dn > 0.0) {
              double mag = __dsub_rn(fabs(z), lam1);
              if (mag < 0.0) mag = 0.0;
              b_new = __ddiv_rn(z >= 0.0 ? mag : -mag, dn);
            }
            if (b_new != b_old) {
              const double d = __dsub_rn(b_new, b_old);
#pragma unroll
              for (int k = 0; k < R; ++k) r[k] = fma(-d, w[k], r[k]);
              if (lane == t) bl = b_new;
              max_delta = fmax(max_delta, fabs(d));
            }
            release();
          }
          if (lane < nc) {
            a.beta[doff + cb + lane] = bl;
            const double ab = fabs(bl);
            acc_l1 += ab;
            acc_l2 = fma(bl, bl, acc_l2);
            acc_max = fmax(acc_max, ab);
          }
        }
        double rss = 0.0;
#pragma unroll
        for (int k = 0; k < R; ++k) rss = fma(r[k], r[k], rss);
        rss = warp_sum(rss);
        const double l1 = warp_sum(acc_l1), l2 = warp_sum(acc_l2), mabs = warp_max(acc_max);
        obj = __dadd_rn(__dadd_rn(__dmul_rn(0.5, rss), __dmul_rn(lam1, l1)),
                        __dmul_rn(__dmul_rn(0.5, lam2), l2));
        sweeps_done = sw + 1;
        if (max_delta <= __dmul_rn(tol, fmax(mabs, 1.0))) {
          conv = 1;
          break;
        }
      }
      // drain copies of the sweep that will not run
      while (seq_cons < seq_issue) {
        mbar_wait(&bars[seq_cons & (NB - 1)], (seq_cons / NB) & 1u);
        ++seq_cons;
      }
      __syncwarp();
      if (lane == 0) {
        a.sweeps[s] = sweeps_done;
        a.converged[s] = conv;
        a.objective[s] = obj;
      }
    }
    unsigned nxt = 0;
    if (lane == 0) nxt = atomicAdd(&g_cdt_queue, 1u) + total_warps;
    item = __shfl_sync(0xffffffffu, nxt, 0);
  }
}

template <int R, int WPC, int RB, int NB>
int launch_cd_tiles(const CdTilesArgs& a, cudaStream_t stream) {
  const size_t smem = static_cast<size_t>(WPC) * (RB * sizeof(double) + NB * sizeof(uint64_t));
  static bool configured = false;
  if (!configured) {
    PAM_CUDA_CHECK(cudaFuncSetAttribute(cd_tiles_kernel<R, WPC, RB, NB>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = true;
  }
  int dev = 0, sms = 148;
  PAM_CUDA_CHECK(cudaGetDevice(&dev));
  PAM_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  void* qaddr = nullptr;
  PAM_CUDA_CHECK(cudaGetSymbolAddress(&qaddr, g_cdt_queue));
  PAM_CUDA_CHECK(cudaMemsetAsync(qaddr, 0, sizeof(unsigned), stream));
  const int64_t ctas = std::max<int64_t>(1, std::min<int64_t>(sms, a.S));
  cd_tiles_kernel<R, WPC, RB, NB><<<(unsigned)ctas, WPC * 32, smem, stream>>>(a);
  PAM_LAUNCH_CHECK("cd_tiles_kernel");
  return PAM_OK;
}

}  // namespace pam

using namespace pam;

// Byte-ring variant of pam_cd_tiles_f64 (same arguments); dispatched from
// cd.cu for tile-packed batches with <= 1024 rows per subdomain.
int pam_cd_tiles_ring(int64_t S, const int64_t* order, const int64_t* row_off, const double* y,
                      const int32_t* perm, const int64_t* dict_off, const int32_t* m_cur,
                      const int64_t* w_off, const uint64_t* tile_mask, const int64_t* col_off,
                      const double* W, const double* lam1, const double* lam2, const double* tol,
                      const int32_t* max_iters, const int32_t* active, int32_t max_rows,
                      double* beta, double* col_sq, int32_t* sweeps, int32_t* converged,
                      double* objective, void* stream) {
  CdTilesArgs a{S, order, row_off, y, perm, dict_off, m_cur, w_off,
                reinterpret_cast<const unsigned long long*>(tile_mask), col_off, W, lam1, lam2, tol,
                max_iters, active, beta, col_sq, sweeps, converged, objective};
  cudaStream_t st = as_stream(stream);
  // ring sized so WPC * RB doubles ~ 200 KB per SM; NB mbarriers per warp
  const char* env = getenv("PAM_RING_WPC");
  const int wpc = env ? atoi(env) : 16;
  if (max_rows <= 128) return launch_cd_tiles<4, 16, 1536, 16>(a, st);
  if (max_rows <= 256) return launch_cd_tiles<8, 16, 1536, 16>(a, st);
  if (max_rows <= 512) {
    if (wpc == 12) return launch_cd_tiles<16, 12, 2048, 16>(a, st);
    return launch_cd_tiles<16, 16, 1568, 16>(a, st);
  }
  if (max_rows <= 1024) return launch_cd_tiles<32, 8, 3136, 16>(a, st);
  return PAM_ERR_UNSUPPORTED;
}
