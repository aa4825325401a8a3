// pam_common.cuh — shared device helpers for the PAM sm_100a kernels.
//
// Numerics policy: every quantity that feeds a tie-sensitive
// decision (log-features exponents, nearest-entry distances, candidate
// positions, ownership) is computed with explicit round-to-nearest
// intrinsics (__dmul_rn/__dadd_rn/__dsub_rn) so nvcc cannot contract it into
// an FMA and the result is bit-identical to numpy's.  Everything else may use
// FMA freely.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>
#include <stdlib.h>

#include "../../include/pam_b200.h"

#ifndef PAM_WARP
#define PAM_WARP 32
#endif

namespace pam {

// ----------------------------------------------------------------------------
// host-side status plumbing
void set_last_error(const char* msg);
int cuda_status(cudaError_t e, const char* where);
#define PAM_CUDA_CHECK(expr)                                   \
  do {                                                         \
    cudaError_t _e = (expr);                                   \
    if (_e != cudaSuccess) return ::pam::cuda_status(_e, #expr); \
  } while (0)
#define PAM_LAUNCH_CHECK(where)                                        \
  do {                                                                 \
    cudaError_t _e = cudaGetLastError();                               \
    if (_e != cudaSuccess) return ::pam::cuda_status(_e, where);       \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ----------------------------------------------------------------------------
// device error word: err[0] = code (first writer wins), err[1] = min index
__device__ __forceinline__ void report_error(int64_t* err, int64_t code, int64_t idx) {
  if (err == nullptr) return;
  atomicMin(reinterpret_cast<unsigned long long*>(err + 1), static_cast<unsigned long long>(idx));
  atomicCAS(reinterpret_cast<unsigned long long*>(err), 0ull, static_cast<unsigned long long>(code));
}

// ----------------------------------------------------------------------------
// warp reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ----------------------------------------------------------------------------
// Exact Gaussian log-feature L = -(sum_k (x_k - c_k)^2) * inv
// with inv = 1 / (2 w^2) (rbf.py:87) and numpy-2.3 einsum summation order
// (rbf.py:90): 1D q0, 2D q0+q1, 3D (q0+q2)+q1.
__device__ __forceinline__ double inv_two_sigma_sq(double w) {
  return __ddiv_rn(1.0, __dmul_rn(2.0, __dmul_rn(w, w)));
}

template <int D>
__device__ __forceinline__ double sqdist_einsum(const double* x, const double* c) {
  if (D == 1) {
    double d0 = __dsub_rn(x[0], c[0]);
    return __dmul_rn(d0, d0);
  } else if (D == 2) {
    double d0 = __dsub_rn(x[0], c[0]);
    double d1 = __dsub_rn(x[1], c[1]);
    return __dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1));
  } else {
    double d0 = __dsub_rn(x[0], c[0]);
    double d1 = __dsub_rn(x[1], c[1]);
    double d2 = __dsub_rn(x[2], c[2]);
    return __dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d2, d2)), __dmul_rn(d1, d1));
  }
}

// np.sum((centers - p)**2, axis=1) order (adaptive.py:162): (q0+q1)+q2
template <int D>
__device__ __forceinline__ double sqdist_npsum(const double* c, const double* p) {
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    double d = __dsub_rn(c[k], p[k]);
    acc = (k == 0) ? __dmul_rn(d, d) : __dadd_rn(acc, __dmul_rn(d, d));
  }
  return acc;
}

template <int D>
__device__ __forceinline__ double log_feature(const double* x, const double* c, double inv) {
  return __dmul_rn(-sqdist_einsum<D>(x, c), inv);
}

// ----------------------------------------------------------------------------
// TMA bulk copy (cp.async.bulk) + mbarrier helpers (sm_90+/sm_100a)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// 32-bit shared-address variants used by the lean streaming kernels (cd.cu, gram.cu)
__device__ __forceinline__ void mbar_wait_s(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ bool mbar_test_s(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_expect_s(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive_s(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

// 16-byte shared load at a 32-bit shared address; volatile keeps it behind
// the mbarrier wait that published the data
__device__ __forceinline__ void lds_v2(uint32_t addr, double& x, double& y) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(addr));
}

// bulk copy whose issue waits on `dep` (a register computed from the shared
// loads of the destination slot): the async-proxy write cannot overtake them
__device__ __forceinline__ void bulk_g2s_dep(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                             double dep) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n\t"
      "// dep %4" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "d"(dep)
      : "memory");
}


inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace pam
