// Microbenchmark: HBM bandwidth of per-warp TMA bulk-copy streams vs request size.
// 148 CTAs x 16 warps, each warp streams its own contiguous region through a
// 3-slot shared-memory ring (the CD kernel's staging pattern), touching the
// data with one shared load per lane so the copies cannot be elided.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_rs tma_request_size.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(512, 1) stream_kernel(const double* src, size_t per_warp_bytes, int req_bytes,
                                                        int stages, double* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot_bytes = 4096;
  unsigned char* ring = sm + (size_t)warp * stages * slot_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + (size_t)16 * stages * slot_bytes) + warp * stages;
  if (lane == 0) {
    for (int i = 0; i < stages; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  const size_t gw = (size_t)blockIdx.x * 16 + warp;
  const char* base = reinterpret_cast<const char*>(src) + gw * per_warp_bytes;
  const long n = (long)(per_warp_bytes / req_bytes);
  long issued = 0;
  auto issue = [&](long i) {
    if (lane == 0) {
      const int st = (int)(i % stages);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bars[st])), "r"(req_bytes));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su32(ring + st * slot_bytes)),
                   "l"(base + i * req_bytes), "r"(req_bytes), "r"(su32(&bars[st]))
                   : "memory");
    }
  };
  for (; issued < stages && issued < n; ++issued) issue(issued);
  double acc = 0.0;
  for (long i = 0; i < n; ++i) {
    const int st = (int)(i % stages);
    const uint32_t par = (uint32_t)((i / stages) & 1);
    uint32_t ok = 0;
    do {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                   : "=r"(ok) : "r"(su32(&bars[st])), "r"(par) : "memory");
    } while (!ok);
    const double* d = reinterpret_cast<const double*>(ring + st * slot_bytes);
    for (int k = lane; k < req_bytes / 8; k += 32) acc += d[k];
    __syncwarp();
    if (issued < n) issue(issued++);
  }
  if (acc == 12345.678) sink[0] = acc;
}

int main() {
  const size_t total = (size_t)12 << 30;  // 12 GB streamed per pass
  const int warps = 148 * 16;
  double* src;
  double* sink;
  cudaMalloc(&src, total);
  cudaMemset(src, 0, total);
  cudaMalloc(&sink, 8);
  const int stages = 3;
  const size_t smem = (size_t)16 * stages * 4096 + 16 * stages * 8;
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int sizes[] = {256, 512, 1024, 1536, 2048, 2560, 3072, 4096};
  for (int s : sizes) {
    size_t per = (total / warps) / s * s;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    stream_kernel<<<148, 512, smem>>>(src, per, s, stages, sink);
    cudaEventRecord(a);
    for (int rep = 0; rep < 3; ++rep) stream_kernel<<<148, 512, smem>>>(src, per, s, stages, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"req_bytes\": %d, \"stages\": %d, \"GBs\": %.1f}\n", s, stages, 3.0 * per * warps / (ms * 1e-3) / 1e9);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
