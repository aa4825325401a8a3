// lat_probe.cu — dependent-chain latencies of the instructions on the CD
// kernel's per-column critical path (one warp, clock64 around 1024-long
// dependent chains): DFMA, DADD, 64-bit SHFL + DADD (one butterfly level),
// LDS.64, mbarrier.test_wait on a completed phase.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_probe tools/lat_probe.cu
#include <cstdio>
#include <cstdint>

__global__ void probe(double* out, long long* cyc, double seed) {
  __shared__ double sh[1024];
  __shared__ uint64_t bar;
  const int lane = threadIdx.x;
  for (int i = lane; i < 1024; i += 32) sh[i] = (i + 1) * 1e-3;
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar)));
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(&bar)));
  }
  __syncwarp();
  double a = seed + lane, b = 1.0000001, c = 1e-9;
  constexpr int N = 1024;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) a = fma(a, b, c);
  t1 = clock64();
  cyc[0] = t1 - t0;
  // DADD chain
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) a = a + c;
  t1 = clock64();
  cyc[1] = t1 - t0;
  // butterfly level: SHFL(hi,lo) + DADD
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) a = a + __shfl_xor_sync(0xffffffffu, a, 1 << (i & 4));
  t1 = clock64();
  cyc[2] = t1 - t0;
  // LDS.64 pointer-chase-like chain (address depends on the loaded value)
  int idx = lane;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) {
    const double v = sh[idx & 1023];
    idx = static_cast<int>(v * 1000.0) + 1;
  }
  t1 = clock64();
  cyc[3] = t1 - t0;
  // mbarrier.test_wait on a completed phase, result feeding the next test
  unsigned ok = 0, acc = 0;
  t0 = clock64();
  for (int i = 0; i < 256; ++i) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"((unsigned)__cvta_generic_to_shared(&bar)), "r"(acc & 0u)
        : "memory");
    acc += ok;
  }
  t1 = clock64();
  cyc[4] = (t1 - t0) * 4;  // scaled to 1024
  // mbarrier.try_wait on a completed phase
  t0 = clock64();
  for (int i = 0; i < 256; ++i) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"((unsigned)__cvta_generic_to_shared(&bar)), "r"(acc & 0u)
        : "memory");
    acc += ok;
  }
  t1 = clock64();
  cyc[5] = (t1 - t0) * 4;
  out[lane] = a + idx + acc;
}

int main() {
  double* d_out;
  long long* d_cyc;
  cudaMalloc(&d_out, 32 * sizeof(double));
  cudaMalloc(&d_cyc, 8 * sizeof(long long));
  probe<<<1, 32>>>(d_out, d_cyc, 0.5);  // warm-up
  probe<<<1, 32>>>(d_out, d_cyc, 0.5);
  long long h[8];
  cudaMemcpy(h, d_cyc, sizeof(h), cudaMemcpyDeviceToHost);
  const char* names[] = {"dfma", "dadd", "shfl64+dadd", "lds64_chain", "mbar_test_wait", "mbar_try_wait"};
  printf("{");
  for (int i = 0; i < 6; ++i) printf("%s\"%s\": %.2f", i ? ", " : "", names[i], h[i] / 1024.0);
  printf("}\n");
  return 0;
}
