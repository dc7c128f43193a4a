// Throughput of the attention softmax instruction mix per 64-key row chunk (registers only):
// 22 FMNMX3, 64 FFMA, 64 MUFU.EX2, 64 FADD, 32 F2FP per thread; 8 warps per SM like the kernel.
#include <cstdio>
#include <cuda_bf16.h>
template <int MODE>
__global__ void __launch_bounds__(256, 1) k(unsigned* out, int iters) {
  float sv[64];
  for (int i = 0; i < 64; ++i) sv[i] = (threadIdx.x * 7 + i) * 1e-3f;
  unsigned acc = 0;
  float m = 0.f, l = 0.f;
  for (int it = 0; it < iters; ++it) {
    float mx0 = fmaxf(sv[0], sv[1]), mx1 = fmaxf(sv[2], sv[3]);
#pragma unroll
    for (int i = 4; i < 64; i += 4) {
      asm("max.f32 %0, %0, %1, %2;" : "+f"(mx0) : "f"(sv[i]), "f"(sv[i + 1]));
      asm("max.f32 %0, %0, %1, %2;" : "+f"(mx1) : "f"(sv[i + 2]), "f"(sv[i + 3]));
    }
    const float mn = fmaxf(m, fmaxf(mx0, mx1) * 0.18f);
    float ls0 = 0.f, ls1 = 0.f;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      float p0 = fmaf(sv[2 * i], 0.18f, -mn), p1 = fmaf(sv[2 * i + 1], 0.18f, -mn);
      if (MODE != 1) { asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(p0)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(p1)); }
      ls0 += p0; ls1 += p1;
      if (MODE != 2) { __nv_bfloat162 h = __floats2bfloat162_rn(p0, p1); acc += *reinterpret_cast<unsigned*>(&h); }
      else acc += __float_as_uint(p0) ^ __float_as_uint(p1);
      sv[2 * i] += 1e-6f * p0;        // keep values live / changing
    }
    l = l * 0.5f + ls0 + ls1;
    m = mn;
  }
  if (acc == 12345u || l == 1.2345f) out[threadIdx.x] = acc;
}
int main() {
  unsigned* d; cudaMalloc(&d, 4096);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* nm[3] = {"full mix", "no ex2", "no f2fp"};
  for (int mode = 0; mode < 3; ++mode)
    for (int threads : {128, 256}) {
      auto kern = mode == 0 ? k<0> : mode == 1 ? k<1> : k<2>;
      kern<<<148, threads>>>(d, 10);
      cudaEventRecord(e0);
      const int iters = 4000;
      kern<<<148, threads>>>(d, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double elems = 148.0 * threads * iters * 64;
      printf("%-10s warps/SM=%d: %.3f ms, %.2f elem/clk/SM (MUFU bound 16)\n", nm[mode], threads / 32, ms, elems / (ms * 1e-3) / 148 / 1.965e9);
    }
  return 0;
}
