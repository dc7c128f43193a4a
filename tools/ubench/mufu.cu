// Microbenchmark: per-SM throughput of ex2.approx (MUFU), FFMA, F2FP bf16x2 pack, FMNMX3 on this GPU.
#include <cstdio>
#include <cuda_bf16.h>
template <int OP>
__global__ void k(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i * 0.1f;
  unsigned acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (OP == 1) a[i] = fmaf(a[i], 0.999f, 0.001f);
      if (OP == 2) { __nv_bfloat162 h = __floats2bfloat162_rn(a[i], a[(i + 1) & 7]); acc += *reinterpret_cast<unsigned*>(&h); a[i] += 1e-7f; }
      if (OP == 3) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(a[(i + 1) & 7]), "f"(a[(i + 2) & 7]));
      if (OP == 4) { unsigned u; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u) : "f"(a[i]), "f"(a[(i + 3) & 7])); acc ^= u; }
      if (OP == 5) { asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
                     if (i & 1) { unsigned u; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u) : "f"(a[i]), "f"(a[i - 1])); acc ^= u; } }
      if (OP == 6) { unsigned u; asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(u) : "r"(__float_as_uint(a[i])), "r"(__float_as_uint(a[(i + 3) & 7]))); acc ^= u; a[i] = __uint_as_float(u); }
    }
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.f || acc == 7) out[threadIdx.x] = s + acc;
}
int main() {
  float* d; cudaMalloc(&d, 4096);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[7] = {"ex2.approx", "ffma", "f2fp.bf16x2 (+fadd)", "fmnmx3", "cvt.rn.bf16x2 only", "ex2 + cvt per 2 (count=ex2)", "prmt"};
  int iters = 20000;
  for (int op = 0; op < 7; ++op) {
    for (int threads : {256, 1024}) {
      auto kern = op == 0 ? k<0> : op == 1 ? k<1> : op == 2 ? k<2> : op == 3 ? k<3> : op == 4 ? k<4> : op == 5 ? k<5> : k<6>;
      kern<<<148, threads>>>(d, 100);
      cudaEventRecord(e0);
      kern<<<148, threads>>>(d, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = 148.0 * threads * iters * 8;
      int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
      printf("%-22s threads/SM=%4d  %.3f ms  %.2f Tops/s  %.2f ops/clk/SM (at %d MHz)\n", names[op], threads, ms,
             ops / ms / 1e9, ops / (ms * 1e-3) / 148 / (clk * 1e3), clk / 1000);
    }
  }
  return 0;
}
