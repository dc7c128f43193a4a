// mbarrier ping-pong latency between two warps of one CTA (clock64 cycles per round trip).
#include <cstdio>
#include <cstdint>
#include "../../paper_2412_02962_b200/csrc/sm100.cuh"
using namespace pcpp::sm100;
template <int MODE>   // 0 try_wait(suspend hint), 1 test_wait spin, 2 try_wait no hint
__device__ __forceinline__ void w8(uint64_t* bar, uint32_t par) {
  if (MODE == 0) mbar_wait(bar, par);
  else if (MODE == 1) mbar_wait_spin(bar, par);
  else {
    uint32_t a = smem_u32(bar), ok = 0;
    while (!ok) asm volatile("{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n" : "=r"(ok) : "r"(a), "r"(par) : "memory");
  }
}
template <int MODE>
__global__ void k(long long* out, int iters, int extra_warps) {
  __shared__ uint64_t bars[2];
  if (threadIdx.x == 0) { mbar_init(&bars[0], 1); mbar_init(&bars[1], 1); fence_barrier_init(); }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  long long t0 = clock64();
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < iters; ++i) { mbar_arrive(&bars[0]); w8<MODE>(&bars[1], i & 1); }
  } else if (warp == 1 && lane == 0) {
    for (int i = 0; i < iters; ++i) { w8<MODE>(&bars[0], i & 1); mbar_arrive(&bars[1]); }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}
int main() {
  long long* d; cudaMalloc(&d, 8 * 148);
  const char* nm[3] = {"try_wait+suspend hint", "test_wait spin", "try_wait no hint"};
  for (int mode = 0; mode < 3; ++mode)
    for (int threads : {64, 320}) {
      auto kern = mode == 0 ? k<0> : mode == 1 ? k<1> : k<2>;
      kern<<<1, threads>>>(d, 1000, 0);
      kern<<<1, threads>>>(d, 10000, 0);
      long long c; cudaDeviceSynchronize(); cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
      printf("%-24s threads=%3d: %.0f clk per round trip (%s)\n", nm[mode], threads, c / 10000.0, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
