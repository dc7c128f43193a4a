// SIMT flash-style partially conditioned attention (fp32 math; fp32-mode parity path and
// bf16 fallback).  §3.3: queries from the local fresh patch; keys/values from
// [top stale band ; local fresh ; bottom stale band] (Eq. 1 context, reading D13 order).
// One CTA = (query block of 64, head, b); 8 warps x 8 queries; K/V streamed in 32-key chunks.
#include "../common.cuh"
#include "../kernels.h"

namespace pcpp {

namespace {
constexpr int QB = 64, KC = 32, HD = 64;
}

template <typename T>
__global__ void __launch_bounds__(256) attn_simt_kernel(const AttnArgs a) {
  pdl_trigger();
  pdl_wait();
  __shared__ float Qs[QB][HD];
  __shared__ float Ks[KC][HD + 1];
  __shared__ float Vs[KC][HD];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int qblk = blockIdx.x, head = blockIdx.y, b = blockIdx.z;
  const int nq = a.h * a.W;
  const int C = a.C, C2 = 2 * a.C;
  const T* Q = reinterpret_cast<const T*>(a.q);
  // load Q block
  for (int e = tid; e < QB * HD; e += 256) {
    int qi = e / HD, d = e % HD;
    int j = qblk * QB + qi;
    float v = 0.f;
    if (j < nq) {
      int r = j / a.W, w = j % a.W;
      v = to_f(Q[(((long long)r * a.B + b) * a.W + w) * C + head * HD + d]);
    }
    Qs[qi][d] = v * 0.125f;        // scale 1/sqrt(64) (reading D12)
  }
  float m[8], l[8], acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { m[i] = -INFINITY; l[i] = 0.f; acc[i][0] = acc[i][1] = 0.f; }

  for (int s = 0; s < a.nsrc; ++s) {
    const T* KV = reinterpret_cast<const T*>(a.src[s].kv);
    const int nk = a.src[s].nkeys > 0 ? min(a.src[s].nkeys, a.src[s].rows * a.W) : a.src[s].rows * a.W;
    for (int k0 = 0; k0 < nk; k0 += KC) {
      __syncthreads();
      for (int e = tid; e < KC * HD; e += 256) {
        int ki = e / HD, d = e % HD;
        int j = k0 + ki;
        float kv = 0.f, vv = 0.f;
        if (j < nk) {
          int r = j / a.W, w = j % a.W;
          const T* p = KV + (((long long)r * a.B + b) * a.W + w) * C2 + head * HD + d;
          kv = to_f(p[0]); vv = to_f(p[C]);
        }
        Ks[ki][d] = kv; Vs[ki][d] = vv;
      }
      __syncthreads();
      const int nvalid = min(KC, nk - k0);
      float sc[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int qi = warp * 8 + i;
        float dot = 0.f;
#pragma unroll 16
        for (int d = 0; d < HD; ++d) dot = fmaf(Qs[qi][d], Ks[lane][d], dot);
        sc[i] = lane < nvalid ? dot : -INFINITY;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float cm = sc[i];
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, d));
        const float mn = fmaxf(m[i], cm);
        const float alpha = (m[i] == -INFINITY) ? 0.f : expf(m[i] - mn);
        m[i] = mn;
        sc[i] = expf(sc[i] - mn);
        l[i] = l[i] * alpha + sc[i];
        acc[i][0] *= alpha; acc[i][1] *= alpha;
      }
      for (int j = 0; j < nvalid; ++j) {
        const float v0 = Vs[j][lane], v1 = Vs[j][lane + 32];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float p = __shfl_sync(0xffffffffu, sc[i], j);
          acc[i][0] = fmaf(p, v0, acc[i][0]);
          acc[i][1] = fmaf(p, v1, acc[i][1]);
        }
      }
    }
  }
  T* O = reinterpret_cast<T*>(a.out);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float ls = l[i];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, d);
    const int j = qblk * QB + warp * 8 + i;
    if (j >= nq) continue;
    const int r = j / a.W, w = j % a.W;
    T* p = O + (((long long)r * a.B + b) * a.W + w) * C + head * HD;
    const float inv = 1.f / ls;
    p[lane] = from_f<T>(acc[i][0] * inv);
    p[lane + 32] = from_f<T>(acc[i][1] * inv);
  }
}

void launch_attn_simt(const AttnArgs& a, cudaStream_t s) {
  dim3 grid((a.h * a.W + QB - 1) / QB, a.C / HD, a.B);
  if (a.dtype == DT_F32) launch_pdl(attn_simt_kernel<float>, dim3(grid), dim3(256), 0, s, a);
  else launch_pdl(attn_simt_kernel<bf16>, dim3(grid), dim3(256), 0, s, a);
}

}  // namespace pcpp
