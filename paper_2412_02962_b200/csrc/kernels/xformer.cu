// Elementwise / row-wise kernels of SDXL's transformer block (the '_xf' models, SURVEY §8(f4),
// DESIGN.md reading D25): LayerNorm over the channels of every token, the GEGLU gate, and the
// layout of the 77-token cross-attention context.  All patch-local (no exchange); HBM-bound.
#include "../common.cuh"
#include "../kernels.h"

namespace pcpp {

namespace {
constexpr int LN_MAXV = 8;     // 8-channel vectors per lane: C <= 32 * 8 * 8 = 2048
}

// LayerNorm (eps 1e-5, biased variance): one warp per token, the token's C values held in registers
// (16-byte vectors, lane-strided: a warp reads the row contiguously), fp32 two-pass mean / variance.
template <typename T>
__global__ void __launch_bounds__(256) layernorm_kernel(const T* __restrict__ x, T* __restrict__ y,
                                                        const float* __restrict__ g, const float* __restrict__ b,
                                                        long long ntok, int C) {
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  const int nv = C / 8;
  for (long long t = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < ntok; t += warps) {
    const T* xr = x + t * C;
    float v[LN_MAXV][8];
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < LN_MAXV; ++i) {
      const int vi = lane + 32 * i;
      if (vi < nv) {
        load8(xr + vi * 8, v[i]);
#pragma unroll
        for (int e = 0; e < 8; ++e) s += v[i][e];
      }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
    const float mu = s / (float)C;
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < LN_MAXV; ++i)
      if (lane + 32 * i < nv) {
#pragma unroll
        for (int e = 0; e < 8; ++e) { const float dlt = v[i][e] - mu; q = fmaf(dlt, dlt, q); }
      }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) q += __shfl_xor_sync(0xffffffffu, q, d);
    const float rs = rsqrtf(q / (float)C + 1e-5f);
    T* yr = y + t * C;
#pragma unroll
    for (int i = 0; i < LN_MAXV; ++i) {
      const int vi = lane + 32 * i;
      if (vi < nv) {
        float o[8];
        const float4 g0 = __ldg(reinterpret_cast<const float4*>(g + vi * 8)), g1 = __ldg(reinterpret_cast<const float4*>(g + vi * 8 + 4));
        const float4 b0 = __ldg(reinterpret_cast<const float4*>(b + vi * 8)), b1 = __ldg(reinterpret_cast<const float4*>(b + vi * 8 + 4));
        const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
        const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = fmaf((v[i][e] - mu) * rs, gg[e], bb[e]);
        store8(yr + vi * 8, o);
      }
    }
  }
}

bool launch_layernorm(const ActView& x, const ActView& y, const float* g, const float* b, cudaStream_t s) {
  if (x.C % 8 || x.C > 32 * 8 * LN_MAXV) return false;
  const long long ntok = (long long)x.rows * x.B * x.W;
  long long blocks = (ntok + 7) / 8;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (x.dtype == DT_F32)
    launch_pdl(layernorm_kernel<float>, dim3((unsigned)blocks), dim3(256), 0, s, reinterpret_cast<const float*>(x.base),
               reinterpret_cast<float*>(y.base), g, b, ntok, x.C);
  else
    launch_pdl(layernorm_kernel<bf16>, dim3((unsigned)blocks), dim3(256), 0, s, reinterpret_cast<const bf16*>(x.base),
               reinterpret_cast<bf16*>(y.base), g, b, ntok, x.C);
  return true;
}

// GEGLU gate: u per token in 64-column blocks [value 64 | gate 64] (the builder interleaves the rows of
// W_ff1 = [W_value; W_gate] so that the fused GEMM epilogue sees a value column and its gate in one
// tile) -> out = value * gelu(gate), exact GELU (x Phi(x) with erff; reading D25).  The unfused path
// (fp32 parity mode / SIMT GEMM).
template <typename T>
__global__ void __launch_bounds__(256) geglu_kernel(const T* __restrict__ u, T* __restrict__ out, long long ntok, int C4) {
  pdl_trigger();
  pdl_wait();
  const int nv = C4 / 8;
  const long long total = ntok * nv;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long t = i / nv;
    const int c = (int)(i - t * nv) * 8;
    const int uc = (c >> 6) * 128 + (c & 63);     // value column of output column c in the blocked order
    float a[8], g[8];
    load8(u + t * 2 * C4 + uc, a);
    load8(u + t * 2 * C4 + uc + 64, g);
#pragma unroll
    for (int e = 0; e < 8; ++e) a[e] *= 0.5f * g[e] * (1.f + erff(g[e] * 0.70710678118654752f));
    store8(out + t * C4 + c, a);
  }
}

void launch_geglu(const ActView& u, const ActView& out, cudaStream_t s) {
  const long long ntok = (long long)u.rows * u.B * u.W;
  const long long total = ntok * (out.C / 8);
  long long blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (u.dtype == DT_F32)
    launch_pdl(geglu_kernel<float>, dim3((unsigned)blocks), dim3(256), 0, s, reinterpret_cast<const float*>(u.base),
               reinterpret_cast<float*>(out.base), ntok, out.C);
  else
    launch_pdl(geglu_kernel<bf16>, dim3((unsigned)blocks), dim3(256), 0, s, reinterpret_cast<const bf16*>(u.base),
               reinterpret_cast<bf16*>(out.base), ntok, out.C);
}

// Context layout for one level: ctx fp32 [B][L][D] -> out [rows][B][W][D] (dtype of the plan) with
// key k = r * W + w; keys k >= L are zero (the attention masks them: AttnSrc.nkeys = L).
template <typename T>
__global__ void ctx_layout_kernel(const float* __restrict__ ctx, T* __restrict__ out, int rows, int B, int W, int L, int D) {
  const long long total = (long long)rows * B * W * D;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int d = (int)(i % D);
    const long long tok = i / D;
    const int w = (int)(tok % W), b = (int)((tok / W) % B), r = (int)(tok / ((long long)W * B));
    const int k = r * W + w;
    out[i] = from_f<T>(k < L ? ctx[((long long)b * L + k) * D + d] : 0.f);
  }
}

void launch_ctx_layout(const float* ctx, const ActView& out, int L, cudaStream_t s) {
  const long long total = (long long)out.rows * out.B * out.W * out.C;
  long long blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (out.dtype == DT_F32)
    ctx_layout_kernel<float><<<(unsigned)blocks, 256, 0, s>>>(ctx, reinterpret_cast<float*>(out.base), out.rows, out.B, out.W, L, out.C);
  else
    ctx_layout_kernel<bf16><<<(unsigned)blocks, 256, 0, s>>>(ctx, reinterpret_cast<bf16*>(out.base), out.rows, out.B, out.W, L, out.C);
}

}  // namespace pcpp
