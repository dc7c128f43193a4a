#include <algorithm>
#include <cstdlib>
// SIMT implicit-GEMM conv3x3 / 1x1 (fp32 accumulate).  Used for:
//  * every contraction in fp32 mode (parity mode, rel-L2 <= 1e-5; no fp32 tensor-core kind exists),
//  * conv_in (Cin = 4) in both modes, and as the bf16 fallback for shapes the tcgen05 path rejects.
// Halo rows (r = -1, rows) come from the padded input tensor (filled by the exchange, reading D8);
// columns outside [0, W) are zero padding.
#include "../common.cuh"
#include "../kernels.h"

namespace pcpp {

namespace {
constexpr int BM = 64, BN = 64, BK = 16;

template <typename TA>
__device__ __forceinline__ float load_a(const GemmArgs& g, int r, int b, int w, bool valid, int k) {
  if (!valid) return 0.f;
  int tap = k / g.cin, c = k - tap * g.cin;
  int dr = 0, dw = 0;
  if (g.taps == 9) { dr = tap / 3 - 1; dw = tap % 3 - 1; }
  int ri = r * g.stride + dr, wi = w * g.stride + dw;
  const ActView& v = (c < g.c0) ? g.a0 : g.a1;
  if (c >= g.c0) c -= g.c0;
  if (wi < 0 || wi >= v.W) return 0.f;
  const TA* p = reinterpret_cast<const TA*>(v.base);
  return to_f(p[(((long long)ri * v.B + b) * v.W + wi) * v.C + c]);
}

__device__ __forceinline__ void store_out(const ActView& v, long long idx, float x) {
  if (v.dtype == DT_F32) reinterpret_cast<float*>(v.base)[idx] = x;
  else reinterpret_cast<bf16*>(v.base)[idx] = __float2bfloat16_rn(x);
}
__device__ __forceinline__ float load_res(const ActView& v, long long idx) {
  return v.dtype == DT_F32 ? reinterpret_cast<const float*>(v.base)[idx]
                           : __bfloat162float(reinterpret_cast<const bf16*>(v.base)[idx]);
}
}  // namespace

template <typename TA, typename TW>
__global__ void __launch_bounds__(256) gemm_simt_kernel(const GemmArgs g) {
  pdl_trigger();
  pdl_wait();
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int M = g.rows_out * g.B * g.w_out;
  const int K = g.taps * g.cin;
  // the 4 A rows this thread loads: mm = ty + 16 i
  int ar[4], ab[4], aw[4]; bool av[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int m = m0 + ty + 16 * i;
    av[i] = m < M;
    int mm = av[i] ? m : 0;
    aw[i] = mm % g.w_out; int t = mm / g.w_out; ab[i] = t % g.B; ar[i] = t / g.B;
  }
  const TW* Wt = reinterpret_cast<const TW*>(g.w);
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  for (int k0 = 0; k0 < K; k0 += BK) {
    const int k = k0 + tx;
    const bool kv = k < K;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      As[tx][ty + 16 * i] = kv ? load_a<TA>(g, ar[i], ab[i], aw[i], av[i], k) : 0.f;
      int n = n0 + ty + 16 * i;
      Bs[tx][ty + 16 * i] = (kv && n < g.N) ? to_f(Wt[(long long)n * K + k]) : 0.f;
    }
    __syncthreads();
    float part[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) part[i][j] = 0.f;
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { a[i] = As[kk][ty * 4 + i]; b[i] = Bs[kk][tx * 4 + i]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) part[i][j] = fmaf(a[i], b[j], part[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] += part[i][j];   // blocked summation (fp32-mode accuracy)
    __syncthreads();
  }
  // epilogue
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int m = m0 + ty * 4 + i;
    if (m >= M) continue;
    int w = m % g.w_out; int t = m / g.w_out; int b = t % g.B; int r = t / g.B;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int n = n0 + tx * 4 + j;
      if (n >= g.N) continue;
      float v = acc[i][j];
      if (g.bias) v += g.bias[n];
      if (g.temb) v += g.temb[b * g.temb_ld + n];
      if (n < g.n_split) {
        long long idx = (((long long)r * g.out.B + b) * g.out.W + w) * g.out.C + n;
        if (g.res.base) v += load_res(g.res, (((long long)r * g.res.B + b) * g.res.W + w) * g.res.C + n);
        store_out(g.out, idx, v);
      } else {
        int n2 = n - g.n_split;
        long long idx = (((long long)r * g.out2.B + b) * g.out2.W + w) * g.out2.C + n2;
        store_out(g.out2, idx, v);
      }
    }
  }
}

void launch_gemm_simt(const GemmArgs& g, cudaStream_t s) {
  const int M = g.rows_out * g.B * g.w_out;
  dim3 grid((M + BM - 1) / BM, (g.N + BN - 1) / BN);
  const int ta = g.a0.dtype;
  if (ta == DT_F32 && g.wdtype == DT_F32) launch_pdl(gemm_simt_kernel<float, float>, dim3(grid), dim3(256), 0, s, g);
  else if (ta == DT_BF16 && g.wdtype == DT_BF16) launch_pdl(gemm_simt_kernel<bf16, bf16>, dim3(grid), dim3(256), 0, s, g);
  else if (ta == DT_F32 && g.wdtype == DT_BF16) launch_pdl(gemm_simt_kernel<float, bf16>, dim3(grid), dim3(256), 0, s, g);
  else launch_pdl(gemm_simt_kernel<bf16, float>, dim3(grid), dim3(256), 0, s, g);
}

// ---------------------------------------------------------------------------------------------
// conv_out: 3x3, Cin -> 4, one warp per output token; lanes split the 9*Cin reduction.
// ---------------------------------------------------------------------------------------------
template <typename TA>
__global__ void __launch_bounds__(256) conv_out_kernel(const ActView in, const float* __restrict__ w,
                                                        const float* __restrict__ bias, const ActView out) {
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const long long tok = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  const long long M = (long long)out.rows * out.B * out.W;
  if (tok >= M) return;
  const int wo = tok % out.W; const long long t = tok / out.W; const int b = t % out.B; const int r = t / out.B;
  const int C = in.C, K = 9 * C;
  const TA* x = reinterpret_cast<const TA*>(in.base);
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int tap = 0; tap < 9; ++tap) {
    const int ri = r + tap / 3 - 1, wi = wo + tap % 3 - 1;
    if (wi < 0 || wi >= in.W) continue;
    const TA* px = x + (((long long)ri * in.B + b) * in.W + wi) * C;
    for (int c = lane; c < C; c += 32) {
      const float a = to_f(px[c]);
#pragma unroll
      for (int o = 0; o < 4; ++o) acc[o] = fmaf(a, w[o * K + tap * C + c], acc[o]);
    }
  }
#pragma unroll
  for (int o = 0; o < 4; ++o)
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) acc[o] += __shfl_xor_sync(0xffffffffu, acc[o], d);
  if (lane == 0) {
    float* po = reinterpret_cast<float*>(out.base) + tok * 4;
#pragma unroll
    for (int o = 0; o < 4; ++o) po[o] = acc[o] + bias[o];
  }
}

// conv_in (Cin = 4, fp32 latent input, bf16 output): thread = output channel (its 36 weights and
// bias in registers); a CTA covers 64 consecutive output tokens of one (row, batch).  The 3 input rows
// x 66 columns of the latent patch are staged in smem once (3 KB; zero outside [0, W)), and each
// thread accumulates 8 tokens at a time in independent registers: per kernel-row the 10 input vectors
// the 8 tokens need are read once (smem broadcast) and serve its 3 taps.  (The previous version, one
// token at a time with a 36-deep dependent FMA chain and 9 global loads per token, took 67 us.)
constexpr int CIN_TOK = 64;
__global__ void __launch_bounds__(320) conv_in_kernel(const ActView in, const float* __restrict__ w,
                                                      const float* __restrict__ bias, const ActView out, int N) {
  pdl_trigger();
  __shared__ float4 xs[3][CIN_TOK + 2];
  const int n = threadIdx.x;
  float wr[36];
  float bi = 0.f;
  if (n < N) {
#pragma unroll
    for (int i = 0; i < 36; ++i) wr[i] = w[n * 36 + i];
    bi = bias ? bias[n] : 0.f;
  }
  pdl_wait();
  const int nwt = (out.W + CIN_TOK - 1) / CIN_TOK;
  const int wt = blockIdx.x % nwt, rb = blockIdx.x / nwt;
  const int b = rb % out.B, r = rb / out.B;
  const int w0 = wt * CIN_TOK;
  const float4* x = reinterpret_cast<const float4*>(in.base);   // [rows (+halo)][B][W] x 4 channels
  for (int i = threadIdx.x; i < 3 * (CIN_TOK + 2); i += blockDim.x) {
    const int dr = i / (CIN_TOK + 2), k = i % (CIN_TOK + 2), wi = w0 - 1 + k;
    xs[dr][k] = (wi >= 0 && wi < in.W) ? __ldg(x + ((long long)(r + dr - 1) * in.B + b) * in.W + wi)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __syncthreads();
  if (n >= N) return;
  const int nw = min(CIN_TOK, out.W - w0);
  bf16* y = reinterpret_cast<bf16*>(out.base) + (((long long)r * out.B + b) * out.W + w0) * out.C + n;
  for (int k0 = 0; k0 < nw; k0 += 8) {
    float acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = bi;
#pragma unroll
    for (int dr = 0; dr < 3; ++dr) {
      float4 v[10];
#pragma unroll
      for (int k = 0; k < 10; ++k) v[k] = xs[dr][k0 + k];
#pragma unroll
      for (int dw = 0; dw < 3; ++dw) {
        const float* wt4 = wr + (dr * 3 + dw) * 4;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          acc[k] = fmaf(v[k + dw].x, wt4[0], acc[k]); acc[k] = fmaf(v[k + dw].y, wt4[1], acc[k]);
          acc[k] = fmaf(v[k + dw].z, wt4[2], acc[k]); acc[k] = fmaf(v[k + dw].w, wt4[3], acc[k]);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (k0 + k < nw) y[(long long)(k0 + k) * out.C] = __float2bfloat16_rn(acc[k]);
  }
}

bool launch_conv_in(const GemmArgs& g, cudaStream_t s) {
  if (!(g.taps == 9 && g.stride == 1 && g.cin == 4 && !g.a1.base && g.a0.dtype == DT_F32 && g.a0.C == 4 &&
        g.wdtype == DT_F32 && g.out.dtype == DT_BF16 && !g.out2.base && !g.res.base && !g.temb && g.N <= 320 &&
        g.out.C == g.N))
    return false;
  const int nwt = (g.w_out + CIN_TOK - 1) / CIN_TOK;
  launch_pdl(conv_in_kernel, dim3((unsigned)(g.rows_out * g.B * nwt)), dim3(((g.N + 31) / 32) * 32), 0, s, g.a0,
             reinterpret_cast<const float*>(g.w), g.bias, g.out, g.N);
  return true;
}

// conv_out v3 (bf16 in, Cin -> 4, fp32 out): the 9*Cin x 4 weights are staged in smem as float4 over
// the 4 outputs, laid out [e][chunk] (chunk = tap * Cin/8 + c/8, e = channel within the 8-channel
// chunk) so a warp's 32 lanes read 32 consecutive float4 (no bank conflicts).  A warp computes 4
// horizontally adjacent tokens per pass (each weight read serves 4 tokens); lanes split the
// 9*Cin/8 16-byte input chunks; the 16 partial sums are reduced with warp shuffles.
__global__ void __launch_bounds__(256) conv_out_v3_kernel(const ActView in, const float* __restrict__ w,
                                                          const float* __restrict__ bias, const ActView out) {
  pdl_trigger();
  extern __shared__ float4 wsm[];
  const int C = in.C, K = 9 * C, nc8 = C / 8, nchunk = 9 * nc8;
  for (int i = threadIdx.x; i < K; i += blockDim.x) {          // weights: not produced by the previous kernel
    const int tap = i / C, cc = i - tap * C;
    wsm[(cc & 7) * nchunk + tap * nc8 + (cc >> 3)] = make_float4(w[i], w[K + i], w[2 * K + i], w[3 * K + i]);
  }
  __syncthreads();
  pdl_wait();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int W = out.W, B = out.B, gpr = W / 4;
  const long long ngroups = (long long)out.rows * B * gpr;
  const bf16* x = reinterpret_cast<const bf16*>(in.base);
  const float4 bv = make_float4(bias[0], bias[1], bias[2], bias[3]);
  for (long long gi = (long long)blockIdx.x * 8 + warp; gi < ngroups; gi += (long long)gridDim.x * 8) {
    const int w0 = (int)(gi % gpr) * 4;
    const long long t = gi / gpr;
    const int b = (int)(t % B), r = (int)(t / B);
    float acc[4][4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int o = 0; o < 4; ++o) acc[q][o] = 0.f;
    for (int j = lane; j < nchunk; j += 32) {
      const int tap = j / nc8, c = (j - tap * nc8) * 8;
      const int dr = tap / 3 - 1, dw = tap - (tap / 3) * 3 - 1;
      const bf16* prow = x + (((long long)(r + dr) * in.B + b) * in.W) * C + c;
      float xv[4][8];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int wi = w0 + q + dw;
        if (wi >= 0 && wi < in.W) load8(prow + (long long)wi * C, xv[q]);
        else {
#pragma unroll
          for (int e = 0; e < 8; ++e) xv[q][e] = 0.f;
        }
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float4 wv = wsm[e * nchunk + j];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          acc[q][0] = fmaf(xv[q][e], wv.x, acc[q][0]); acc[q][1] = fmaf(xv[q][e], wv.y, acc[q][1]);
          acc[q][2] = fmaf(xv[q][e], wv.z, acc[q][2]); acc[q][3] = fmaf(xv[q][e], wv.w, acc[q][3]);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int o = 0; o < 4; ++o)
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) acc[q][o] += __shfl_xor_sync(0xffffffffu, acc[q][o], d);
    if (lane < 4) {
      const int q = lane;
      float4 v;
      v.x = acc[0][0]; v.y = acc[0][1]; v.z = acc[0][2]; v.w = acc[0][3];
#pragma unroll
      for (int qq = 1; qq < 4; ++qq)
        if (q == qq) { v.x = acc[qq][0]; v.y = acc[qq][1]; v.z = acc[qq][2]; v.w = acc[qq][3]; }
      float4* po = reinterpret_cast<float4*>(reinterpret_cast<float*>(out.base) + (((long long)r * out.B + b) * out.W + w0 + q) * 4);
      *po = make_float4(v.x + bv.x, v.y + bv.y, v.z + bv.z, v.w + bv.w);
    }
  }
}

// conv_out with warp-level tensor-core MMAs (bf16 in, Cin -> 4, fp32 out): out[t][o] = bias[o] +
// sum_{tap, c} x[t + tap][c] W[o][tap C + c] as 16-token x 8-output (4 real) tiles of
// mma.sync.m16n8k16 (fp32 accumulation).  The fp32 weights are split w = hi + lo (both bf16, lo =
// bf16(w - hi)) and each K step issues the two MMAs, so the weights keep ~16 mantissa bits (x is bf16
// exactly).  The K index inside a 16-channel step is permuted so that lane (g, t) holds channels
// 4t .. 4t + 3 of its tokens: one 8-byte load per token row (full 32-byte sectors) and one 8-byte smem
// load per weight half; A and B use the same permutation, so the sum is unchanged.  CTA = 4 warps =
// 64 consecutive output tokens of one (row, batch); the 3x3 reuse is served by L1.
constexpr int COUT_TOK = 64;
__device__ __forceinline__ void mma_bf16_16816(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__global__ void __launch_bounds__(128) conv_out_mma_kernel(const ActView in, const float* __restrict__ w,
                                                           const float* __restrict__ bias, const ActView out) {
  pdl_trigger();
  extern __shared__ __align__(16) uint8_t csm[];
  const int C = in.C, K = 9 * C, Kp = K + 16;                 // row pad: conflict-free 8-byte reads
  bf16* whi = reinterpret_cast<bf16*>(csm);                   // [4][Kp]
  bf16* wlo = whi + 4 * Kp;
  for (int i = threadIdx.x; i < K / 4; i += blockDim.x * 4) {    // weights (static: before the PDL wait), float4
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k4 = i + u * blockDim.x;                      // float4 index within a row of K / 4
      if (k4 >= K / 4) break;
#pragma unroll
      for (int o = 0; o < 4; ++o) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(w + (size_t)o * K) + k4);
        const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const bf16 h = __float2bfloat16_rn(vv[e]);
          whi[o * Kp + 4 * k4 + e] = h;
          wlo[o * Kp + 4 * k4 + e] = __float2bfloat16_rn(vv[e] - __bfloat162float(h));
        }
      }
    }
  }
  __syncthreads();
  pdl_wait();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int nwt = (out.W + COUT_TOK - 1) / COUT_TOK;
  const int wt = blockIdx.x % nwt, rb = blockIdx.x / nwt;
  const int b = rb % out.B, r = rb / out.B;
  const int wA = wt * COUT_TOK + warp * 16 + g;               // this lane's two tokens: wA, wA + 8
  const bf16* x = reinterpret_cast<const bf16*>(in.base);
  float d[4] = {0.f, 0.f, 0.f, 0.f};
  const bool bl = g < 4;                                      // B columns (outputs) 4..7 are zero
  const uint2 z2 = make_uint2(0u, 0u);
  for (int tap = 0; tap < 9; ++tap) {
    const int dr = tap / 3 - 1, dw = tap % 3 - 1;
    const int w0 = wA + dw, w1 = wA + 8 + dw;
    const bool v0 = w0 >= 0 && w0 < in.W, v1 = w1 >= 0 && w1 < in.W;
    const bf16* row = x + (((long long)(r + dr) * in.B + b) * in.W) * C + 4 * t;
    const bf16* p0 = row + (long long)w0 * C;
    const bf16* p1 = row + (long long)w1 * C;
    const bf16* ph = whi + g * Kp + tap * C + 4 * t;
    const bf16* pl = wlo + g * Kp + tap * C + 4 * t;
    // batches of U K steps: all loads of a batch are issued before its MMAs (the MMAs chain through d,
    // so the compiler would otherwise issue each load just before its use)
    constexpr int U = 8;
    for (int cb = 0; cb < C; cb += 16 * U) {
      uint2 a0[U], a1[U], bh[U], bo[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c0 = cb + 16 * u;
        const bool kin = c0 < C;
        a0[u] = (kin && v0) ? __ldg(reinterpret_cast<const uint2*>(p0 + c0)) : z2;
        a1[u] = (kin && v1) ? __ldg(reinterpret_cast<const uint2*>(p1 + c0)) : z2;
        bh[u] = (kin && bl) ? *reinterpret_cast<const uint2*>(ph + c0) : z2;
        bo[u] = (kin && bl) ? *reinterpret_cast<const uint2*>(pl + c0) : z2;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t af[4] = {a0[u].x, a1[u].x, a0[u].y, a1[u].y};   // (g, k 2t..), (g+8, ..), (g, k 2t+8..), (g+8, ..)
        mma_bf16_16816(d, af, bh[u].x, bh[u].y);
        mma_bf16_16816(d, af, bo[u].x, bo[u].y);
      }
    }
  }
  if (t < 2) {                                                // outputs 2t, 2t + 1 of tokens wA, wA + 8
    const float b0 = bias[2 * t], b1 = bias[2 * t + 1];
    float* po = reinterpret_cast<float*>(out.base) + (((long long)r * out.B + b) * out.W) * 4 + 2 * t;
    if (wA < out.W) *reinterpret_cast<float2*>(po + (long long)wA * 4) = make_float2(d[0] + b0, d[1] + b1);
    if (wA + 8 < out.W) *reinterpret_cast<float2*>(po + (long long)(wA + 8) * 4) = make_float2(d[2] + b0, d[3] + b1);
  }
}

void launch_conv_out(const ActView& in, const float* w, const float* bias, const ActView& out, cudaStream_t s) {
  if (in.dtype == DT_BF16 && in.C % 16 == 0 && out.C == 4 && (size_t)(9 * in.C + 16) * 16 <= 100 * 1024) {
    const int nwt = (out.W + COUT_TOK - 1) / COUT_TOK;
    const size_t smem = (size_t)(9 * in.C + 16) * 4 * 2 * 2;
    static bool attr = false;
    if (!attr) { cudaFuncSetAttribute(conv_out_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024); attr = true; }
    launch_pdl(conv_out_mma_kernel, dim3((unsigned)(out.rows * out.B * nwt)), dim3(128), smem, s, in, w, bias, out);
    return;
  }

  if (in.dtype == DT_BF16 && in.C % 8 == 0 && out.C == 4 && out.W % 4 == 0 && (size_t)in.C * 9 * 16 <= 48 * 1024) {
    const long long ngroups = (long long)out.rows * out.B * (out.W / 4);
    const long long blocks = std::min<long long>((ngroups + 7) / 8, 148 * 2);
    launch_pdl(conv_out_v3_kernel, dim3((unsigned)blocks), dim3(256), (size_t)in.C * 9 * 16, s, in, w, bias, out);
    return;
  }
  const long long M = (long long)out.rows * out.B * out.W;
  dim3 grid((unsigned)((M + 7) / 8));
  if (in.dtype == DT_F32) launch_pdl(conv_out_kernel<float>, dim3(grid), dim3(256), 0, s, in, w, bias, out);
  else launch_pdl(conv_out_kernel<bf16>, dim3(grid), dim3(256), 0, s, in, w, bias, out);
}

}  // namespace pcpp
