#include <algorithm>
// HBM-/launch-bound elementwise kernels of the step: latent prep, nearest upsample, the fused
// CFG (Eq. 2) + DDIM update, the timestep embedding, and the pack/unpack
// segment copier used for band staging and the loopback exchange.
#include "../common.cuh"
#include "../kernels.h"

namespace pcpp {

// ---- latent [h][W][4] fp32 -> xin [h][2][W][4] fp32 (rows 0..h-1; halos untouched) ------------
__global__ void prep_latent_kernel(const float4* __restrict__ lat, float4* __restrict__ xin, int h, int W, int B) {
  pdl_trigger();
  pdl_wait();
  const long long n = (long long)h * W;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / W, w = i % W;
    const float4 v = lat[i];
    for (int b = 0; b < B; ++b) xin[(r * B + b) * W + w] = v;     // every CFG branch held by this rank
  }
}
void launch_prep_latent(const float* latent, const ActView& xin, cudaStream_t s) {
  const long long n = (long long)xin.rows * xin.W;
  int blocks = (int)((n + 255) / 256); if (blocks > 1184) blocks = 1184;
  launch_pdl(prep_latent_kernel, dim3(blocks), dim3(256), 0, s, reinterpret_cast<const float4*>(latent),
                                             reinterpret_cast<float4*>(xin.base), xin.rows, xin.W, xin.B);
}

// ---- nearest x2 upsample (16-byte vectors) ------------------------------------------------------
__global__ void upsample2_kernel(const uint4* __restrict__ in, uint4* __restrict__ out,
                                 int h, int B, int W, int nv /*16B vectors per token*/) {
  pdl_trigger();
  pdl_wait();
  const long long n = (long long)2 * h * B * 2 * W * nv;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int v = (int)(i % nv); long long t = i / nv;
    const int wo = (int)(t % (2 * W)); t /= (2 * W);
    const int b = (int)(t % B); const int ro = (int)(t / B);
    out[i] = in[((((long long)(ro >> 1)) * B + b) * W + (wo >> 1)) * nv + v];
  }
}
void launch_upsample2(const ActView& in, const ActView& out, cudaStream_t s) {
  const int nv = (int)(in.C * dtype_size(in.dtype) / 16);
  const long long n = (long long)out.rows * out.B * out.W * nv;
  int blocks = (int)((n + 255) / 256); if (blocks > 1184 * 2) blocks = 1184 * 2;
  launch_pdl(upsample2_kernel, dim3(blocks), dim3(256), 0, s, reinterpret_cast<const uint4*>(in.base), reinterpret_cast<uint4*>(out.base),
                                          in.rows, in.B, in.W, nv);
}

// ---- CFG + DDIM -------------------------------------------------------------------------------
// eps_hat = eps_u + s (eps_c - eps_u);  x0 = (x - sqrt(1-ab) eps_hat)/sqrt(ab);
// x' = sqrt(ab_prev) x0 + sqrt(1-ab_prev) eps_hat     (b = 0 uncond, b = 1 cond; reading D11)
__global__ void cfg_ddim_kernel(const float4* __restrict__ eps, float4* __restrict__ lat, int h, int W,
                                float s_cfg, const double* __restrict__ coef, const int* __restrict__ k_dev) {
  pdl_trigger();
  pdl_wait();
  const int k = *k_dev;
  const float sa = (float)coef[4 * k + 0], s1a = (float)coef[4 * k + 1];
  const float sp = (float)coef[4 * k + 2], s1p = (float)coef[4 * k + 3];
  const float inv_sa = (float)(1.0 / coef[4 * k + 0]);
  (void)sa;
  const long long n = (long long)h * W;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / W, w = i % W;
    const float4 eu = eps[(r * 2 + 0) * W + w], ec = eps[(r * 2 + 1) * W + w];
    float4 x = lat[i];
    float e[4] = {eu.x + s_cfg * (ec.x - eu.x), eu.y + s_cfg * (ec.y - eu.y),
                  eu.z + s_cfg * (ec.z - eu.z), eu.w + s_cfg * (ec.w - eu.w)};
    float* xv = &x.x;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const float x0 = (xv[c] - s1a * e[c]) * inv_sa;
      xv[c] = sp * x0 + s1p * e[c];
    }
    lat[i] = x;
  }
}
void launch_cfg_ddim(const float* eps, float* latent, int h, int W, float s_cfg, const double* coef,
                     const int* k_dev, cudaStream_t s) {
  const long long n = (long long)h * W;
  int blocks = (int)((n + 255) / 256); if (blocks > 1184) blocks = 1184;
  launch_pdl(cfg_ddim_kernel, dim3(blocks), dim3(256), 0, s, reinterpret_cast<const float4*>(eps), reinterpret_cast<float4*>(latent),
                                         h, W, s_cfg, coef, k_dev);
}

// DPM-Solver++(2M), multistep data prediction (north star "DDIM/DPM-solver"; reading D23)
__global__ void cfg_dpmpp_kernel(const float4* __restrict__ eps, float4* __restrict__ lat, float4* __restrict__ x0h,
                                 int h, int W, float s_cfg, const double* __restrict__ coef, const int* __restrict__ k_dev) {
  pdl_trigger();
  pdl_wait();
  const int k = *k_dev;
  const float inv_a = (float)coef[6 * k + 0], sig = (float)coef[6 * k + 1];
  const float A = (float)coef[6 * k + 2], Bc = (float)coef[6 * k + 3];
  const float w0 = (float)coef[6 * k + 4], w1 = (float)coef[6 * k + 5];
  const long long n = (long long)h * W;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / W, w = i % W;
    const float4 eu = eps[(r * 2 + 0) * W + w], ec = eps[(r * 2 + 1) * W + w];
    float4 x = lat[i];
    float4 xp = x0h[i];
    const float e[4] = {eu.x + s_cfg * (ec.x - eu.x), eu.y + s_cfg * (ec.y - eu.y),
                        eu.z + s_cfg * (ec.z - eu.z), eu.w + s_cfg * (ec.w - eu.w)};
    float* xv = &x.x;
    float* pv = &xp.x;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const float x0 = (xv[c] - sig * e[c]) * inv_a;
      const float D = w1 != 0.f ? fmaf(w0, x0, w1 * pv[c]) : x0;   // first-order steps never read the history
      xv[c] = fmaf(A, xv[c], Bc * D);
      pv[c] = x0;
    }
    lat[i] = x;
    x0h[i] = xp;
  }
}
void launch_cfg_dpmpp(const float* eps, float* latent, float* x0_hist, int h, int W, float s_cfg,
                      const double* coef, const int* k_dev, cudaStream_t s) {
  const long long n = (long long)h * W;
  int blocks = (int)((n + 255) / 256); if (blocks > 1184) blocks = 1184;
  launch_pdl(cfg_dpmpp_kernel, dim3(blocks), dim3(256), 0, s, reinterpret_cast<const float4*>(eps),
             reinterpret_cast<float4*>(latent), reinterpret_cast<float4*>(x0_hist), h, W, s_cfg, coef, k_dev);
}

// Philox4x64-10 (Salmon et al. SC'11): counter (c0, c1, c2, c3), key (k0, k1) -> 4 x 64-bit words
__device__ __forceinline__ void philox4x64_10(unsigned long long c[4], unsigned long long k0, unsigned long long k1) {
  const unsigned long long M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  const unsigned long long W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const unsigned long long hi0 = __umul64hi(M0, c[0]), lo0 = M0 * c[0];
    const unsigned long long hi1 = __umul64hi(M1, c[2]), lo1 = M1 * c[2];
    const unsigned long long n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
    k0 += W0; k1 += W1;
  }
}

__global__ void cfg_ancestral_kernel(const float4* __restrict__ eps, float4* __restrict__ lat, int h, int W, int row0,
                                     float s_cfg, const double* __restrict__ coef, unsigned long long seed,
                                     const int* __restrict__ k_dev) {
  pdl_trigger();
  pdl_wait();
  const int k = *k_dev;
  const float sa = (float)coef[5 * k + 0], s1a = (float)coef[5 * k + 1], sp = (float)coef[5 * k + 2];
  const float ce = (float)coef[5 * k + 3], sig = (float)coef[5 * k + 4];
  const float inv_sa = 1.f / sa;
  const long long n = (long long)h * W;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / W, w = i % W;
    unsigned long long c[4] = {(unsigned long long)((row0 + r) * W + w), (unsigned long long)k, 0ull, 0ull};
    philox4x64_10(c, seed, 0ull);
    double z[4];
#pragma unroll
    for (int j = 0; j < 2; ++j) {                    // Box-Muller in fp64 (reading D24)
      const double u1 = ((double)(c[2 * j] >> 11) + 0.5) * 0x1.0p-53, u2 = (double)(c[2 * j + 1] >> 11) * 0x1.0p-53;
      const double rad = sqrt(-2.0 * log(u1));
      double sn, cs;
      sincospi(2.0 * u2, &sn, &cs);
      z[2 * j] = rad * cs; z[2 * j + 1] = rad * sn;
    }
    const float4 eu = eps[(r * 2 + 0) * W + w], ec = eps[(r * 2 + 1) * W + w];
    float4 x = lat[i];
    const float e[4] = {eu.x + s_cfg * (ec.x - eu.x), eu.y + s_cfg * (ec.y - eu.y),
                        eu.z + s_cfg * (ec.z - eu.z), eu.w + s_cfg * (ec.w - eu.w)};
    float* xv = &x.x;
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      const float x0 = (xv[cc] - s1a * e[cc]) * inv_sa;
      xv[cc] = sp * x0 + ce * e[cc] + sig * (float)z[cc];
    }
    lat[i] = x;
  }
}
void launch_cfg_ancestral(const float* eps, float* latent, int h, int W, int row0, float s_cfg, const double* coef,
                          unsigned long long seed, const int* k_dev, cudaStream_t s) {
  const long long n = (long long)h * W;
  int blocks = (int)((n + 255) / 256); if (blocks > 1184) blocks = 1184;
  launch_pdl(cfg_ancestral_kernel, dim3(blocks), dim3(256), 0, s, reinterpret_cast<const float4*>(eps),
             reinterpret_cast<float4*>(latent), h, W, row0, s_cfg, coef, seed, k_dev);
}

__global__ void step_end_kernel(int* k_dev) {
  pdl_trigger();
  pdl_wait(); *k_dev += 1; }
void launch_step_end(int* k_dev, cudaStream_t s) { launch_pdl(step_end_kernel, dim3(1), dim3(1), 0, s, k_dev); }

// ---- timestep embedding (reading D19) --------------------------------------------------------
// hid[j] = SiLU(W1[j] . sinusoid(tau) + b1[j]) ; emb[b][j] = W2[j] . hid + b2[j] (+ cond[j] if b = 1)
__global__ void temb_hidden_kernel(const float* __restrict__ w1, const float* __restrict__ b1,
                                   const int* __restrict__ taus, const int* __restrict__ k_dev,
                                   int T, int S, float* __restrict__ hid) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float e[];
  const float tau = (float)taus[*k_dev];
  const int half = S / 2;
  for (int j = threadIdx.x; j < half; j += blockDim.x) {
    const double f = exp(-log(10000.0) * (double)j / (double)half);
    const double a = (double)tau * f;
    e[j] = (float)cos(a);
    e[half + j] = (float)sin(a);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (row >= T) return;
  float acc = 0.f;
  for (int i = lane; i < S; i += 32) acc = fmaf(w1[(long long)row * S + i], e[i], acc);
  for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
  if (lane == 0) { const float y = acc + b1[row]; hid[row] = y / (1.f + expf(-y)); }
}
__global__ void temb_out_kernel(const float* __restrict__ w2, const float* __restrict__ b2,
                                const float* __restrict__ cond, const float* __restrict__ hid, int T,
                                float* __restrict__ emb) {
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (row >= T) return;
  float acc = 0.f;
  for (int i = lane; i < T; i += 32) acc = fmaf(w2[(long long)row * T + i], hid[i], acc);
  for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
  if (lane == 0) {
    const float y = acc + b2[row];
    emb[row] = y;
    emb[T + row] = y + cond[row];
  }
}
void launch_temb(const float* w1, const float* b1, const float* w2, const float* b2, const float* cond,
                 const int* taus, const int* k_dev, int T, int S, float* hid, float* emb, cudaStream_t s) {
  launch_pdl(temb_hidden_kernel, dim3((T + 7) / 8), dim3(256), S * sizeof(float), s, w1, b1, taus, k_dev, T, S, hid);
  launch_pdl(temb_out_kernel, dim3((T + 7) / 8), dim3(256), 0, s, w2, b2, cond, hid, T, emb);
}
// out[b][j] = Wt[j] . SiLU(emb[b]) + bt[j]   for every ResBlock's temb projection at once
__global__ void temb_proj_kernel(const float* __restrict__ wt, const float* __restrict__ bt,
                                 const float* __restrict__ emb, int T, int J, float* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float se[];
  for (int i = threadIdx.x; i < 2 * T; i += blockDim.x) { const float y = emb[i]; se[i] = y / (1.f + expf(-y)); }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (row >= J) return;
  float a0 = 0.f, a1 = 0.f;
  for (int i = lane; i < T; i += 32) { const float wv = wt[(long long)row * T + i]; a0 = fmaf(wv, se[i], a0); a1 = fmaf(wv, se[T + i], a1); }
  for (int d = 16; d > 0; d >>= 1) { a0 += __shfl_xor_sync(0xffffffffu, a0, d); a1 += __shfl_xor_sync(0xffffffffu, a1, d); }
  if (lane == 0) { out[row] = a0 + bt[row]; out[J + row] = a1 + bt[row]; }
}
void launch_temb_proj(const float* wt, const float* bt, const float* emb, int T, int J, float* out, cudaStream_t s) {
  launch_pdl(temb_proj_kernel, dim3((J + 7) / 8), dim3(256), 2 * T * sizeof(float), s, wt, bt, emb, T, J, out);
}

// All S steps' temb projections at once (plan / set_cond time): nb <= 8 embedding vectors per pass,
// so the [J][T] matrix is read once per 4 steps instead of once per step.  Same per-vector
// arithmetic and summation order as temb_proj_kernel.  out[v][J], emb[v][T].
__global__ void temb_proj_multi_kernel(const float* __restrict__ wt, const float* __restrict__ bt,
                                       const float* __restrict__ emb, int T, int J, int nb, float* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float se[];
  for (int i = threadIdx.x; i < nb * T; i += blockDim.x) { const float y = emb[i]; se[i] = y / (1.f + expf(-y)); }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (row >= J) return;
  float a[8];
#pragma unroll
  for (int v = 0; v < 8; ++v) a[v] = 0.f;
  for (int i = lane; i < T; i += 32) {
    const float wv = wt[(long long)row * T + i];
#pragma unroll
    for (int v = 0; v < 8; ++v) if (v < nb) a[v] = fmaf(wv, se[v * T + i], a[v]);
  }
#pragma unroll
  for (int v = 0; v < 8; ++v) {
    if (v >= nb) break;
    for (int d = 16; d > 0; d >>= 1) a[v] += __shfl_xor_sync(0xffffffffu, a[v], d);
    if (lane == 0) out[(long long)v * J + row] = a[v] + bt[row];
  }
}
void launch_temb_proj_multi(const float* wt, const float* bt, const float* emb, int T, int J, int nb, float* out, cudaStream_t s) {
  launch_pdl(temb_proj_multi_kernel, dim3((J + 7) / 8), dim3(256), (size_t)nb * T * sizeof(float), s, wt, bt, emb, T, J, nb, out);
}
// per step: tproj <- tproj_all[k] (k = the device step counter)
__global__ void temb_select_kernel(const float* __restrict__ all, const int* __restrict__ k_dev, int n, float* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const float* src = all + (long long)(*k_dev) * n;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = src[i];
}
void launch_temb_select(const float* all, const int* k_dev, int n, float* out, cudaStream_t s) {
  launch_pdl(temb_select_kernel, dim3((unsigned)std::min(148, (n + 255) / 256)), dim3(256), 0, s, all, k_dev, n, out);
}

// ---- segment copier: pack / unpack / loopback exchange ------------------------------------------
// One CTA per segment slice; 16-byte vectors, coalesced.  Segments are 16-byte aligned (rows of
// B*W*C elements with W*C a multiple of 8).
__global__ void copy_segments_kernel(const CopySeg* __restrict__ segs, int nseg) {
  pdl_trigger();
  pdl_wait();
  for (int sidx = blockIdx.y; sidx < nseg; sidx += gridDim.y) {
    const CopySeg sg = segs[sidx];
    const long long nv = (long long)(sg.bytes / 16);
    const uint4* src = reinterpret_cast<const uint4*>(sg.src);
    uint4* dst = reinterpret_cast<uint4*>(sg.dst);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (long long)gridDim.x * blockDim.x)
      dst[i] = src[i];
  }
}
void launch_copy_segments(const CopySeg* segs_dev, int nseg, unsigned long long max_bytes, cudaStream_t s) {
  if (nseg <= 0) return;
  unsigned long long gx = (max_bytes / 16 + 255) / 256;
  if (gx < 1) gx = 1;
  if (gx > 296) gx = 296;
  dim3 grid((unsigned)gx, nseg < 65535 ? nseg : 65535);
  launch_pdl(copy_segments_kernel, dim3(grid), dim3(256), 0, s, segs_dev, nseg);
}

void launch_memset_zero(void* p, size_t bytes, cudaStream_t s) { cudaMemsetAsync(p, 0, bytes, s); }

__global__ void spin_kernel(long long cycles) {
  const long long t0 = clock64();
  while (clock64() - t0 < cycles) {}
}
void launch_spin(long long cycles, cudaStream_t s) { spin_kernel<<<1, 1, 0, s>>>(cycles); }

}  // namespace pcpp
