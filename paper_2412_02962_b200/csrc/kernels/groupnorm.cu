// GroupNorm(32) with fresh local statistics combined with stale global statistics
// (§3.3 "same approach in DistriFusion"; reading D7):
//   m_i  = (sum x, sum x^2) per (b, g) over this rank's fresh patch           [gn_stats]
//   M    = m_i (n=1) | sum_j m_j (sync) | M_{t+1} - m_{i,t+1} + m_i (async)   [gn_apply prologue]
//   y    = SiLU?( gamma (x - mu) / sqrt(var + eps) + beta ),  mu = M1/N, var = max(M2/N - mu^2, 0)
// HBM-bound: stats reads x once, apply reads x once and writes y once (vectorised 16 B accesses).
// Both kernels are deterministic (fixed-order reductions), so loopback and NCCL runs agree bitwise.
#include "../common.cuh"
#include "../kernels.h"

namespace pcpp {

namespace {
constexpr int G = 32;
constexpr int NT = 256;
}

int gn_stats_chunks(int rows, int W) {
  long long tok = (long long)rows * W;
  long long c = tok / 64;                 // at least 64 tokens per chunk
  if (c < 1) c = 1;
  if (c > 128) c = 128;                   // x B = 2 -> up to 256 CTAs (~1.7 waves on 148 SMs)
  return (int)c;
}

template <typename T>
__device__ __forceinline__ void ld8(const ActView& v, int r, int b, int w, int c, float* out) {
  const T* p = reinterpret_cast<const T*>(v.base) + (((long long)r * v.B + b) * v.W + w) * v.C + c;
  load8(p, out);
}

template <typename T>
__global__ void __launch_bounds__(NT) gn_stats_kernel(const GnStatsArgs a) {
  extern __shared__ float red[];                   // [NTL][nv][16]
  __shared__ double chs[2][2560];
  __shared__ bool amlast;
  const int b = blockIdx.y, chunk = blockIdx.x;
  const int W = a.x0.W, rows = a.x0.rows, B = a.x0.B, C = a.C;
  const int nv = C / 8;
  const int vpt = (nv + NT - 1) / NT;              // vectors per thread (1 or 2)
  const int nvl = (nv + vpt - 1) / vpt;            // distinct vector lanes
  const int ntl = NT / nvl;                        // token lanes
  const int tid = threadIdx.x;
  const int vl = tid % nvl, tl = tid / nvl;
  const long long ntok = (long long)rows * W;
  const long long t0 = ntok * chunk / a.nchunk, t1 = ntok * (chunk + 1) / a.nchunk;
  float s[2][8], q[2][8];
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int e = 0; e < 8; ++e) { s[u][e] = 0.f; q[u][e] = 0.f; }
  if (tl < ntl) {
    for (long long t = t0 + tl; t < t1; t += ntl) {
      const int r = (int)(t / W), w = (int)(t % W);
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (u >= vpt) break;
        const int v = vl * vpt + u;
        if (v >= nv) break;
        const int c = v * 8;
        float x[8];
        if (c < a.c0) ld8<T>(a.x0, r, b, w, c, x); else ld8<T>(a.x1, r, b, w, c - a.c0, x);
#pragma unroll
        for (int e = 0; e < 8; ++e) { s[u][e] += x[e]; q[u][e] = fmaf(x[e], x[e], q[u][e]); }
      }
    }
  }
  // per-thread partials -> smem, layout red[(tl*nv + v)*16 + e*2 + {0,1}]
  for (int u = 0; u < vpt; ++u) {
    const int v = vl * vpt + u;
    if (tl < ntl && v < nv)
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        red[((long long)tl * nv + v) * 16 + e * 2 + 0] = s[u][e];
        red[((long long)tl * nv + v) * 16 + e * 2 + 1] = q[u][e];
      }
  }
  __syncthreads();
  for (int c = tid; c < C; c += NT) {                // fixed-order reduction over token lanes
    const int v = c / 8, e = c % 8;
    double ss = 0.0, qq = 0.0;
    for (int l = 0; l < ntl; ++l) {
      ss += red[((long long)l * nv + v) * 16 + e * 2 + 0];
      qq += red[((long long)l * nv + v) * 16 + e * 2 + 1];
    }
    chs[0][c] = ss; chs[1][c] = qq;
  }
  __syncthreads();
  const int cg = C / G;
  if (tid < G) {
    double ss = 0.0, qq = 0.0;
    for (int c = tid * cg; c < (tid + 1) * cg; ++c) { ss += chs[0][c]; qq += chs[1][c]; }
    double* pp = a.partial + (((long long)b * a.nchunk + chunk) * G + tid) * 2;
    pp[0] = ss; pp[1] = qq;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const unsigned total = gridDim.x * gridDim.y;
    amlast = (atomicAdd(a.counter, 1u) == total - 1);
  }
  __syncthreads();
  if (amlast) {
    __threadfence();
    for (int i = tid; i < B * G; i += NT) {
      const int bb = i / G, g = i % G;
      double ss = 0.0, qq = 0.0;
      for (int ch = 0; ch < a.nchunk; ++ch) {
        const volatile double* pp = a.partial + (((long long)bb * a.nchunk + ch) * G + g) * 2;
        ss += pp[0]; qq += pp[1];
      }
      a.m_out[i * 2 + 0] = ss;
      a.m_out[i * 2 + 1] = qq;
    }
    if (tid == 0) *a.counter = 0u;                // ready for the next launch / graph replay
  }
}

void launch_gn_stats(const GnStatsArgs& a, cudaStream_t s) {
  const int nv = a.C / 8;
  const int vpt = (nv + NT - 1) / NT;
  const int nvl = (nv + vpt - 1) / vpt;
  const int ntl = NT / nvl;
  const size_t smem = (size_t)ntl * nv * 16 * sizeof(float);
  dim3 grid(a.nchunk, a.x0.B);
  if (a.x0.dtype == DT_F32) gn_stats_kernel<float><<<grid, NT, smem, s>>>(a);
  else gn_stats_kernel<bf16><<<grid, NT, smem, s>>>(a);
}

void gn_init() {   // dynamic smem <= 40 KB (C <= 2560) on top of 40 KB static
  cudaFuncSetAttribute(gn_stats_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  cudaFuncSetAttribute(gn_stats_kernel<bf16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
}

template <typename TI, typename TO>
__global__ void __launch_bounds__(NT) gn_apply_kernel(const GnApplyArgs a) {
  __shared__ float mu_s[2 * G], rs_s[2 * G];
  const int B = a.x0.B;
  for (int i = threadIdx.x; i < B * G; i += NT) {
    double M1, M2;
    if (a.mode == 0) {
      M1 = a.m_fresh[2 * i]; M2 = a.m_fresh[2 * i + 1];
    } else if (a.mode == 1) {
      M1 = 0.0; M2 = 0.0;
      for (int j = 0; j < a.nranks; ++j) { M1 += a.mall[(j * B * G + i) * 2]; M2 += a.mall[(j * B * G + i) * 2 + 1]; }
    } else {
      M1 = 0.0; M2 = 0.0;
      for (int j = 0; j < a.nranks; ++j) { M1 += a.mall[(j * B * G + i) * 2]; M2 += a.mall[(j * B * G + i) * 2 + 1]; }
      M1 = M1 - a.m_prev[2 * i] + a.m_fresh[2 * i];
      M2 = M2 - a.m_prev[2 * i + 1] + a.m_fresh[2 * i + 1];
    }
    const double mu = M1 / a.count;
    double var = M2 / a.count - mu * mu;
    if (var < 0.0) var = 0.0;
    mu_s[i] = (float)mu;
    rs_s[i] = (float)(1.0 / sqrt(var + 1e-5));
  }
  __syncthreads();
  const int C = a.C, cg = C / G, nv = C / 8;
  const int W = a.x0.W;
  const long long total = (long long)a.x0.rows * B * W * nv;
  for (long long idx = (long long)blockIdx.x * NT + threadIdx.x; idx < total; idx += (long long)gridDim.x * NT) {
    const int v = (int)(idx % nv);
    const long long tok = idx / nv;
    const int w = (int)(tok % W); const long long t2 = tok / W; const int b = (int)(t2 % B); const int r = (int)(t2 / B);
    const int c = v * 8;
    float x[8];
    if (c < a.c0) ld8<TI>(a.x0, r, b, w, c, x); else ld8<TI>(a.x1, r, b, w, c - a.c0, x);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int ch = c + e, g = ch / cg;
      float y = (x[e] - mu_s[b * G + g]) * rs_s[b * G + g] * a.gamma[ch] + a.beta[ch];
      x[e] = a.silu ? silu_f(y) : y;
    }
    TO* po = reinterpret_cast<TO*>(a.out.base) + (((long long)r * a.out.B + b) * a.out.W + w) * a.out.C + c;
    store8(po, x);
  }
}

void launch_gn_apply(const GnApplyArgs& a, cudaStream_t s) {
  const long long total = (long long)a.x0.rows * a.x0.B * a.x0.W * (a.C / 8);
  long long blocks = (total + NT - 1) / NT;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (a.x0.dtype == DT_F32) gn_apply_kernel<float, float><<<(unsigned)blocks, NT, 0, s>>>(a);
  else gn_apply_kernel<bf16, bf16><<<(unsigned)blocks, NT, 0, s>>>(a);
}

}  // namespace pcpp
