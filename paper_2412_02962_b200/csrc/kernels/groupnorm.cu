// GroupNorm(32) with fresh local statistics combined with stale global statistics
// (§3.3 "same approach in DistriFusion"; reading D7):
//   m_i  = (sum x, sum x^2) per (b, g) over this rank's fresh patch           [gn_stats]
//   M    = m_i (n=1) | sum_j m_j (sync) | M_{t+1} - m_{i,t+1} + m_i (async)   [gn_apply prologue]
//   y    = SiLU?( gamma (x - mu) / sqrt(var + eps) + beta ),  mu = M1/N, var = max(M2/N - mu^2, 0)
// HBM-bound: stats reads x once, apply reads x once and writes y once.  Thread mapping: each thread
// owns fixed 8-channel vectors (16 B) of every token it visits, so its gamma/beta and group ids are
// registers and each warp reads contiguous 16 B vectors of one token row (coalesced).
// Deterministic: fixed-order reductions only (loopback == NCCL bitwise, graph == eager bitwise).
#include "../common.cuh"
#include "../kernels.h"

namespace pcpp {

namespace {
constexpr int G = 32;
constexpr int NT = 256;

struct Lanes { int nv, vpt, nvl, ntl; };
__host__ __device__ __forceinline__ Lanes lanes_for(int C) {
  Lanes L;
  L.nv = C / 8;
  L.vpt = (L.nv + NT - 1) / NT;          // vectors per thread (1 or 2)
  L.nvl = (L.nv + L.vpt - 1) / L.vpt;    // distinct vector lanes
  L.ntl = NT / L.nvl;                    // token lanes
  return L;
}
}  // namespace

int gn_stats_chunks(int rows, int W) {
  long long tok = (long long)rows * W;
  long long c = tok / 32;                 // >= 32 tokens per chunk
  if (c < 1) c = 1;
  if (c > 128) c = 128;                   // x B = 2 -> up to 256 CTAs
  return (int)c;
}

template <typename T>
__device__ __forceinline__ const T* vptr(const ActView& v, long long rowtok, int c) {
  return reinterpret_cast<const T*>(v.base) + rowtok * v.C + c;
}

// ---- stats -------------------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(NT) gn_stats_kernel(const GnStatsArgs a) {
  extern __shared__ float red[];                   // [ntl][nv][16]
  __shared__ double chs[2][2560];
  __shared__ bool amlast;
  const int b = blockIdx.y, chunk = blockIdx.x;
  const int W = a.x0.W, B = a.x0.B, C = a.C;
  const Lanes L = lanes_for(C);
  const int tid = threadIdx.x;
  const int vl = tid % L.nvl, tl = tid / L.nvl;
  const long long ntok = (long long)a.x0.rows * W;
  const long long t0 = ntok * chunk / a.nchunk, t1 = ntok * (chunk + 1) / a.nchunk;
  float s[2][8], q[2][8];
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int e = 0; e < 8; ++e) { s[u][e] = 0.f; q[u][e] = 0.f; }
  if (tl < L.ntl) {
    long long t = t0 + tl;
    int r = (int)(t / W), w = (int)(t % W);
    for (; t < t1; t += L.ntl) {
      const long long rowtok = ((long long)r * B + b) * W + w;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (u >= L.vpt) break;
        const int v = vl * L.vpt + u;
        if (v >= L.nv) break;
        const int c = v * 8;
        float x[8];
        if (c < a.c0) load8(vptr<T>(a.x0, rowtok, c), x); else load8(vptr<T>(a.x1, rowtok, c - a.c0), x);
#pragma unroll
        for (int e = 0; e < 8; ++e) { s[u][e] += x[e]; q[u][e] = fmaf(x[e], x[e], q[u][e]); }
      }
      w += L.ntl;
      while (w >= W) { w -= W; ++r; }
    }
  }
  for (int u = 0; u < L.vpt; ++u) {
    const int v = vl * L.vpt + u;
    if (tl < L.ntl && v < L.nv)
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        red[((long long)tl * L.nv + v) * 16 + e * 2 + 0] = s[u][e];
        red[((long long)tl * L.nv + v) * 16 + e * 2 + 1] = q[u][e];
      }
  }
  __syncthreads();
  for (int c = tid; c < C; c += NT) {                // fixed-order reduction over token lanes
    const int v = c / 8, e = c % 8;
    double ss = 0.0, qq = 0.0;
    for (int l = 0; l < L.ntl; ++l) {
      ss += red[((long long)l * L.nv + v) * 16 + e * 2 + 0];
      qq += red[((long long)l * L.nv + v) * 16 + e * 2 + 1];
    }
    chs[0][c] = ss; chs[1][c] = qq;
  }
  __syncthreads();
  const int cg = C / G;
  if (tid < 2 * G) {                                  // partial layout [B][G][2][nchunk]
    const int g = tid >> 1, k = tid & 1;
    double acc = 0.0;
    for (int c = g * cg; c < (g + 1) * cg; ++c) acc += chs[k][c];
    a.partial[(((long long)b * G + g) * 2 + k) * a.nchunk + chunk] = acc;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) amlast = (atomicAdd(a.counter, 1u) == gridDim.x * gridDim.y - 1);
  __syncthreads();
  if (!amlast) return;
  __threadfence();
  // last CTA: 2*B*G sums over nchunk partials; warp-per-sum, lane-strided loads, fixed-order tree
  const int warp = tid >> 5, lane = tid & 31;
  for (int i = warp; i < B * G * 2; i += NT / 32) {
    const double* pp = a.partial + (long long)i * a.nchunk;
    double acc = 0.0;
    for (int c = lane; c < a.nchunk; c += 32) acc += __ldcg(pp + c);
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
    if (lane == 0) a.m_out[i] = acc;                  // [B][G][2]
  }
  if (tid == 0) *a.counter = 0u;                      // ready for the next launch / graph replay
}

void launch_gn_stats(const GnStatsArgs& a, cudaStream_t s) {
  const Lanes L = lanes_for(a.C);
  const size_t smem = (size_t)L.ntl * L.nv * 16 * sizeof(float);
  dim3 grid(a.nchunk, a.x0.B);
  if (a.x0.dtype == DT_F32) gn_stats_kernel<float><<<grid, NT, smem, s>>>(a);
  else gn_stats_kernel<bf16><<<grid, NT, smem, s>>>(a);
}

// ---- apply -------------------------------------------------------------------------------------
template <typename TI, typename TO>
__global__ void __launch_bounds__(NT) gn_apply_kernel(const GnApplyArgs a, int tok_per_cta) {
  __shared__ float mu_s[2 * G], rs_s[2 * G];
  const int B = a.x0.B;
  for (int i = threadIdx.x; i < B * G; i += NT) {
    double M1, M2;
    if (a.mode == 0) {
      M1 = a.m_fresh[2 * i]; M2 = a.m_fresh[2 * i + 1];
    } else {
      M1 = 0.0; M2 = 0.0;
      for (int j = 0; j < a.nranks; ++j) { M1 += a.mall[(j * B * G + i) * 2]; M2 += a.mall[(j * B * G + i) * 2 + 1]; }
      if (a.mode == 2) {
        M1 = M1 - a.m_prev[2 * i] + a.m_fresh[2 * i];
        M2 = M2 - a.m_prev[2 * i + 1] + a.m_fresh[2 * i + 1];
      }
    }
    const double mu = M1 / a.count;
    double var = M2 / a.count - mu * mu;
    if (var < 0.0) var = 0.0;
    mu_s[i] = (float)mu;
    rs_s[i] = (float)(1.0 / sqrt(var + 1e-5));
  }
  __syncthreads();
  const int C = a.C, cg = C / G, W = a.x0.W;
  const Lanes L = lanes_for(C);
  const int vl = threadIdx.x % L.nvl, tl = threadIdx.x / L.nvl;
  if (tl >= L.ntl) return;
  // per-thread affine y = x * A[b][e] + Bc[b][e] for its (<= 2) vectors
  float A[2][2][8], Bc[2][2][8];
  int cvec[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int v = vl * L.vpt + u;
    cvec[u] = (u < L.vpt && v < L.nv) ? v * 8 : -1;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int ch = cvec[u] < 0 ? 0 : cvec[u] + e, g = ch / cg;
      const float ga = a.gamma[ch], be = a.beta[ch];
#pragma unroll
      for (int bb = 0; bb < 2; ++bb) {
        const int bi = bb < B ? bb : 0;
        const float rs = rs_s[bi * G + g] * ga;
        A[u][bb][e] = rs;
        Bc[u][bb][e] = be - mu_s[bi * G + g] * rs;
      }
    }
  }
  const long long ntok = (long long)a.x0.rows * B * W;           // (r, b, w) tokens in layout order
  const long long T0 = (long long)blockIdx.x * tok_per_cta;
  const long long T1 = T0 + tok_per_cta < ntok ? T0 + tok_per_cta : ntok;
  long long T = T0 + tl;
  int w = (int)(T % W);
  long long rb = T / W;
  for (; T < T1; T += L.ntl) {
    const int b = (int)(rb % B);
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if (cvec[u] < 0) continue;
      const int c = cvec[u];
      float x[8];
      if (c < a.c0) load8(vptr<TI>(a.x0, T, c), x); else load8(vptr<TI>(a.x1, T, c - a.c0), x);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float y = fmaf(x[e], b ? A[u][1][e] : A[u][0][e], b ? Bc[u][1][e] : Bc[u][0][e]);
        x[e] = a.silu ? silu_f(y) : y;
      }
      // out has the same (r, b, w) geometry; it may be a padded tensor (base = row 0)
      store8(reinterpret_cast<TO*>(a.out.base) + T * a.out.C + c, x);
    }
    w += L.ntl;
    while (w >= W) { w -= W; ++rb; }
  }
}

void launch_gn_apply(const GnApplyArgs& a, cudaStream_t s) {
  const Lanes L = lanes_for(a.C);
  const long long ntok = (long long)a.x0.rows * a.x0.B * a.x0.W;
  long long per = (long long)L.ntl * 8;                           // ~8 tokens per token lane
  long long blocks = (ntok + per - 1) / per;
  if (blocks > 148 * 8) { blocks = 148 * 8; per = (ntok + blocks - 1) / blocks; }
  if (a.x0.dtype == DT_F32) gn_apply_kernel<float, float><<<(unsigned)blocks, NT, 0, s>>>(a, (int)per);
  else gn_apply_kernel<bf16, bf16><<<(unsigned)blocks, NT, 0, s>>>(a, (int)per);
}

void gn_init() {   // dynamic smem <= 40 KB (C <= 2560) on top of 40 KB static
  cudaFuncSetAttribute(gn_stats_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  cudaFuncSetAttribute(gn_stats_kernel<bf16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
}

}  // namespace pcpp
