// GroupNorm(32) with fresh local statistics combined with stale global statistics
// (§3.3 "same approach in DistriFusion"; reading D7):
//   m_i  = (sum x, sum x^2) per (b, g) over this rank's fresh patch           [gn_stats]
//   M    = m_i (n=1) | sum_j m_j (sync) | M_{t+1} - m_{i,t+1} + m_i (async)   [gn_apply prologue]
//   y    = SiLU?( gamma (x - mu) / sqrt(var + eps) + beta ),  mu = M1/N, var = max(M2/N - mu^2, 0)
// HBM-bound: stats reads x once, apply reads x once and writes y once.  Thread mapping: each thread
// owns fixed 8-channel vectors (16 B) of every token it visits, so its gamma/beta and group ids are
// registers and each warp reads contiguous 16 B vectors of one token row (coalesced).
// Deterministic: fixed-order reductions only (loopback == NCCL bitwise, graph == eager bitwise).
#include <cstdlib>
#include <type_traits>
#include "../common.cuh"
#include "../kernels.h"

namespace pcpp {

namespace {
constexpr int G = 32;
constexpr int NT = 512;

struct Lanes { int nv, vpt, nvl, ntl; };
__host__ __device__ __forceinline__ Lanes lanes_for(int C) {
  Lanes L;
  L.nv = C / 8;
  L.vpt = (L.nv + NT - 1) / NT;          // vectors per thread (1 for C <= 4096)
  L.nvl = (L.nv + L.vpt - 1) / L.vpt;    // distinct vector lanes
  L.ntl = NT / L.nvl;                    // token lanes
  return L;
}
}  // namespace

// CTAs of gn_stats: at most one wave, and >= 2 tokens per token lane (wide C leaves few token lanes per
// CTA: C = 2560 has one, so a fixed 64 tokens per CTA starved the kernel at 32 CTAs -- 54 us for 10 MB)
int gn_stats_chunks(int rows, int W, int C) {
  const long long tok = (long long)rows * 2 * W;
  long long c = tok / (2 * lanes_for(C).ntl);
  if (c < 1) c = 1;
  if (c > 148) c = 148;
  return (int)c;
}

template <typename T>
__device__ __forceinline__ const T* vptr(const ActView& v, long long rowtok, int c) {
  return reinterpret_cast<const T*>(v.base) + rowtok * v.C + c;
}

// ---- stats -------------------------------------------------------------------------------------
// One wave of <= 148 CTAs; CTA `chunk` covers layout tokens [T0, T1) (all (r, b, w) in memory order:
// address T*C + c).  Thread = (fixed 8-channel vector lane, token lane); token lanes stride by ntl
// with 4 independent 16 B loads in flight; per-thread fp32 sums over its few tokens, then a
// fixed-order per-(b, g) reduction in fp64 into the CTA's partial slot partial[chunk][B=2][G][2].
// The slots are summed by gn_finalize (the same finalize as the GEMM-epilogue-fused statistics).
template <typename T>
__global__ void __launch_bounds__(NT) gn_stats_kernel(const GnStatsArgs a) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float red[];                   // [ntl][nv][2 b][8][2]
  const int chunk = blockIdx.x;
  const int W = a.x0.W, B = a.x0.B, C = a.C;
  const Lanes L = lanes_for(C);
  const int tid = threadIdx.x;
  const int vl = tid % L.nvl, tl = tid / L.nvl;
  const long long ntok = (long long)a.x0.rows * B * W;
  const long long T0 = ntok * chunk / a.nchunk, T1 = ntok * (chunk + 1) / a.nchunk;
  const int v = vl * L.vpt;                        // vpt == 1 for every supported C
  if (tl < L.ntl && v < L.nv) {
    float s[2][8], q[2][8];
#pragma unroll
    for (int bb = 0; bb < 2; ++bb)
#pragma unroll
      for (int e = 0; e < 8; ++e) { s[bb][e] = 0.f; q[bb][e] = 0.f; }
    const int c = v * 8;
    const bool second = c >= a.c0;
    const ActView& src = second ? a.x1 : a.x0;
    const int cc = second ? c - a.c0 : c;
    long long Tt = T0 + tl;
    int w = (int)(Tt % W), bq = (int)((Tt / W) % B);
    constexpr int U = sizeof(T) == 2 ? 8 : 4;      // 16-byte loads in flight per thread
    for (; Tt < T1; Tt += (long long)U * L.ntl) {
      float x[U][8];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const long long Tk = Tt + (long long)k * L.ntl;
        if (Tk < T1) load8(vptr<T>(src, Tk, cc), x[k]);
        else {
#pragma unroll
          for (int e = 0; e < 8; ++e) x[k][e] = 0.f;
        }
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        if (bq == 0) {
#pragma unroll
          for (int e = 0; e < 8; ++e) { s[0][e] += x[k][e]; q[0][e] = fmaf(x[k][e], x[k][e], q[0][e]); }
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) { s[1][e] += x[k][e]; q[1][e] = fmaf(x[k][e], x[k][e], q[1][e]); }
        }
        w += L.ntl;
        while (w >= W) { w -= W; bq = (bq + 1 == B) ? 0 : bq + 1; }
      }
    }
#pragma unroll
    for (int bb = 0; bb < 2; ++bb)
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        red[(((long long)tl * L.nv + v) * 2 + bb) * 16 + e * 2 + 0] = s[bb][e];
        red[(((long long)tl * L.nv + v) * 2 + bb) * 16 + e * 2 + 1] = q[bb][e];
      }
  }
  __syncthreads();
  const int cg = C / G;
  if (tid < 2 * G * 2) {                             // fixed-order per-(b, g, stat) sums -> this CTA's slot
    const int bb = tid / (2 * G), g = (tid >> 1) % G, k = tid & 1;
    double acc = 0.0;
    if (bb < B)
      for (int c = g * cg; c < (g + 1) * cg; ++c) {
        const int vv = c / 8, e = c % 8;
        for (int l = 0; l < L.ntl; ++l) acc += red[(((long long)l * L.nv + vv) * 2 + bb) * 16 + e * 2 + k];
      }
    a.partial[(size_t)chunk * 128 + tid] = acc;      // [slot][b][g][2]
  }
}

// ---- finalize of the GEMM-fused statistics ------------------------------------------------------
// CTA (b, g): 128 threads stride over the slots in fp64, then a fixed-order tree.
__global__ void __launch_bounds__(128) gn_finalize_kernel(const double* __restrict__ part, int nslots,
                                                          double* __restrict__ m_out) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x;                  // b * G + g
  double s = 0.0, q = 0.0;
  for (int k = threadIdx.x; k < nslots; k += 128) {
    const double2 v = __ldcg(reinterpret_cast<const double2*>(part + (size_t)k * 128) + i);
    s += v.x; q += v.y;
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) { s += __shfl_xor_sync(0xffffffffu, s, d); q += __shfl_xor_sync(0xffffffffu, q, d); }
  __shared__ double red[4][2];
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { red[warp][0] = s; red[warp][1] = q; }
  __syncthreads();
  if (threadIdx.x == 0) {
    m_out[2 * i] = (red[0][0] + red[1][0]) + (red[2][0] + red[3][0]);
    m_out[2 * i + 1] = (red[0][1] + red[1][1]) + (red[2][1] + red[3][1]);
  }
}

// m_out holds [B][G][2] (B = the rank's CFG batch: 2, or 1 with the CFG device split)
void launch_gn_finalize(const double* part, int nslots, int B, double* m_out, cudaStream_t s) {
  launch_pdl(gn_finalize_kernel, dim3(B * G), dim3(128), 0, s, part, nslots, m_out);
}

// stats pass over x (+ x1 for a channel concat) and the finalize of its per-CTA slots
void launch_gn_stats(const GnStatsArgs& a, cudaStream_t s, bool finalize) {
  const Lanes L = lanes_for(a.C);
  const size_t smem = (size_t)L.ntl * L.nv * 32 * sizeof(float);
  if (a.x0.dtype == DT_F32) launch_pdl(gn_stats_kernel<float>, dim3(a.nchunk), dim3(NT), smem, s, a);
  else launch_pdl(gn_stats_kernel<bf16>, dim3(a.nchunk), dim3(NT), smem, s, a);
  if (finalize) launch_gn_finalize(a.partial, a.nchunk, a.x0.B, a.m_out, s);
}

// ---- apply -------------------------------------------------------------------------------------
// the fresh local sums m[b][g][k] from the producer's slots (nslots <= GN_MERGE_MAX_SLOTS = 48): 4
// threads per entry, each summing every 4th slot in order, then the 4 in fixed order (deterministic);
// CTA 0 publishes them to m_write
__device__ __forceinline__ void gn_slots_sum(const GnApplyArgs& a, double* mf) {
  __shared__ double red[4][128];
  const int e = threadIdx.x & 127, q = threadIdx.x >> 7;     // NT = 512: q in [0, 4)
  // every load of the thread in flight at once (nslots <= 48: at most 12), then summed in slot order
  double v[12];
#pragma unroll
  for (int i = 0; i < 12; ++i) {
    const int k = q + 4 * i;
    v[i] = k < a.nslots ? __ldcg(a.part + (size_t)k * 128 + e) : 0.0;
  }
  double acc = 0.0;
#pragma unroll
  for (int i = 0; i < 12; ++i) acc += v[i];
  red[q][e] = acc;
  __syncthreads();
  if (threadIdx.x < 128) {
    const double v = (red[0][e] + red[1][e]) + (red[2][e] + red[3][e]);
    mf[e] = v;
    if (blockIdx.x == 0 && e < a.x0.B * 2 * G) a.m_write[e] = v;
  }
  __syncthreads();
}

__device__ __forceinline__ void gn_prep(const GnApplyArgs& a, float* mu_s, float* rs_s) {
  const int B = a.x0.B;
  __shared__ double mf_s[128];
  if (a.nslots > 0) gn_slots_sum(a, mf_s);
  const double* mf = a.nslots > 0 ? mf_s : a.m_fresh;
  for (int i = threadIdx.x; i < B * G; i += NT) {
    double M1, M2;
    if (a.mode == 0) {
      M1 = mf[2 * i]; M2 = mf[2 * i + 1];
    } else {
      M1 = 0.0; M2 = 0.0;
      for (int j = 0; j < a.nranks; ++j) { M1 += a.mall[(j * B * G + i) * 2]; M2 += a.mall[(j * B * G + i) * 2 + 1]; }
      if (a.mode == 2) {
        M1 = M1 - a.m_prev[2 * i] + mf[2 * i];
        M2 = M2 - a.m_prev[2 * i + 1] + mf[2 * i + 1];
      }
    }
    const double mu = M1 / a.count;
    double var = M2 / a.count - mu * mu;
    if (var < 0.0) var = 0.0;
    mu_s[i] = (float)mu;
    rs_s[i] = (float)(1.0 / sqrt(var + 1e-5));
  }
}

// Wide apply: every thread of the grid owns one fixed 8-channel vector lane v = gid % nv (so its
// affine coefficients for both CFG branches live in registers) and walks the tokens t = gid / nv,
// + lanes, ... (lanes = threads / nv); consecutive threads read consecutive 16-byte vectors of a
// token row (coalesced) and each keeps 4 independent loads in flight.  One wave of <= 2 CTAs/SM, so
// the statistics prologue is paid once per CTA.
template <typename TI, typename TO>
__global__ void __launch_bounds__(512) gn_apply_wide_kernel(const GnApplyArgs a, int lanes) {
  pdl_trigger();
  pdl_wait();
  __shared__ float mu_s[2 * G], rs_s[2 * G];
  const int B = a.x0.B, C = a.C, cg = C / G, nv = C / 8, W = a.x0.W;
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = gid < lanes * nv;
  const int v = gid % nv;
  const int c = v * 8;
  const bool second = a.x1.base != nullptr && c >= a.c0;
  const TI* src = reinterpret_cast<const TI*>(second ? a.x1.base : a.x0.base) + (second ? c - a.c0 : c);
  const int sC = second ? a.x1.C : a.x0.C;
  TO* dst = reinterpret_cast<TO*>(a.out.base) + c;
  const int ntok = a.x0.rows * B * W;
  // the first 4 token vectors are loaded before the statistics prologue (they do not depend on it)
  float x[4][8];
  int t0 = gid / nv;
  if (active) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int t = t0 + k * lanes;
      if (t < ntok) load8(src + (long long)t * sC, x[k]);
    }
  }
  // the affine parameters are in flight during the statistics prologue too
  float ga8[8], be8[8];
  if (active) { load8(a.gamma + c, ga8); load8(a.beta + c, be8); }
  gn_prep(a, mu_s, rs_s);
  __syncthreads();
  if (!active) return;
  float A[2][8], Bc[2][8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int g = (c + e) / cg;
    const float ga = ga8[e], be = be8[e];
#pragma unroll
    for (int bb = 0; bb < 2; ++bb) {
      const int bi = bb < B ? bb : 0;
      const float rs = rs_s[bi * G + g] * ga;
      A[bb][e] = rs;
      Bc[bb][e] = be - mu_s[bi * G + g] * rs;
    }
  }
  for (;;) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int t = t0 + k * lanes;
      if (t >= ntok) continue;
      const int bb = (t / W) % B;
      float* xv = x[k];
      if (bb) {
#pragma unroll
        for (int e = 0; e < 8; ++e) xv[e] = fmaf(xv[e], A[1][e], Bc[1][e]);
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) xv[e] = fmaf(xv[e], A[0][e], Bc[0][e]);
      }
      if (a.silu) {
#pragma unroll
        for (int e = 0; e < 8; ++e) xv[e] = std::is_same<TO, bf16>::value ? silu_bf16out(xv[e]) : silu_f(xv[e]);
      }
      store8(dst + (long long)t * a.out.C, xv);
    }
    t0 += 4 * lanes;
    if (t0 >= ntok) break;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int t = t0 + k * lanes;
      if (t < ntok) load8(src + (long long)t * sC, x[k]);
    }
  }
}

void launch_gn_apply(const GnApplyArgs& a, cudaStream_t s) {
  const int nv = a.C / 8;
  const long long ntok = (long long)a.x0.rows * a.x0.B * a.x0.W;
  long long blocks = (ntok * nv + 512 * 4 - 1) / (512 * 4);
  if (blocks > 148 * 2) blocks = 148 * 2;
  if (blocks < 1) blocks = 1;
  int lanes = (int)(blocks * 512 / nv);
  if (lanes < 1) { lanes = 1; blocks = (nv + 511) / 512; }
  if (a.x0.dtype == DT_F32) launch_pdl(gn_apply_wide_kernel<float, float>, dim3((unsigned)blocks), dim3(512), 0, s, a, lanes);
  else launch_pdl(gn_apply_wide_kernel<bf16, bf16>, dim3((unsigned)blocks), dim3(512), 0, s, a, lanes);
}

void gn_init() {   // dynamic smem: ntl * nv * 32 floats <= 66 KB (ntl * nv <= 512)
  cudaFuncSetAttribute(gn_stats_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  cudaFuncSetAttribute(gn_stats_kernel<bf16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
}

}  // namespace pcpp
