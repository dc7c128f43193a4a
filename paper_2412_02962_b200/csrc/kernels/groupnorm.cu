// GroupNorm(32) with fresh local statistics combined with stale global statistics
// (§3.3 "same approach in DistriFusion"; reading D7):
//   m_i  = (sum x, sum x^2) per (b, g) over this rank's fresh patch           [gn_stats]
//   M    = m_i (n=1) | sum_j m_j (sync) | M_{t+1} - m_{i,t+1} + m_i (async)   [gn_apply prologue]
//   y    = SiLU?( gamma (x - mu) / sqrt(var + eps) + beta ),  mu = M1/N, var = max(M2/N - mu^2, 0)
// HBM-bound: stats reads x once, apply reads x once and writes y once.  Thread mapping: each thread
// owns fixed 8-channel vectors (16 B) of every token it visits, so its gamma/beta and group ids are
// registers and each warp reads contiguous 16 B vectors of one token row (coalesced).
// Deterministic: fixed-order reductions only (loopback == NCCL bitwise, graph == eager bitwise).
#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include "../common.cuh"
#include "../kernels.h"
#include "../sm100.cuh"

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
// address T*C + c), which are contiguous in memory (per source tensor for a channel concat).  The
// TMA engine streams them into a ring of STATS_NS shared-memory stages of `ts` tokens (1-D bulk
// copies: ~96 KB in flight per SM without holding a register -- the register-load version had ~60 KB
// in flight, stalled on every batch of loads and reached 1.15 TB/s).  Thread = (fixed 8-channel vector
// lane, token lane) reads its 16-byte vectors of each stage from shared memory; per-thread fp32 sums,
// then a fixed-order per-(b, g) reduction in fp64 (4 threads per entry, combined in order) into the
// CTA's partial slot partial[chunk][B=2][G][2].  The slots are summed by gn_finalize (the same
// finalize as the GEMM-epilogue-fused statistics) or by the apply kernel.
constexpr int STATS_NS = 4;
constexpr int STATS_STAGE = 24 * 1024;
__host__ __device__ __forceinline__ int stats_ts(int C, int es) { const int t = STATS_STAGE / (C * es); return t < 1 ? 1 : t; }

template <typename T>
__global__ void __launch_bounds__(NT) gn_stats_kernel(const GnStatsArgs a) {
  pdl_trigger();
  extern __shared__ __align__(128) uint8_t gsm[];
  const int chunk = blockIdx.x;
  const int W = a.x0.W, B = a.x0.B, C = a.C, c0 = a.c0, c1 = C - a.c0;
  const int ts = stats_ts(C, (int)sizeof(T));
  const int SB = ts * C * (int)sizeof(T);
  uint64_t* full = reinterpret_cast<uint64_t*>(gsm + STATS_NS * SB);
  const Lanes L = lanes_for(C);
  const int tid = threadIdx.x;
  const int vl = tid % L.nvl, tl = tid / L.nvl;
  const long long ntok = (long long)a.x0.rows * B * W;
  const long long T0 = ntok * chunk / a.nchunk, T1 = ntok * (chunk + 1) / a.nchunk;
  const int nst = (int)((T1 - T0 + ts - 1) / ts);
  if (tid == 0) {
    for (int i = 0; i < STATS_NS; ++i) sm100::mbar_init(&full[i], 1);
    sm100::fence_barrier_init();
  }
  __syncthreads();
  pdl_wait();
  auto issue = [&](int i) {          // stage i: tokens [T0 + i ts, ...) -> slot i % NS
    const long long t0 = T0 + (long long)i * ts;
    const int n = (int)min((long long)ts, T1 - t0);
    uint8_t* st = gsm + (i % STATS_NS) * SB;
    uint64_t* bar = &full[i % STATS_NS];
    sm100::mbar_arrive_expect_tx(bar, (uint32_t)(n * C * sizeof(T)));
    sm100::bulk_load(st, reinterpret_cast<const T*>(a.x0.base) + t0 * c0, (uint32_t)(n * c0 * sizeof(T)), bar);
    if (c1) sm100::bulk_load(st + (size_t)ts * c0 * sizeof(T), reinterpret_cast<const T*>(a.x1.base) + t0 * c1,
                             (uint32_t)(n * c1 * sizeof(T)), bar);
  };
  if (tid == 0)
    for (int i = 0; i < STATS_NS && i < nst; ++i) issue(i);
  float s[2][8], q[2][8];
#pragma unroll
  for (int bb = 0; bb < 2; ++bb)
#pragma unroll
    for (int e = 0; e < 8; ++e) { s[bb][e] = 0.f; q[bb][e] = 0.f; }
  const int c = vl * 8;
  const bool act = tl < L.ntl && vl < L.nv;
  const bool second = c >= c0;
  for (int i = 0; i < nst; ++i) {
    const long long t0 = T0 + (long long)i * ts;
    const int n = (int)min((long long)ts, T1 - t0);
    sm100::mbar_wait(&full[i % STATS_NS], (uint32_t)((i / STATS_NS) & 1));
    if (act) {
      const T* st = reinterpret_cast<const T*>(gsm + (i % STATS_NS) * SB);
      const T* src = second ? st + (size_t)ts * c0 + (c - c0) : st + c;
      const int sC = second ? c1 : c0;
      for (int t = tl; t < n; t += L.ntl) {
        float x[8];
        load8(src + (size_t)t * sC, x);
        const int bq = (int)(((t0 + t) / W) % B);
        if (bq == 0) {
#pragma unroll
          for (int e = 0; e < 8; ++e) { s[0][e] += x[e]; q[0][e] = fmaf(x[e], x[e], q[0][e]); }
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) { s[1][e] += x[e]; q[1][e] = fmaf(x[e], x[e], q[1][e]); }
        }
      }
    }
    __syncthreads();                               // every thread is done with this slot
    if (tid == 0 && i + STATS_NS < nst) issue(i + STATS_NS);
  }
  // per-thread sums -> smem (the ring is free), then per (b, g, stat) 4 threads in fixed order
  float* red = reinterpret_cast<float*>(gsm);      // [ntl][nv][2 b][8][2]
  if (act) {
#pragma unroll
    for (int bb = 0; bb < 2; ++bb)
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        red[(((long long)tl * L.nv + vl) * 2 + bb) * 16 + e * 2 + 0] = s[bb][e];
        red[(((long long)tl * L.nv + vl) * 2 + bb) * 16 + e * 2 + 1] = q[bb][e];
      }
  }
  __syncthreads();
  __shared__ double part4[4][128];
  const int cg = C / G;
  {
    const int ent = tid & 127, qq = tid >> 7;       // entry (b, g, stat), quarter of the channel range
    const int bb = ent / (2 * G), g = (ent >> 1) % G, k = ent & 1;
    double acc = 0.0;
    if (bb < B)
      for (int cc = g * cg + qq; cc < (g + 1) * cg; cc += 4) {
        const int vv = cc / 8, e = cc % 8;
        for (int l = 0; l < L.ntl; ++l) acc += red[(((long long)l * L.nv + vv) * 2 + bb) * 16 + e * 2 + k];
      }
    part4[qq][ent] = acc;
  }
  __syncthreads();
  if (tid < 128)
    a.partial[(size_t)chunk * 128 + tid] = (part4[0][tid] + part4[1][tid]) + (part4[2][tid] + part4[3][tid]);
}

static size_t stats_smem(int C, int es) {
  const Lanes L = lanes_for(C);
  const size_t ring = (size_t)STATS_NS * stats_ts(C, es) * C * es + STATS_NS * 8;
  const size_t red = (size_t)L.ntl * L.nv * 32 * sizeof(float);
  return ring > red ? ring : red;
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
  if (a.x0.dtype == DT_F32) launch_pdl(gn_stats_kernel<float>, dim3(a.nchunk), dim3(NT), stats_smem(a.C, 4), s, a);
  else launch_pdl(gn_stats_kernel<bf16>, dim3(a.nchunk), dim3(NT), stats_smem(a.C, 2), s, a);
  if (finalize) launch_gn_finalize(a.partial, a.nchunk, a.x0.B, a.m_out, s);
}

// ---- apply -------------------------------------------------------------------------------------
// the fresh local sums m[b][g][k] from the producer's slots (any count; one per producer CTA, <= 148 at
// n = 1): 4 threads per entry, thread q summing slots q, q + 4, ... in order (12 loads in flight per
// batch), then the 4 in fixed order (deterministic); CTA 0 publishes them to m_write.  Summing here
// replaces a gn_finalize launch (one dependent launch per GroupNorm layer).
__device__ __forceinline__ void gn_slots_sum(const GnApplyArgs& a, double* mf) {
  __shared__ double red[4][128];
  const int e = threadIdx.x & 127, q = threadIdx.x >> 7;     // NT = 512: q in [0, 4)
  double acc = 0.0;
  for (int base = 0; base < a.nslots; base += 48) {
    double v[12];
#pragma unroll
    for (int i = 0; i < 12; ++i) {
      const int k = base + q + 4 * i;
      v[i] = k < a.nslots ? __ldcg(a.part + (size_t)k * 128 + e) : 0.0;
    }
#pragma unroll
    for (int i = 0; i < 12; ++i) acc += v[i];
  }
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

// Streaming apply (single-source input): the CTA's contiguous token range moves through a ring of
// STATS_NS shared-memory stages by 1-D bulk copies (TMA engine) -- loads in flight while the
// statistics prologue runs and while earlier stages are transformed -- and every stage is normalised
// in place and leaves by one bulk store.  Thread = fixed 8-channel vector lane (coefficients in
// registers) x token lane.  One CTA per SM.
template <typename T>
__global__ void __launch_bounds__(NT) gn_apply_bulk_kernel(const GnApplyArgs a) {
  pdl_trigger();
  extern __shared__ __align__(128) uint8_t gsm[];
  __shared__ float mu_s[2 * G], rs_s[2 * G];
  const int B = a.x0.B, C = a.C, cg = C / G, W = a.x0.W;
  const int ts = stats_ts(C, (int)sizeof(T));
  const int SB = ts * C * (int)sizeof(T);
  uint64_t* full = reinterpret_cast<uint64_t*>(gsm + STATS_NS * SB);
  const Lanes L = lanes_for(C);
  const int tid = threadIdx.x;
  const int vl = tid % L.nvl, tl = tid / L.nvl;
  const long long ntok = (long long)a.x0.rows * B * W;
  const long long T0 = ntok * blockIdx.x / gridDim.x, T1 = ntok * (blockIdx.x + 1) / gridDim.x;
  const int nst = (int)((T1 - T0 + ts - 1) / ts);
  if (tid == 0) {
    for (int i = 0; i < STATS_NS; ++i) sm100::mbar_init(&full[i], 1);
    sm100::fence_barrier_init();
  }
  __syncthreads();
  pdl_wait();
  const T* xin = reinterpret_cast<const T*>(a.x0.base);
  T* yout = reinterpret_cast<T*>(a.out.base);
  auto issue = [&](int i) {
    const long long t0 = T0 + (long long)i * ts;
    const int n = (int)min((long long)ts, T1 - t0);
    uint64_t* bar = &full[i % STATS_NS];
    sm100::mbar_arrive_expect_tx(bar, (uint32_t)(n * C * sizeof(T)));
    sm100::bulk_load(gsm + (i % STATS_NS) * SB, xin + t0 * C, (uint32_t)(n * C * sizeof(T)), bar);
  };
  if (tid == 0)
    for (int i = 0; i < STATS_NS && i < nst; ++i) issue(i);
  const int c = vl * 8;
  const bool act = tl < L.ntl && vl < L.nv;
  float ga8[8], be8[8];
  if (act) { load8(a.gamma + c, ga8); load8(a.beta + c, be8); }
  gn_prep(a, mu_s, rs_s);                          // overlaps the loads in flight
  __syncthreads();
  float A[2][8], Bc[2][8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int g = act ? (c + e) / cg : 0;
#pragma unroll
    for (int bb = 0; bb < 2; ++bb) {
      const int bi = bb < B ? bb : 0;
      const float rs = rs_s[bi * G + g] * ga8[e];
      A[bb][e] = rs;
      Bc[bb][e] = be8[e] - mu_s[bi * G + g] * rs;
    }
  }
  for (int i = 0; i < nst; ++i) {
    const long long t0 = T0 + (long long)i * ts;
    const int n = (int)min((long long)ts, T1 - t0);
    T* st = reinterpret_cast<T*>(gsm + (i % STATS_NS) * SB);
    sm100::mbar_wait(&full[i % STATS_NS], (uint32_t)((i / STATS_NS) & 1));
    if (act) {
      for (int t = tl; t < n; t += L.ntl) {
        float x[8];
        T* p = st + (size_t)t * C + c;
        load8(p, x);
        const int bq = (int)(((t0 + t) / W) % B);
#pragma unroll
        for (int e = 0; e < 8; ++e) x[e] = fmaf(x[e], bq ? A[1][e] : A[0][e], bq ? Bc[1][e] : Bc[0][e]);
        if (a.silu) {
#pragma unroll
          for (int e = 0; e < 8; ++e) x[e] = std::is_same<T, bf16>::value ? silu_bf16out(x[e]) : silu_f(x[e]);
        }
        store8(p, x);
      }
    }
    sm100::fence_proxy_async_smem();               // the generic writes are visible to the bulk store
    __syncthreads();
    if (tid == 0) {
      sm100::bulk_store(yout + t0 * C, st, (uint32_t)(n * C * sizeof(T)));
      sm100::bulk_commit();
      if (i >= 1 && i - 1 + STATS_NS < nst) {      // slot of stage i - 1: its store has read it -> refill
        sm100::bulk_wait_read<1>();
        issue(i - 1 + STATS_NS);
      }
    }
  }
  if (tid == 0) sm100::bulk_wait_read<0>();        // the stores have read smem (they complete with the grid)
}

void launch_gn_apply(const GnApplyArgs& a, cudaStream_t s) {
  if (!a.x1.base && a.out.dtype == a.x0.dtype && a.out.C == a.C && a.x0.C == a.C) {
    const long long ntok = (long long)a.x0.rows * a.x0.B * a.x0.W;
    const int es = a.x0.dtype == DT_F32 ? 4 : 2;
    const long long stages = (ntok + stats_ts(a.C, es) - 1) / stats_ts(a.C, es);
    const int grid = (int)std::max<long long>(1, std::min<long long>(148, stages));
    const size_t smem = (size_t)STATS_NS * stats_ts(a.C, es) * a.C * es + STATS_NS * 8;
    if (es == 4) launch_pdl(gn_apply_bulk_kernel<float>, dim3(grid), dim3(NT), smem, s, a);
    else launch_pdl(gn_apply_bulk_kernel<bf16>, dim3(grid), dim3(NT), smem, s, a);
    return;
  }

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

void gn_init() {   // dynamic smem: the stage ring (<= 4 x 24 KB + barriers) or the reduction scratch (<= 64 KB)
  cudaFuncSetAttribute(gn_stats_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
  cudaFuncSetAttribute(gn_stats_kernel<bf16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
  cudaFuncSetAttribute(gn_apply_bulk_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
  cudaFuncSetAttribute(gn_apply_bulk_kernel<bf16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
}

}  // namespace pcpp
