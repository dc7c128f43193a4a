// tcgen05 implicit-GEMM conv3x3 / 1x1 (bf16 x bf16 -> fp32 in TMEM), sm_100a.
//
//   D[m][n] = sum_{tap, c} A_tap[m][c] * Wt[n][tap*Cin + c]  (+ bias + temb + residual in the epilogue)
//
// * A (activations, layout [rows][B][W][C]) is loaded by TMA as a 4-D box (64 ch, Wbox, Bbox, Rbox)
//   of 128 output tokens, shifted by the tap (dr, dw): rows come from the padded tensor (halo rows
//   filled by the stale-halo exchange, reading D8), columns outside [0, W) are zero-filled by TMA.
//   The concat input of up-block 1x1 skips is two K ranges from two tensor maps (no concat copy).
// * B (weights [N][taps*Cin], K-major) is a 2-D TMA box (64, BN).
// * Warp roles (192 threads): warp 0 TMA producer, warp 1 MMA issuer (one elected thread issues
//   tcgen05.mma 128 x BN x 16), warps 2-5 epilogue (tcgen05.ld -> fused bias/temb/residual -> bf16).
// * SWIZZLE_128B K-major smem tiles, STAGES-deep mbarrier ring between TMA and MMA.
#include <cuda.h>
#include <cstdio>
#include "../common.cuh"
#include "../kernels.h"
#include "../sm100.cuh"

namespace pcpp {

struct TcGemmParams {
  CUtensorMap ma0, ma1, mb;
  int nk0, nkc, taps, pad, stride;
  int rows_out, w_out, B;
  int Wbox, Bbox, Rbox, nWt, m_tiles;
  int N, n_split;
  unsigned a_bytes;
  const float* bias; const float* temb; int temb_ld;
  ActView res, out, out2;
};

template <int BN>
struct TcCfg {
  static constexpr int A_BYTES = 128 * 128;
  static constexpr int B_BYTES = BN * 128;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int STAGES = (196608 / STAGE) > 8 ? 8 : (196608 / STAGE);
  static constexpr int TMEM_COLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
  static constexpr int SMEM = 1024 + STAGES * STAGE + 256;
};

template <int BN>
__global__ void __launch_bounds__(192, 1) gemm_tc_kernel(const __grid_constant__ TcGemmParams p) {
  using Cfg = TcCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + Cfg::STAGES * Cfg::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE);
  uint64_t* empty = full + Cfg::STAGES;
  uint64_t* tfull = empty + Cfg::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch(&p.ma0); sm100::tma_prefetch(&p.ma1); sm100::tma_prefetch(&p.mb);
    for (int s = 0; s < Cfg::STAGES; ++s) { sm100::mbar_init(&full[s], 1); sm100::mbar_init(&empty[s], 1); }
    sm100::mbar_init(tfull, 1);
    sm100::fence_barrier_init();
  }
  if (warp == 1) sm100::tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
  sm100::fence_before();
  __syncthreads();
  sm100::fence_after();
  const uint32_t tmem = *tmem_slot;

  // output tile -> (r0, b0, w0)
  const int t = blockIdx.x;
  int r0, b0, w0;
  if (p.Bbox == 2) { r0 = t * p.Rbox; b0 = 0; w0 = 0; }
  else { const int wt = t % p.nWt; const int tb = t / p.nWt; b0 = tb % p.B; r0 = tb / p.B; w0 = wt * p.Wbox; }
  const int n0 = blockIdx.y * BN;
  const int nsteps = p.taps * p.nkc;

  if (warp == 0) {
    if (lane == 0) {
      for (int s = 0; s < nsteps; ++s) {
        const int st = s % Cfg::STAGES;
        const uint32_t ph = (s / Cfg::STAGES) & 1;
        sm100::mbar_wait(&empty[st], ph ^ 1);
        const int tap = s / p.nkc, kc = s - tap * p.nkc;
        const int dr = p.taps == 9 ? tap / 3 - 1 : 0, dw = p.taps == 9 ? tap % 3 - 1 : 0;
        sm100::mbar_arrive_expect_tx(&full[st], p.a_bytes + Cfg::B_BYTES);
        if (kc < p.nk0)
          sm100::tma_load_4d(sA + st * Cfg::A_BYTES, &p.ma0, &full[st], kc * 64, w0 * p.stride + dw, b0, r0 * p.stride + dr + p.pad);
        else
          sm100::tma_load_4d(sA + st * Cfg::A_BYTES, &p.ma1, &full[st], (kc - p.nk0) * 64, w0 * p.stride + dw, b0, r0 * p.stride + dr + p.pad);
        sm100::tma_load_2d(sB + st * Cfg::B_BYTES, &p.mb, &full[st], s * 64, n0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = sm100::idesc_bf16(128, BN, 0, 0);
      for (int s = 0; s < nsteps; ++s) {
        const int st = s % Cfg::STAGES;
        const uint32_t ph = (s / Cfg::STAGES) & 1;
        sm100::mbar_wait(&full[st], ph);
        sm100::fence_after();
        const uint32_t a_base = sm100::smem_u32(sA + st * Cfg::A_BYTES);
        const uint32_t b_base = sm100::smem_u32(sB + st * Cfg::B_BYTES);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint64_t ad = sm100::sdesc_sw128(a_base + k * 32, 16, 1024);
          const uint64_t bd = sm100::sdesc_sw128(b_base + k * 32, 16, 1024);
          sm100::mma_bf16_ss(tmem, ad, bd, idesc, (s | k) != 0);
        }
        sm100::mma_commit(&empty[st]);
      }
      sm100::mma_commit(tfull);
    }
  } else {
    // epilogue: warp w reads TMEM lanes [32 (w%4), 32 (w%4) + 32)
    const int q = warp & 3;
    const int m = q * 32 + lane;
    const int wi = m % p.Wbox, bi = (m / p.Wbox) % p.Bbox, ri = m / (p.Wbox * p.Bbox);
    const int r = r0 + ri, b = b0 + bi, w = w0 + wi;
    const bool valid = (m < p.Wbox * p.Bbox * p.Rbox) && r < p.rows_out && w < p.w_out;
    sm100::mbar_wait(tfull, 0);
    sm100::fence_after();
    const bool second = n0 >= p.n_split;
    const ActView& ov = second ? p.out2 : p.out;
    const int ncol0 = second ? n0 - p.n_split : n0;
    const long long orow = (((long long)r * ov.B + b) * ov.W + w) * ov.C + ncol0;
    const long long rrow = p.res.base ? (((long long)r * p.res.B + b) * p.res.W + w) * p.res.C + n0 : 0;
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      uint32_t v[32];
      sm100::tmem_ld32(tmem + (uint32_t(q * 32) << 16) + c, v);
      sm100::tmem_wait_ld();
      if (!valid) continue;
      float f[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(v[i]);
      if (p.bias) {
#pragma unroll
        for (int i = 0; i < 32; ++i) f[i] += __ldg(p.bias + n0 + c + i);
      }
      if (p.temb) {
#pragma unroll
        for (int i = 0; i < 32; ++i) f[i] += __ldg(p.temb + b * p.temb_ld + n0 + c + i);
      }
      if (p.res.base) {
        float rv[8];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          load8(reinterpret_cast<const bf16*>(p.res.base) + rrow + c + 8 * j, rv);
#pragma unroll
          for (int i = 0; i < 8; ++i) f[8 * j + i] += rv[i];
        }
      }
      if (ov.dtype == DT_BF16) {
        bf16* po = reinterpret_cast<bf16*>(ov.base) + orow + c;
#pragma unroll
        for (int j = 0; j < 4; ++j) store8(po + 8 * j, f + 8 * j);
      } else {
        float* po = reinterpret_cast<float*>(ov.base) + orow + c;
#pragma unroll
        for (int j = 0; j < 4; ++j) store8(po + 8 * j, f + 8 * j);
      }
    }
  }
  sm100::fence_before();
  __syncthreads();
  if (warp == 1) sm100::tmem_dealloc<Cfg::TMEM_COLS>(tmem);
}

// ---------------------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn f = nullptr;
  if (!f) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      f = reinterpret_cast<EncodeTiledFn>(p);
  }
  return f;
}

bool tc_available() { return encode_fn() != nullptr; }
void* tma_encode_fn() { return reinterpret_cast<void*>(encode_fn()); }

// 4-D map over a [rows(+2 pad)][B][W][C] bf16 activation tensor; box (64, Wbox, Bbox, Rbox) output
// tokens.  Stride-2 convs use TMA element strides 2 along W and rows: the box spans 2*Wbox x 2*Rbox
// input elements and delivers every second one (Wbox x Rbox), so A stays one dense SW128 tile.
static bool encode_act(CUtensorMap* m, const ActView& v, int pad, int Wbox, int Bbox, int Rbox, int stride) {
  const size_t es = 2;
  char* base = reinterpret_cast<char*>(v.base) - (size_t)pad * v.B * v.W * v.C * es;
  cuuint64_t dims[4] = {(cuuint64_t)v.C, (cuuint64_t)v.W, (cuuint64_t)v.B, (cuuint64_t)(v.rows + 2 * pad)};
  cuuint64_t strides[3] = {(cuuint64_t)v.C * es, (cuuint64_t)v.W * v.C * es, (cuuint64_t)v.B * v.W * v.C * es};
  cuuint32_t box[4] = {64, (cuuint32_t)(Wbox * stride), (cuuint32_t)Bbox, (cuuint32_t)(Rbox * stride)};
  cuuint32_t estr[4] = {1, (cuuint32_t)stride, 1, (cuuint32_t)stride};
  return encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
static bool encode_w(CUtensorMap* m, const void* w, int K, int N, int BN) {
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)N};
  cuuint64_t strides[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)BN};
  cuuint32_t estr[2] = {1, 1};
  return encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(w), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int pick_bn(const GemmArgs& g) {
  const int cands[4] = {256, 160, 128, 64};
  for (int bn : cands) {
    if (g.N % bn) continue;
    if (g.n_split < g.N && g.n_split % bn) continue;
    return bn;
  }
  return 0;
}

bool gemm_tc_supported(const GemmArgs& g) {
  if (!tc_available()) return false;
  if (g.a0.dtype != DT_BF16 || g.wdtype != DT_BF16) return false;
  if (g.a1.base && g.a1.dtype != DT_BF16) return false;
  if (g.stride != 1 && !(g.stride == 2 && g.taps == 9)) return false;
  if (g.cin % 64 || g.c0 % 64) return false;
  if (g.out.dtype != DT_BF16 && g.out.dtype != DT_F32) return false;
  if (g.res.base && g.res.dtype != DT_BF16) return false;
  if (g.out2.base && g.out2.dtype != g.out.dtype) return false;
  if (!pick_bn(g)) return false;
  if (g.B != 2 && g.w_out < 128) return false;
  return true;
}

template <int BN>
static void launch_bn(const TcGemmParams& p, cudaStream_t s) {
  dim3 grid(p.m_tiles, p.N / BN);
  gemm_tc_kernel<BN><<<grid, 192, TcCfg<BN>::SMEM, s>>>(p);
}

void gemm_tc_init() {
  cudaFuncSetAttribute(gemm_tc_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcCfg<256>::SMEM);
  cudaFuncSetAttribute(gemm_tc_kernel<160>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcCfg<160>::SMEM);
  cudaFuncSetAttribute(gemm_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcCfg<128>::SMEM);
  cudaFuncSetAttribute(gemm_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcCfg<64>::SMEM);
}

bool launch_gemm_tc(const GemmArgs& g, cudaStream_t s) {
  TcGemmParams p;
  memset(&p, 0, sizeof p);
  const int BN = pick_bn(g);
  // tile geometry: 128 output tokens = Wbox x Bbox x Rbox in (w, b, r) layout order
  if (g.w_out >= 128) { p.Wbox = 128; p.Bbox = 1; p.Rbox = 1; }
  else if (g.B == 2 && 128 % (2 * g.w_out) == 0) { p.Wbox = g.w_out; p.Bbox = 2; p.Rbox = 128 / (2 * g.w_out); }
  else { p.Wbox = g.w_out; p.Bbox = 1; p.Rbox = 1; }
  p.nWt = (g.w_out + p.Wbox - 1) / p.Wbox;
  if (p.Bbox == 2) p.m_tiles = (g.rows_out + p.Rbox - 1) / p.Rbox;
  else p.m_tiles = g.rows_out * g.B * p.nWt;
  p.taps = g.taps; p.pad = g.taps == 9 ? 1 : 0; p.stride = g.stride;
  p.nkc = g.cin / 64; p.nk0 = g.c0 / 64;
  p.rows_out = g.rows_out; p.w_out = g.w_out; p.B = g.B;
  p.N = g.N; p.n_split = g.n_split < g.N ? g.n_split : (1 << 30);
  p.a_bytes = 128u * p.Wbox * p.Bbox * p.Rbox;
  p.bias = g.bias; p.temb = g.temb; p.temb_ld = g.temb_ld;
  p.res = g.res; p.out = g.out; p.out2 = g.out2;
  if (!encode_act(&p.ma0, g.a0, p.pad, p.Wbox, p.Bbox, p.Rbox, g.stride)) return false;
  if (!encode_act(&p.ma1, g.a1.base ? g.a1 : g.a0, p.pad, p.Wbox, p.Bbox, p.Rbox, g.stride)) return false;
  if (!encode_w(&p.mb, g.w, g.taps * g.cin, g.N, BN)) return false;
  switch (BN) {
    case 256: launch_bn<256>(p, s); break;
    case 160: launch_bn<160>(p, s); break;
    case 128: launch_bn<128>(p, s); break;
    default: launch_bn<64>(p, s); break;
  }
  return true;
}

}  // namespace pcpp
