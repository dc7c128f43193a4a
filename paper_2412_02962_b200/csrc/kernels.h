// Internal launcher interface between the runtime (plan/exec) and the kernels.
// Activation layout everywhere: [rows][B][W][C], C innermost (SURVEY §8(a) "Layouts"):
// a band of rows over both CFG branches is one contiguous range, and C is the
// contiguous K dimension of every contraction.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstddef>

namespace pcpp {

struct ActView {
  void* base = nullptr;   // element (r,b,w,c) at base + (((r*B + b)*W + w)*C + c) * esize;
                          // r may be -1 / rows for padded (halo-carrying) tensors
  int rows = 0, B = 0, W = 0, C = 0;
  int dtype = 0;          // DT_F32 / DT_BF16
};

// D[m][n] = sum_tap sum_c A_tap[m][c] * Wt[n][tap*Cin + c]  (+ bias[n] + temb[b][n] + res[m][n])
// m enumerates output tokens (r, b, w) in layout order; tap (dr, dw) in row-major 3x3 order.
struct GemmArgs {
  ActView a0, a1;         // K-channel sources: channels [0, c0) from a0, [c0, Cin) from a1
  int c0 = 0;             // == a0.C ; a1.base == nullptr when single-source
  int cin = 0;            // total input channels
  int taps = 1;           // 1 (1x1) or 9 (3x3, padding 1 through halo rows + zero columns)
  int stride = 1;         // 1 or 2
  int rows_out = 0, w_out = 0, B = 0;
  const void* w = nullptr; int wdtype = 0;   // [N][taps*cin]
  int N = 0;
  const float* bias = nullptr;               // [N]
  const float* temb = nullptr; int temb_ld = 0;   // temb[b*temb_ld + n]
  ActView res;                               // residual with out's geometry (base==nullptr: none)
  ActView out, out2; int n_split = 1 << 30;  // cols >= n_split -> out2[col - n_split]
  float* ws = nullptr; size_t ws_elems = 0;  // split-K fp32 workspace (optional)
  // optional fused GroupNorm(32) statistics of `out` (tcgen05 path only): partial sums land in
  // gn_part [slots][B=2][G=32][2] fp64 and *gn_slots (host) receives the slot count, 0 if the
  // launch did not produce them (the consumer then runs the standalone stats kernel)
  double* gn_part = nullptr; int* gn_slots = nullptr;
  // GEGLU epilogue (the _XF feed-forward, reading D25): D has N columns in 64-column blocks
  // [value 64 | gate 64] (the builder interleaves W_ff1's rows); out gets N / 2 columns
  // out[:, 64 k + j] = (D[:, 128 k + j] + bias) * gelu(D[:, 128 k + 64 + j] + bias)
  int geglu = 0;
};
void launch_gemm_simt(const GemmArgs& g, cudaStream_t s);

// conv3x3 with N = 4 (conv_out): out fp32 [rows][B][W][4]
void launch_conv_out(const ActView& in, const float* w /*[4][9*Cin] fp32*/, const float* bias,
                     const ActView& out, cudaStream_t s);

// Partially conditioned attention: Q from the local patch; K/V from up to 3 row
// sources [top band ; local ; bottom band] each laid out [rows][B][W][2C] (K cols [0,C), V [C,2C)).
// nkeys > 0: only the first nkeys keys (token order r * W + w) of the source are attended (the
// 77-token cross-attention context, padded to whole rows); 0 = all rows * W keys.
struct AttnSrc { const void* kv = nullptr; int rows = 0; int nkeys = 0; };
struct AttnArgs {
  const void* q = nullptr;    // [h][B][W][C]
  AttnSrc src[3]; int nsrc = 0;
  int h = 0, B = 0, W = 0, C = 0;
  void* out = nullptr;        // [h][B][W][C]
  int dtype = 0;
  float* ws = nullptr; size_t ws_elems = 0;   // split-KV fp32 workspace (optional)
};
void launch_attn_simt(const AttnArgs& a, cudaStream_t s);

// GroupNorm(32).  Stats: fresh local sums m[b][g][{sum, sumsq}] (fp64) of the rank's patch.
struct GnStatsArgs {
  ActView x0, x1; int c0 = 0; int C = 0;
  double* partial = nullptr;     // [nchunk][2][G][2] scratch (per-CTA slots, summed by gn_finalize)
  double* m_out = nullptr;       // [B][G][2]
  int nchunk = 0;
};
void launch_gn_stats(const GnStatsArgs& a, cudaStream_t s, bool finalize = true);   // finalize: m_out from the slots
// m_out[b][g][k] = sum over slots of part[slot][b][g][k] (fp64, fixed order): the finalize of the
// GEMM-epilogue-fused statistics
void launch_gn_finalize(const double* part, int nslots, int B, double* m_out, cudaStream_t s);
int gn_stats_chunks(int rows, int W, int C);
void gn_init();

// mode 0: M = m_fresh (n = 1)
// mode 1: M = sum_j mall[j]                           (warm-up / sync: fresh global)
// mode 2: M = sum_j mall_prev[j] - m_prev + m_fresh  (async: stale global, corrected, reading D7)
struct GnApplyArgs {
  ActView x0, x1; int c0 = 0; int C = 0;
  ActView out;
  const float* gamma = nullptr; const float* beta = nullptr; int silu = 0;
  int mode = 0; int nranks = 1;
  const double* m_fresh = nullptr; const double* m_prev = nullptr; const double* mall = nullptr;
  double count = 0;              // N = H_l W_l C/G (global)
  // nslots > 0: m_fresh is not read but summed here from the producer's per-CTA partial slots
  // part[slot][B=2][G][2] (fixed order; no finalize launch), and CTA 0 writes it to m_write
  const double* part = nullptr; int nslots = 0; double* m_write = nullptr;
};
void launch_gn_apply(const GnApplyArgs& a, cudaStream_t s);

// SDXL transformer block (kernels/xformer.cu; reading D25): LayerNorm of every token over its C
// channels (false if C is unsupported); GEGLU gate out[:, 64k + j] = u[:, 128k + j] * gelu(u[:, 128k + 64 + j])
// (u in the blocked [value 64 | gate 64] column order of the interleaved W_ff1); the context
// [B][L][D] fp32 laid out as the rows of a [rows][B][W][D] key source (keys >= L zero)
bool launch_layernorm(const ActView& x, const ActView& y, const float* gamma, const float* beta, cudaStream_t s);
void launch_geglu(const ActView& u, const ActView& out, cudaStream_t s);
void launch_ctx_layout(const float* ctx, const ActView& out, int L, cudaStream_t s);

// latent [h][W][4] fp32 -> padded xin [h][2][W][4] fp32 (both CFG branches)
void launch_prep_latent(const float* latent, const ActView& xin, cudaStream_t s);
// nearest x2: in [h][B][W][C] -> out [2h][B][2W][C]
void launch_upsample2(const ActView& in, const ActView& out, cudaStream_t s);
// Eq. 2 + DDIM: eps [h][2][W][4] fp32; latent [h][W][4] fp32 in place; coef[k*4 + {sa,s1a,sp,s1p}]
void launch_cfg_ddim(const float* eps, float* latent, int h, int W, float s_cfg,
                     const double* coef, const int* k_dev, cudaStream_t s);
// Eq. 2 + DPM-Solver++(2M) (reading D23): x0 = (x - sigma eps) / alpha; x <- A x + Bc (w0 x0 + w1 x0_hist);
// x0_hist <- x0.  coef[k*6 + {1/alpha, sigma, A, Bc, w0, w1}]
void launch_cfg_dpmpp(const float* eps, float* latent, float* x0_hist, int h, int W, float s_cfg,
                      const double* coef, const int* k_dev, cudaStream_t s);
// Eq. 2 + the ancestral sampler (Eq. 3-4 as eta = 1 on the ladder, reading D24): x <- sqrt(ab') x0 +
// c_eps eps + sigma z, z = Box-Muller(Philox4x64-10((row0 + r) * W + w, k, 0, 0; key (seed, 0))).
// coef[k*5 + {sqrt(ab), sqrt(1-ab), sqrt(ab'), c_eps, sigma}]; row0 = global row of the patch.
void launch_cfg_ancestral(const float* eps, float* latent, int h, int W, int row0, float s_cfg, const double* coef,
                          unsigned long long seed, const int* k_dev, cudaStream_t s);
void launch_step_end(int* k_dev, cudaStream_t s);

// timestep embedding: emb[b][T] for tau = taus[*k_dev]; then tproj[b][j] for all ResBlocks
void launch_temb(const float* w1, const float* b1, const float* w2, const float* b2,
                 const float* cond, const int* taus, const int* k_dev, int T, int S,
                 float* hid /*[T]*/, float* emb /*[2][T]*/, cudaStream_t s);
void launch_temb_proj(const float* wt /*[J][T]*/, const float* bt, const float* emb, int T, int J,
                      float* out /*[2][J]*/, cudaStream_t s);
void launch_temb_proj_multi(const float* wt, const float* bt, const float* emb, int T, int J, int nb, float* out,
                            cudaStream_t s);
void launch_temb_select(const float* all, const int* k_dev, int n, float* out, cudaStream_t s);

// pack / unpack / loopback exchange: many contiguous 16-byte-multiple segments in one launch
struct CopySeg { const void* src; void* dst; unsigned long long bytes; };
void launch_copy_segments(const CopySeg* segs_dev, int nseg, unsigned long long max_bytes, cudaStream_t s);

// PEER backend barrier (kernels/peer.cu): every rank publishes ++(*epoch) into remote[j] (= peer j's
// flags[me]) and waits until flags[j] >= epoch for every peer j != me.
struct PeerBarrier {
  unsigned long long* epoch = nullptr;         // local counter (this rank's arena)
  const unsigned long long* flags = nullptr;   // local [n], written by the peers
  unsigned long long* remote[8] = {};          // peer j's flags[me] (IPC-mapped)
  int n = 1, me = 0;
};
void launch_peer_barrier(const PeerBarrier& b, cudaStream_t s);

void launch_memset_zero(void* p, size_t bytes, cudaStream_t s);
// one thread spinning ~cycles clocks (delay injection on the comm stream, tests only)
void launch_spin(long long cycles, cudaStream_t s);

}  // namespace pcpp
