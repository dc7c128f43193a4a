/*
 * libpcpp -- Partially Conditioned Patch Parallelism (arXiv 2412.02962) on B200 (sm_100a).
 *
 * C ABI.  Plain pointers and sizes only; no torch or C++ types cross this boundary, and no
 * exception crosses it.  Citations: P:<line> §<section> of the paper text.
 *
 * The method (§3, §3.1): the latent x_t in R^{H x W x C} is cut into n horizontal
 * patches of h = H/n rows, one per GPU.  Each GPU runs the denoiser on its own fresh patch; a
 * self-attention layer's keys/values are the local patch plus the lower/upper p*h rows of the
 * neighbouring patches (Eq. 1), taken stale from the previous diffusion step and moved by
 * asynchronous neighbour send/recv (§3.2) instead of DistriFusion's all-gather.  GroupNorm
 * uses fresh local + stale global statistics and conv3x3 uses stale 1-row halos (§3.3).
 * The first `warmup_steps` steps are synchronous.  CFG (Eq. 2, s = 5) runs as batch 2 on
 * every GPU; the sampler is 50-step DDIM.
 *
 * Threading: one plan per GPU per process; calls on one plan are not thread-safe.
 * Streams: all work is enqueued on the plan's compute stream (cfg.stream, or a library-owned
 * stream when NULL); pcpp_step is asynchronous, pcpp_sample synchronises before returning.
 * Errors: every call returns a pcpp_status; pcpp_last_error() gives a thread-local message.
 * A CUDA or NCCL failure poisons the plan: later calls return PCPP_ERR_STATE.
 */
#ifndef PCPP_H_
#define PCPP_H_

#include <stddef.h>

#if defined(__GNUC__)
#define PCPP_API __attribute__((visibility("default")))
#else
#define PCPP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PCPP_OK = 0,
  PCPP_ERR_INVALID = 1,      /* bad argument; nothing was allocated */
  PCPP_ERR_STATE = 2,        /* call out of order (wrong step index, poisoned plan, ...) */
  PCPP_ERR_CUDA = 3,
  PCPP_ERR_NCCL = 4,
  PCPP_ERR_OOM = 5,
  PCPP_ERR_UNSUPPORTED = 6
} pcpp_status;

enum { PCPP_FP32 = 0, PCPP_BF16 = 1 };                       /* precision */
enum { PCPP_SCHEME_PCPP = 0,                                 /* stale partial bands, p2p (§3.2-3.3) */
       PCPP_SCHEME_FULLMAP = 1,                              /* DistriFusion full-map all-gather */
       PCPP_SCHEME_SYNC = 2 };                               /* every step synchronous */
enum { PCPP_MODEL_TINY = 0, PCPP_MODEL_SDXL = 1,            /* config T / SDXL-shaped */
       PCPP_MODEL_TINY_XF = 2, PCPP_MODEL_SDXL_XF = 3 };     /* the same stacks with SDXL's full transformer
                                                                block in every attention layer: LayerNorm,
                                                                self-attention, LayerNorm, cross-attention to a
                                                                77-token context, LayerNorm, GEGLU feed-forward
                                                                (§2.1; DESIGN D25) */
#define PCPP_CTX_LEN 77                                       /* context tokens of the _XF models (D26) */
enum { PCPP_COMM_NCCL = 0,       /* one process per GPU; bands by grouped ncclSend/Recv on a comm stream */
       PCPP_COMM_LOOPBACK = 1,   /* all n virtual ranks in this process on one GPU; transfers = device copies */
       PCPP_COMM_PEER = 2 };     /* one process per GPU; bands as one-sided stores into the peers' device
                                    memory (CUDA IPC mapping: NVLink stores across GPUs) + device flag
                                    barriers -- see pcpp_peer_handle / pcpp_peer_connect */
enum { PCPP_KERNELS_AUTO = 0, PCPP_KERNELS_SIMT = 1 };        /* bf16: tcgen05 kernels (AUTO) or SIMT */

typedef struct pcpp_plan_s* pcpp_plan_t;                     /* opaque; owned by libpcpp */

typedef struct {
  int rank, world;            /* NCCL / PEER: this process's rank, world == n_patches (x 2 with cfg_split).  Rank r owns latent
                                 rows [r*H/n, (r+1)*H/n).  LOOPBACK: ignored (all n virtual ranks
                                 run in this process on one GPU). */
  int num_steps;              /* S (DDIM steps), >= 1; 50 in the paper */
  float guidance_scale;       /* s >= 1 (Eq. 2); 5 in the paper */
  int precision;              /* PCPP_FP32 | PCPP_BF16 (bf16 storage, fp32 accumulate) */
  int scheme;                 /* PCPP_SCHEME_* */
  int model;                  /* PCPP_MODEL_* */
  const float* weights;       /* HOST blob, fp32, manifest order (pcpp_manifest_*); copied into the
                                 plan at pcpp_plan; the caller keeps ownership */
  size_t weights_len;         /* number of floats in the blob; must equal pcpp_weights_len(model) */
  const void* nccl_id;        /* 128-byte ncclUniqueId from pcpp_get_unique_id() on rank 0, broadcast
                                 by the caller (NCCL only) */
  void* stream;               /* cudaStream_t for compute; NULL = library-owned */
  int comm_backend;           /* PCPP_COMM_NCCL | PCPP_COMM_LOOPBACK */
  int kernels;                /* PCPP_KERNELS_AUTO | PCPP_KERNELS_SIMT */
  int use_graphs;             /* 1: replay per-step CUDA graphs ("CUDA Graph"); 0: eager */
  int scheduler;              /* PCPP_SCHED_DDIM (0, default) | PCPP_SCHED_DPMPP2M (1): DPM-Solver++(2M)
                                 on the same timestep ladder (north star "DDIM/DPM-solver"; DESIGN.md
                                 reading D23) | PCPP_SCHED_ANCESTRAL (2): the DDPM ancestral sampler of
                                 Eq. 3-4 on the same ladder (eta = 1, reading D24).
                                 Elementwise and patch-local: no exchange. */
  unsigned long long noise_seed; /* ANCESTRAL: key of the counter-based noise z (Philox4x64-10 on
                                 (global latent token, step); independent of n and of the rank) */
  int cfg_split;              /* 1: the CFG device split of DistriFusion / the paper (§2.2; P:134, P:155:
                                 "4 devices = 2 patches"): world = 2 * n_patches ranks; rank r runs CFG branch
                                 r / n (0 uncond, 1 cond) as batch 1 on patch r % n, exchanges bands / halos /
                                 GN sums within its branch group, and swaps eps with its partner (same patch,
                                 other branch) every step before CFG + DDIM.  PEER / LOOPBACK backends, non-_XF
                                 models (PCPP_ERR_UNSUPPORTED otherwise).  0 (default): CFG as batch 2 on every
                                 rank (reading D11). */
} pcpp_config;

#define PCPP_SCHED_DDIM 0
#define PCPP_SCHED_DPMPP2M 1
#define PCPP_SCHED_ANCESTRAL 2

#define PCPP_MAX_LAYERS 128

typedef struct {
  int n_conv, n_gn, n_attn;             /* exchange-bearing layers per forward */
  int h_latent;                         /* patch rows of the latent, H/n */
  int attn_h[PCPP_MAX_LAYERS];          /* per attention layer: patch rows h_l at its level */
  int attn_r[PCPP_MAX_LAYERS];          /* per attention layer: band rows r_l = rows(p, h_l) (Eq. 1, D1/D3) */
  /* bytes received per step, summed over all ranks, by class {0: attn, 1: conv, 2: gn} */
  long long bytes_async[3];             /* PCPP async step -- closed form */
  long long bytes_warmup[3];            /* synchronous warm-up step */
  long long bytes_fullmap[3];           /* DistriFusion-style async step */
  long long bytes_counted_async[3];     /* counted from the plan's own exchange descriptors (this plan's
                                           scheme, all ranks); valid after pcpp_plan */
  long long bytes_counted_warmup[3];
  double last_step_ms;                  /* device time of the last pcpp_step (CUDA events) */
  long long device_bytes;               /* device memory held by the plan */
  int n_kernels_per_step;               /* kernel launches per step (all virtual ranks) */
  int graphs;                           /* 1 if steps replay CUDA graphs */
  int tc_kernels;                       /* 1 if the tcgen05 contraction kernels are in use */
  double step_flops;                    /* algorithmic flops of one async step (conv/GEMM 2MNK + attention
                                           4 q kv C B), summed over the ranks this plan holds */
  double step_flops_rank_max;           /* the same for the busiest single rank (interior) */
  long long arena_bytes_per_rank;       /* activation tensors of one rank after the liveness-based memory
                                           plan (tensors with disjoint live ranges within a step share
                                           memory; parity-buffered / exchanged / halo tensors pinned) */
  long long arena_bytes_unplanned;      /* the same with every tensor in its own range */
  int simt_fallbacks;                   /* launches of a captured step that asked for the tcgen05 path but ran
                                           the SIMT kernel (unsupported shape); 0 on every SDXL/tiny shape */
  int backend;                          /* effective PCPP_COMM_* (n == 1 always runs LOOPBACK) */
  char comm_lib[192];                   /* NCCL backend: path of the libnccl that was loaded ("" otherwise) */
  long long bytes_eps;                  /* cfg_split: eps bytes swapped between branch partners per step (all ranks) */
} pcpp_info;

/* ---- setup ------------------------------------------------------------------------------- */

/* Fill *cfg with defaults: S = 50, s = 5, BF16, PCPP scheme, SDXL model, LOOPBACK, graphs on. */
PCPP_API void pcpp_config_default(pcpp_config* cfg);

/* Writes a 128-byte ncclUniqueId to out128 (host memory).  Call on rank 0 only. */
PCPP_API pcpp_status pcpp_get_unique_id(void* out128);

/* Weight manifest of a model (D17/D18).  Layouts: conv [Cout][3][3][Cin],
 * linear [out][in], vectors [C]; the blob is their concatenation in manifest order. */
PCPP_API size_t pcpp_weights_len(int model);
PCPP_API int pcpp_manifest_count(int model);
/* entry i: name (NUL-terminated, truncated to name_cap), shape (up to 4 dims), returns ndim or -1 */
PCPP_API int pcpp_manifest_entry(int model, int i, char* name, int name_cap, long long shape[4]);

/* Plan a PCPP run.  H, W, C are LATENT dimensions (e.g. 128, 128, 4 for 1024^2).  Checks, before any
 * allocation (PCPP_ERR_INVALID): 1 <= n <= 8; C == 4; H % (n * 2^(levels-1)) == 0 (SDXL: H % 4n);
 * W % 2^(levels-1) == 0; W a multiple of 8 (tiny) / 32 (SDXL, 16-byte rows at every level);
 * 0 <= p <= 1 (p > 1 is undefined); warmup_steps >= 1 when n > 1 (reading D20);
 * warmup_steps <= num_steps; NCCL: world == n.
 * Allocates the arena, uploads the weights, initialises NCCL (NCCL backend) and (if
 * cfg->use_graphs) captures the per-parity step graphs lazily on first use.  On success *out
 * owns everything; release with pcpp_destroy. */
PCPP_API pcpp_status pcpp_plan(int H, int W, int C, int n_patches, double cond_fraction, int warmup_steps,
                      const pcpp_config* cfg, pcpp_plan_t* out);

/* Host-only planning math (no GPU touched): fills the geometry and closed-form byte fields of
 * *info exactly as pcpp_plan would.  Used by CPU tests. */
PCPP_API pcpp_status pcpp_plan_info(int H, int W, int C, int n_patches, double cond_fraction, int warmup_steps,
                           const pcpp_config* cfg, pcpp_info* info);

/* Host-only: the NCCL issue schedule of rank cfg->rank for one step (sync = warm-up step or not).
 * Writes up to cap records of 5 ints {op (0 send, 1 recv, 2 all-gather), peer (-1 for all-gather),
 * bytes, class (0 attn, 1 conv, 2 gn), group (exchange ordinal; ops of one group are issued inside
 * one ncclGroupStart/End)} in issue order; returns the record count (or -1 on invalid arguments).
 * Every rank issues its groups in the same layer order, so tagless NCCL p2p matching pairs the
 * k-th send a->b with the k-th recv b<-a (App. A). */
PCPP_API int pcpp_plan_schedule(int H, int W, int C, int n_patches, double cond_fraction, int warmup_steps,
                                const pcpp_config* cfg, int sync, int* out, int cap);

/* ---- execution ----------------------------------------------------------------------------- */

/* Set the condition vector c (HOST, temb-dim floats: 1280 SDXL / 512 tiny); the cond branch adds
 * it to the timestep embedding (reading D11).  Copied; asynchronous on the compute stream. */
PCPP_API pcpp_status pcpp_set_cond(pcpp_plan_t plan, const float* cond_host);

/* _XF models only: set the cross-attention context (HOST fp32 [2][PCPP_CTX_LEN][ctx_dim], ctx_dim =
 * 2048 SDXL_XF / 256 TINY_XF; [0] = the unconditional branch's context, [1] = the prompt's; reading
 * D26).  The per-layer context keys/values (ctx W_k, ctx W_v) are computed here, once per context,
 * by the same GEMM kernels -- the context does not change across the S steps.  Must be called before
 * the first pcpp_step / pcpp_sample of an _XF plan (PCPP_ERR_STATE otherwise); PCPP_ERR_INVALID for
 * the other models.  Synchronises the compute stream. */
PCPP_API pcpp_status pcpp_set_context(pcpp_plan_t plan, const float* ctx_host);

/* One denoising step k = t: UNet forward on this rank's patch for both CFG branches (batch 2),
 * the exchanges of §3.2, then CFG (Eq. 2) + DDIM on the patch, in place.
 * latent: DEVICE fp32.  NCCL: this rank's patch [h][W][C].  LOOPBACK: the full map [H][W][C].
 * t must equal the plan's step counter (0 after pcpp_plan / pcpp_reset), else PCPP_ERR_STATE;
 * steps k < warmup_steps run synchronously.  Asynchronous on the compute stream. */
PCPP_API pcpp_status pcpp_step(pcpp_plan_t plan, float* latent, int t);

/* Whole sample: reset, set cond, copy x_T (HOST) in, S steps, gather x_0 (HOST, full [H][W][C]
 * map on every rank).  Host buffers: x_T is this rank's patch (NCCL) or the full map (LOOPBACK).
 * Synchronises before returning. */
PCPP_API pcpp_status pcpp_sample(pcpp_plan_t plan, const float* xT_host, const float* cond_host, float* x0_host);

/* k <- 0; stale buffers are invalidated (the next step is a warm-up step). */
PCPP_API pcpp_status pcpp_reset(pcpp_plan_t plan);

PCPP_API pcpp_status pcpp_query(pcpp_plan_t plan, pcpp_info* out);

/* ---- PEER backend (App. A: one-sided, batched signalling) ---------------------------------
 * After pcpp_plan on every rank: each rank calls pcpp_peer_handle (64 bytes: the CUDA IPC handle of
 * its arena), the caller all-gathers the n handles over any host transport, and each rank calls
 * pcpp_peer_connect with the n handles concatenated in rank order.  Every rank's plan has the same
 * arena layout, so rank i pushes a band to rank j's buffer at the same offset in j's mapping.
 * Protocol per step k: a device barrier (all peers finished step k-1), then the pushes of step k are
 * issued on the comm stream behind their producers and consumed at step k+1 (async steps), or on
 * the compute stream followed by a barrier (warm-up steps).  pcpp_step, pcpp_sample, pcpp_profile
 * (with the exchange kind) and pcpp_destroy are COLLECTIVE for this backend: every rank calls them
 * in the same order.  A barrier that waits > 60 s traps (poisoning the plan).
 * Errors: PCPP_ERR_STATE if the plan is not a PEER plan or is already connected; PCPP_ERR_CUDA if a
 * handle cannot be opened.  pcpp_step before pcpp_peer_connect returns PCPP_ERR_STATE. */
#define PCPP_PEER_HANDLE_BYTES 64
PCPP_API pcpp_status pcpp_peer_handle(pcpp_plan_t plan, void* out64);
PCPP_API pcpp_status pcpp_peer_connect(pcpp_plan_t plan, const void* handles);

/* Per-kind device time of one step, measured in isolation: the ops of `kind_mask` (1 conv/GEMM,
 * 2 attention, 4 GroupNorm, 8 exchanges, 16 other elementwise) of a step of type `sync` are captured
 * alone into a CUDA graph and replayed `iters` times between CUDA events on the plan's stream
 * (after one untimed replay).  Reports the mean ms per step and the algorithmic work of those ops
 * (flops = 2MNK for contractions, 4 q kv C B for attention; bytes = HBM bytes for GroupNorm,
 * exchanged bytes for exchanges).  Does not advance the step counter; buffer contents are left
 * stale -- call pcpp_reset before the next sample.  latent: as for pcpp_step. */
typedef struct { double ms; double flops; double bytes; int launches; } pcpp_prof;
PCPP_API pcpp_status pcpp_profile(pcpp_plan_t plan, float* latent, int kind_mask, int sync, int iters, pcpp_prof* out);

/* COMM_OFF debug mode (SURVEY §8(d) "communication fully hidden"): with on != 0, asynchronous steps
 * (k >= warmup_steps) skip every neighbour exchange -- no NCCL send/recv, no loopback copy -- and
 * read whatever the stale buffers hold, so the step time minus the COMM_OFF step time is the
 * exposed (non-overlapped) communication.  Warm-up steps still exchange.  The results are NOT the
 * method's (stale data stays older than one step): timing only.  Drops cached step graphs; call
 * between steps.  PCPP_ERR_INVALID on a NULL plan. */
PCPP_API pcpp_status pcpp_debug_comm_off(pcpp_plan_t plan, int on);

/* GEMM timeline debug aid: with PCPP_GEMM_TRACE=1 in the environment, every 1-CTA tensor-core GEMM
 * launch records %globaltimer stamps (ns) per CTA into a ring of 32 launches x 148 CTAs x 8 stamps
 * {0 entry, 1 after griddepcontrol.wait, 2 first operand stage landed, 3 last MMA issued, 4 first
 * accumulator ready, 5 epilogue done, 6 exit, 7 unused} (0 where a CTA did not run).  Copies the ring
 * (32 * 148 * 8 u64) to HOST `out` (caller-owned, >= that size), clears it, and returns the number of launches
 * recorded so far (the ring slot of launch i is i % 32), 0 if tracing is off, -1 on a CUDA error. */
PCPP_API int pcpp_debug_gemm_trace(unsigned long long* out);
PCPP_API void pcpp_destroy(pcpp_plan_t plan);
PCPP_API const char* pcpp_last_error(void);

/* ---- kernel-level entry points (testing / benchmarking one hot op through the ABI) -----------
 * All pointers DEVICE, layouts [rows][B][W][C] (C innermost); dtype PCPP_FP32 or PCPP_BF16 for
 * activations; enqueued on `stream` (cudaStream_t, NULL = default).  Return PCPP_ERR_INVALID on
 * unsupported shapes, PCPP_ERR_OOM if a workspace cannot be allocated.  They share one library
 * workspace per device and purpose (split-K / split-KV / GroupNorm partials): do not call them
 * concurrently from several host threads or streams. */

/* conv3x3 (pad 1, stride 1|2) or 1x1 GEMM (taps = 1).  x: [rows_in + 2][B][W_in][Cin] when taps = 9
 * (row 0 and row rows_in+1 are the halo rows), [rows_in][B][W_in][Cin] when taps = 1.
 * w: [Cout][taps][Cin] (dtype of x, or fp32 when x is fp32).  bias fp32 [Cout] (nullable).
 * temb fp32 [B][Cout] (nullable).  res: like y (nullable).  y: [rows_out][B][W_out][Cout].
 * impl: PCPP_KERNELS_AUTO (tcgen05 for bf16 when supported) | PCPP_KERNELS_SIMT. */
PCPP_API pcpp_status pcpp_op_conv(const void* x, int rows_in, int B, int W_in, int Cin, int taps, int stride,
                         const void* w, const float* bias, const float* temb, const void* res, void* y,
                         int Cout, int dtype, int impl, void* stream);

/* Partially conditioned attention over up to 3 K/V row sources (each [rows_s][B][W][2C], K in
 * columns [0,C), V in [C,2C)); q, out: [h][B][W][C]; heads = C/64, scale 1/8. */
PCPP_API pcpp_status pcpp_op_attention(const void* q, const void* const* kv, const int* kv_rows, int nsrc,
                              int h, int B, int W, int C, void* out, int dtype, int impl, void* stream);

/* GroupNorm(32) over x [rows][B][W][C]: m_out[B][32][2] (fp64 local sums); then apply with
 * mode 0 (M = m_out) -> y = SiLU?(gamma (x - mu)/sqrt(var + 1e-5) + beta); count = rows*W*C/32. */
PCPP_API pcpp_status pcpp_op_groupnorm(const void* x, int rows, int B, int W, int C, const float* gamma,
                              const float* beta, int silu, void* y, double* m_out, int dtype, void* stream);

/* Band pack: copy rows [r0, r0 + nrows) of src ([rows][row_bytes]) to dst, contiguous. */
PCPP_API pcpp_status pcpp_op_pack_rows(const void* src, long long row_bytes, int r0, int nrows, void* dst, void* stream);

/* Fused CFG + DDIM update of step k of an S-step schedule: eps [h][2][W][4] fp32, latent [h][W][4]. */
PCPP_API pcpp_status pcpp_op_cfg_ddim(const float* eps, float* latent, int h, int W, float guidance, int num_steps,
                             int k, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PCPP_H_ */
