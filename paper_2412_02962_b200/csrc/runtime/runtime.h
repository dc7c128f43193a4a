// libpcpp runtime: plan (layer program + memory layout + weights), exchange descriptors,
// executor (eager or CUDA-graph replay), NCCL / loopback backends.
#pragma once
#include <cuda_runtime.h>
#include <string>
#include <vector>
#include <memory>
#include "../common.cuh"
#include "../kernels.h"
#include "../../../include/pcpp.h"

namespace pcpp {

constexpr int GN_G = 32;
constexpr int B_CFG = 2;

// ---- tensors ------------------------------------------------------------------------------------
struct TDesc {
  std::string name;
  int level = 0, rows = 0, W = 0, C = 0, dtype = 0;
  int B = 0;         // batch of the tensor (0: the plan's batch per rank, P.B)
  int pad = 0;       // 1: rows -1 and `rows` exist (conv halo rows, zero at image borders)
  int dbl = 0;       // 1: one buffer per step parity (its rows are sent to neighbours)
  int xdst = 0;      // 1: written by other ranks inside a step (own memory range, never shared)
  size_t bytes = 0;  // per parity, including halo rows
  size_t off[2] = {0, 0};   // offsets in the rank arena
};

// ---- ops ------------------------------------------------------------------------------------------
enum OpK { OP_TEMB, OP_PREP, OP_HALO, OP_CONV, OP_GEMM, OP_GN, OP_KVX, OP_ATTN, OP_UPS, OP_CONVOUT,
           OP_CFGDDIM, OP_END, OP_LN, OP_GEGLU, OP_XATTN, OP_EPSX };

struct Op {
  OpK k;
  int in0 = -1, in1 = -1, out = -1, out2 = -1, res = -1;
  int stride = 1, taps = 1, silu = 0;
  int n_split = 1 << 30;
  long long w = -1;         // element offset into wmat (or wf32 when w_f32)
  int w_f32 = 0;
  long long b = -1, g = -1, be = -1;   // element offsets into wf32 (bias, gamma, beta)
  int temb_off = -1;        // column offset into tproj [2][J]
  int xid = -1;             // exchange id (halo / gn / attn index)
  int N = 0;                // output channels for GEMM/CONV
  int gn_fuse = -1;         // GEMM/CONV: GroupNorm index whose statistics its epilogue produces
  int geglu = 0;            // GEMM: GEGLU epilogue (out has N/2 channels); tmp = the [.., N] fallback tensor
  int tmp = -1;
};

// ---- exchange buffers --------------------------------------------------------------------------
struct HaloX { int t; int stride; };
struct GnX   { int C; int rows, W; size_t off_m[2], off_mall[2], off_part; int nchunk; double count; };
struct AttnX { int kv; int level; int h, W, C; int r; size_t off_top[2], off_bot[2]; size_t off_gat[2]; };
// cross-attention of an _XF layer: keys/values of the context, [ctx_rows(level)][B][W_l][2C] (global,
// shared by the virtual ranks), produced at pcpp_set_context by a GEMM of the level's laid-out context
struct XAttnX { int level, C; long long w; void* kv = nullptr; };

// A symbolic buffer reference, resolved per rank to a device pointer.
enum BufKind { BK_TENSOR, BK_TOP, BK_BOT, BK_GAT, BK_GNM, BK_GNMALL };
struct BufRef { int kind; int id; int par; long long byte_off; };
// One transfer of a step's exchange (global view over all ranks).
struct Xfer { int cls; int src_rank, dst_rank; BufRef src, dst; size_t bytes; };
// How a backend should realise one exchange point.
struct XGroup {
  int cls = 0;                   // 0 attn, 1 conv, 2 gn
  int allgather = 0;             // NCCL: one ncclAllGather instead of p2p
  BufRef ag_send{}, ag_recv{};   // allgather buffers (own rank)
  size_t ag_bytes = 0;           // per-rank contribution
  std::vector<Xfer> remote;      // cross-rank data (also the counted ledger)
  std::vector<Xfer> local;       // post-exchange local copies (dual halo write, band unpack)
  int wait = 0;                  // consumer needs it this step (sync)
};

struct NcclApi;   // dlopen'd NCCL entry points

struct RankMem { char* arena = nullptr; size_t bytes = 0; };

struct Plan {
  // configuration
  int H = 0, W = 0, C = 0, n = 1, warmup = 1, S = 50;
  double p = 0.0;
  pcpp_config cfg{};
  int dtype = DT_BF16;
  int levels = 1, C0 = 128, T = 512, SIN = 128;
  int nr = 1;            // virtual ranks held here (world for loopback, 1 for NCCL / PEER)
  // CFG device split (cfg_split, §2.2): 2 groups of n ranks, group b runs CFG
  // branch b (b = 0 uncond, 1 cond) as batch 1 over the n patches; rank r = b * n + patch
  bool split = false;
  int B = 2;             // CFG batch per rank (2, or 1 with the split)
  int nb = 1;            // branch groups (2 with the split)
  int world = 1;         // n * nb
  int patch_of(int r) const { return r % n; }
  int branch_of(int r) const { return split ? r / n : 0; }
  int grank(int b, int i) const { return b * n + i; }
  int rank0 = 0;         // global rank of virtual rank 0
  bool loopback = true;
  // loopback test mode (PCPP_LOOPBACK_ASYNC=1): the exchange copies run on the comm stream S1 with the
  // NCCL backend's event protocol (one step of slack), optionally behind a per-exchange spin of
  // PCPP_XCH_DELAY x (1..5) k-cycles (delay injection: the results must not change)
  bool xasync = false; long long xdelay = 0;
  bool comm_off = false;
  size_t arena_tensor_bytes = 0;     // activation part of the rank arena after the memory plan             // pcpp_debug_comm_off: async steps skip their exchanges
  bool use_tc = false;

  // program
  std::vector<TDesc> td;
  std::vector<Op> ops;
  std::vector<HaloX> halos;
  std::vector<GnX> gns;
  std::vector<AttnX> attns;
  std::vector<XAttnX> xattns;
  bool xf = false; int ctx_dim = 0; bool ctx_set = false;
  float* ctx_f32 = nullptr;                 // [2][77][ctx_dim] as given
  void* ctx_level[3] = {nullptr, nullptr, nullptr};   // laid-out context per level [ctx_rows][2][W_l][ctx_dim]
  int ctx_rows(int level) const { const int Wl = W >> level; return (77 + Wl - 1) / Wl; }
  int J = 0;             // total temb projection width (sum of ResBlock Cout)
  // manifest
  std::vector<std::string> man_name;
  std::vector<std::vector<long long>> man_shape;
  std::vector<long long> man_off;
  size_t blob_len = 0;
  // weight upload list: (blob_off, numel, to_f32_arena, arena_off)
  struct Up { long long blob_off, numel; int f32; long long off; };
  std::vector<Up> uploads;
  long long wmat_len = 0, wf32_len = 0;
  // temb parameter offsets (wf32)
  long long t_w1 = 0, t_b1 = 0, t_w2 = 0, t_b2 = 0, t_wt = 0, t_bt = 0;

  // per-rank memory
  size_t rank_bytes = 0;
  size_t off_epart = 0;                 // per-rank GEMM-fused GN statistics partials
  std::vector<int> gn_slots;            // [nr][ngn]: slots the producer GEMM wrote (0: not fused)
  std::vector<RankMem> rm;
  // global memory
  void* wmat = nullptr;  float* wf32 = nullptr;
  float* emb = nullptr; float* hid = nullptr; float* tproj = nullptr; float* cond = nullptr;
  int* taus = nullptr; double* coef = nullptr; int* k_dev = nullptr;
  float* tproj_all = nullptr; float* emb_all = nullptr; int* kseq = nullptr;   // [S][2][J] temb projections, precomputed
  double* coef_dpm = nullptr;   // DPM-Solver++(2M): [S][6] {1/alpha, sigma, sigma'/sigma, -alpha'(e^-h - 1), w0, w1}
  float* x0_hist = nullptr;     // DPM-Solver++(2M) data-prediction history, [nr][h][W][4] fp32
  double* coef_anc = nullptr;   // ancestral (eta = 1): [S][5] {sqrt(ab), sqrt(1-ab), sqrt(ab'), c_eps, sigma}
  float* ws = nullptr; size_t ws_elems = 0;   // split-K workspace
  std::vector<cudaEvent_t> op_ev; bool op_ev_on = false;   // per-op timing (PCPP_OP_TIMING, pcpp_profile)
  std::vector<void*> gallocs;

  // exchange descriptors: [sync][par] per exchange op index
  std::vector<XGroup> xg[2][2];        // indexed by exchange-op ordinal
  std::vector<int> op_xord;            // op index -> exchange ordinal (-1 if none)
  CopySeg* segs_dev = nullptr;         // all loopback/local copy segments
  struct SegRange { int first = 0, count = 0; unsigned long long maxb = 0; };
  std::vector<SegRange> seg_remote[2][2], seg_local[2][2];

  // execution state
  cudaStream_t s0 = nullptr, s1 = nullptr; bool own_s0 = false;
  cudaEvent_t ev_fork = nullptr, ev_x = nullptr, ev_join = nullptr, ev_t0 = nullptr, ev_t1 = nullptr;
  cudaGraphExec_t graphs[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  float* graph_latent = nullptr;
  int k = 0;
  bool poisoned = false;
  int launches_per_step = 0;
  NcclApi* nccl = nullptr;
  void* comm = nullptr;   // ncclComm_t

  // PEER backend (PCPP_COMM_PEER): exchanges are one-sided pushes into the peers' arenas (CUDA IPC
  // mappings; NVLink stores across GPUs) + device flag barriers (kernels/peer.cu)
  int backend = PCPP_COMM_LOOPBACK;     // effective backend (n == 1 runs LOOPBACK)
  bool peer_connected = false;
  char* peer_base[8] = {};              // every rank's arena in this address space (own at [rank0])
  size_t off_sig = 0, off_x0g = 0, off_lat = 0;   // flags + epoch; gathered x_0 [H][W][4]; latent patch [h][W][4]
  PeerBarrier bar;
  std::vector<SegRange> seg_push[2][2]; // [sync][par] per exchange ordinal: this rank's pushes
  SegRange seg_x0;                      // final gather of x_0 into every rank's x0g
  CopySeg* push_dev = nullptr;
  int simt_fallbacks = 0;               // launches of a captured step that fell back from tcgen05 to SIMT

  ~Plan();
};

// builder / layout (runtime.cpp)
pcpp_status build_program(Plan& P, int model);
pcpp_status validate(int H, int W, int C, int n, double p, int w, const pcpp_config* cfg);
void compute_ledgers(Plan& P, pcpp_info* info);
size_t plan_memory(Plan& P);
pcpp_status temb_precompute(Plan& P);
pcpp_status plan_allocate(Plan& P);
pcpp_status plan_upload_weights(Plan& P, const float* blob);
pcpp_status plan_build_exchanges(Plan& P);
pcpp_status plan_init_comm(Plan& P);
pcpp_status plan_peer_connect(Plan& P, const void* handles);
void peer_barrier(Plan& P, cudaStream_t s);
const char* comm_lib_path();
pcpp_status plan_autotune(Plan& P);
enum { K_GEMM = 1, K_ATTN = 2, K_GN = 4, K_XCH = 8, K_MISC = 16, K_END = 32, K_ALL = 63 };
pcpp_status run_step(Plan& P, float* latent, int sync, int par, unsigned mask = K_ALL);
pcpp_status context_setup(Plan& P, const float* ctx_host);
// algorithmic work of the ops of one kind in one step (all virtual ranks): flops, bytes, launches
void op_work(const Plan& P, unsigned kind, int sync, double* flops, double* bytes, int* launches);
int band_rows(double p, int h);
long long simt_fallback_count();
void print_op_timing(Plan& P, float* latent, int sync, int par);
const char* set_error(const char* fmt, ...);

// kernels init
void kernels_init();

}  // namespace pcpp
