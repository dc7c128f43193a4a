#include <cstdlib>
// extern "C" boundary of libpcpp (include/pcpp.h).  No exception crosses it.
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <vector>
#include "runtime.h"
#include "nccl_api.h"

namespace pcpp {
int gemm_trace_copy(unsigned long long* host, int max_launches);
const char* last_error_msg();
XGroup make_group_public(const Plan& P, const Op& op, int sync, int par, std::vector<Xfer>& lb);
void launch_gemm_auto(const GemmArgs& g, bool allow_tc, cudaStream_t s);
void launch_attn_auto(const AttnArgs& a, bool allow_tc, cudaStream_t s);
bool tc_available();
}

using namespace pcpp;

struct pcpp_plan_s { std::unique_ptr<Plan> P; float* lat_dev = nullptr; float* full_dev = nullptr;
                     cudaEvent_t ev_in = nullptr, ev_out = nullptr; };

#define CKS(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { set_error("CUDA %s at %s:%d: %s", #x, __FILE__, __LINE__, cudaGetErrorString(e_)); return PCPP_ERR_CUDA; } } while (0)
#define GUARD_BEGIN try {
#define GUARD_END } catch (const std::bad_alloc&) { set_error("host allocation failed"); return PCPP_ERR_OOM; } \
                  catch (...) { set_error("internal error"); return PCPP_ERR_INVALID; }

extern "C" {

void pcpp_config_default(pcpp_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof *c);
  c->rank = 0; c->world = 1; c->num_steps = 50; c->guidance_scale = 5.0f;
  c->precision = PCPP_BF16; c->scheme = PCPP_SCHEME_PCPP; c->model = PCPP_MODEL_SDXL;
  c->comm_backend = PCPP_COMM_LOOPBACK; c->kernels = PCPP_KERNELS_AUTO; c->use_graphs = 1;
}

const char* pcpp_last_error(void) { return last_error_msg(); }

pcpp_status pcpp_get_unique_id(void* out128) {
  if (!out128) { set_error("out128 is NULL"); return PCPP_ERR_INVALID; }
  NcclApi* api = nccl_api();
  if (!api) return PCPP_ERR_NCCL;
  ncclUniqueId id;
  if (api->GetUniqueId(&id) != 0) { set_error("ncclGetUniqueId failed"); return PCPP_ERR_NCCL; }
  std::memcpy(out128, &id, 128);
  return PCPP_OK;
}

// ---- manifest (host-only builder run on a minimal geometry) ----------------------------------
static Plan* manifest_plan(int model) {
  static std::mutex mu;
  static std::map<int, std::unique_ptr<Plan>> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(model);
  if (it != cache.end()) return it->second.get();
  if (model < PCPP_MODEL_TINY || model > PCPP_MODEL_SDXL_XF) return nullptr;
  auto P = std::make_unique<Plan>();
  pcpp_config_default(&P->cfg);
  P->cfg.model = model;
  P->H = 32; P->W = 32; P->C = 4; P->n = 1; P->p = 0.0; P->S = 1; P->dtype = DT_BF16;
  build_program(*P, model);
  Plan* raw = P.get();
  cache[model] = std::move(P);
  return raw;
}

size_t pcpp_weights_len(int model) {
  Plan* P = manifest_plan(model);
  return P ? P->blob_len : 0;
}
int pcpp_manifest_count(int model) {
  Plan* P = manifest_plan(model);
  return P ? (int)P->man_name.size() : -1;
}
int pcpp_manifest_entry(int model, int i, char* name, int cap, long long shape[4]) {
  Plan* P = manifest_plan(model);
  if (!P || i < 0 || i >= (int)P->man_name.size()) return -1;
  if (name && cap > 0) { std::strncpy(name, P->man_name[i].c_str(), cap - 1); name[cap - 1] = 0; }
  const auto& s = P->man_shape[i];
  for (int d = 0; d < 4; ++d) if (shape) shape[d] = d < (int)s.size() ? s[d] : 0;
  return (int)s.size();
}

// ---- plan info (host only) ----------------------------------------------------------------------
static void fill_info(Plan& P, pcpp_info* info) {
  std::memset(info, 0, sizeof *info);
  info->n_conv = 0; info->n_gn = (int)P.gns.size(); info->n_attn = (int)P.attns.size();
  for (const Op& o : P.ops) if (o.k == OP_CONV || o.k == OP_CONVOUT) info->n_conv++;
  info->h_latent = P.H / P.n;
  info->backend = P.backend;
  // activation bytes of one rank arena after the memory plan, and without it (every tensor its own range)
  if (!P.arena_tensor_bytes) plan_memory(P);
  info->arena_bytes_per_rank = (long long)P.arena_tensor_bytes;
  {
    long long unplanned = 0;
    for (const TDesc& d : P.td) unplanned += (long long)((d.bytes + 255) & ~size_t(255)) * (d.dbl ? 2 : 1);
    info->arena_bytes_unplanned = unplanned;
  }
  for (size_t a = 0; a < P.attns.size() && a < PCPP_MAX_LAYERS; ++a) { info->attn_h[a] = P.attns[a].h; info->attn_r[a] = P.attns[a].r; }
  // closed forms: summed over receiving ranks, one step
  const long long n = P.n, es = (long long)dtype_size(P.dtype), nb = P.nb;
  if (n > 1) {
    for (const HaloX& hx : P.halos) {
      const TDesc& d = P.td[hx.t];
      const long long rowb = (long long)P.B * d.W * d.C * dtype_size(d.dtype);
      const long long v = nb * (hx.stride == 1 ? 2 : 1) * (n - 1) * rowb;
      info->bytes_async[1] += v; info->bytes_warmup[1] += v; info->bytes_fullmap[1] += v;
    }
    for (const GnX& g : P.gns) {
      (void)g;
      const long long v = nb * n * (n - 1) * (long long)P.B * GN_G * 2 * 8;
      info->bytes_async[2] += v; info->bytes_warmup[2] += v; info->bytes_fullmap[2] += v;
    }
    for (const AttnX& a : P.attns) {
      const long long rowb = (long long)P.B * a.W * 2 * a.C * es;
      info->bytes_async[0] += nb * 2 * (n - 1) * a.r * rowb;
      info->bytes_warmup[0] += nb * (n - 1) * (long long)a.h * n * rowb;
      info->bytes_fullmap[0] += nb * (n - 1) * (long long)a.h * n * rowb;
    }
  }
  compute_ledgers(P, info);
  long long nk = 0;
  for (const Op& o : P.ops) {
    switch (o.k) {
      case OP_TEMB: nk += 1; break;
      case OP_HALO: case OP_KVX: nk += 1; break;
      case OP_GN: nk += 2 * P.nr + (P.n > 1); break;
      case OP_END: nk += 1; break;
      default: nk += P.nr;
    }
  }
  // exact once a step has been enqueued (counted at the launches), else the static estimate
  info->n_kernels_per_step = P.launches_per_step > 0 ? P.launches_per_step : (int)nk;
  double fl = 0, by = 0; int nl = 0;
  op_work(P, K_GEMM | K_ATTN, 0, &fl, &by, &nl);
  info->step_flops = fl;
  // busiest rank: an interior rank (or rank 0 when n <= 2)
  Plan& Q = P;
  const int sv_nr = Q.nr, sv_r0 = Q.rank0;
  Q.nr = 1; Q.rank0 = P.n > 2 ? 1 : 0;
  op_work(Q, K_GEMM | K_ATTN, 0, &fl, &by, &nl);
  Q.nr = sv_nr; Q.rank0 = sv_r0;
  info->step_flops_rank_max = fl;
}

static pcpp_status setup_plan(Plan& P, int H, int W, int C, int n, double p, int w, const pcpp_config* cfg) {
  pcpp_status st = validate(H, W, C, n, p, w, cfg);
  if (st != PCPP_OK) return st;
  P.cfg = *cfg; P.H = H; P.W = W; P.C = C; P.n = n; P.p = p; P.warmup = w; P.S = cfg->num_steps;
  P.dtype = cfg->precision == PCPP_FP32 ? DT_F32 : DT_BF16;
  P.split = cfg->cfg_split != 0; P.B = P.split ? 1 : 2; P.nb = P.split ? 2 : 1; P.world = n * P.nb;
  P.loopback = cfg->comm_backend == PCPP_COMM_LOOPBACK || P.world == 1;
  P.backend = P.loopback ? PCPP_COMM_LOOPBACK : cfg->comm_backend;
  P.xasync = P.loopback && n > 1 && getenv("PCPP_LOOPBACK_ASYNC") && atoi(getenv("PCPP_LOOPBACK_ASYNC")) != 0;
  P.xdelay = (P.xasync && getenv("PCPP_XCH_DELAY")) ? atoll(getenv("PCPP_XCH_DELAY")) : 0;
  P.nr = P.loopback ? P.world : 1;
  P.rank0 = P.loopback ? 0 : cfg->rank;
  return build_program(P, cfg->model);
}

pcpp_status pcpp_plan_info(int H, int W, int C, int n, double p, int w, const pcpp_config* cfg, pcpp_info* info) {
  GUARD_BEGIN
  if (!info) { set_error("info is NULL"); return PCPP_ERR_INVALID; }
  Plan P;
  pcpp_status st = setup_plan(P, H, W, C, n, p, w, cfg);
  if (st != PCPP_OK) return st;
  fill_info(P, info);
  return PCPP_OK;
  GUARD_END
}

int pcpp_plan_schedule(int H, int W, int C, int n, double p, int w, const pcpp_config* cfg, int sync, int* out, int cap) {
  try {
    Plan P;
    if (setup_plan(P, H, W, C, n, p, w, cfg) != PCPP_OK) return -1;
    const int me = cfg->comm_backend == PCPP_COMM_NCCL ? cfg->rank : 0;
    int cnt = 0, grp = 0;
    auto put = [&](int op, int peer, long long bytes, int cls, int g) {
      if (out && cnt < cap) { int* r = out + 5 * cnt; r[0] = op; r[1] = peer; r[2] = (int)bytes; r[3] = cls; r[4] = g; }
      ++cnt;
    };
    std::vector<Xfer> lb;
    for (const Op& op : P.ops) {
      if (!((op.k == OP_HALO || op.k == OP_KVX || op.k == OP_GN) && P.n > 1)) continue;
      XGroup G = make_group_public(P, op, sync ? 1 : 0, 0, lb);
      if (G.allgather) put(2, -1, (long long)G.ag_bytes, G.cls, grp);
      else
        for (const Xfer& x : G.remote) {
          if (x.src_rank == me) put(0, x.dst_rank, (long long)x.bytes, x.cls, grp);
          if (x.dst_rank == me) put(1, x.src_rank, (long long)x.bytes, x.cls, grp);
        }
      ++grp;
    }
    return cnt;
  } catch (...) { return -1; }
}

pcpp_status pcpp_plan(int H, int W, int C, int n, double p, int w, const pcpp_config* cfg, pcpp_plan_t* out) {
  GUARD_BEGIN
  if (!out) { set_error("out is NULL"); return PCPP_ERR_INVALID; }
  *out = nullptr;
  auto h = std::make_unique<pcpp_plan_s>();
  h->P = std::make_unique<Plan>();
  Plan& P = *h->P;
  pcpp_status st = setup_plan(P, H, W, C, n, p, w, cfg);
  if (st != PCPP_OK) return st;
  if (!cfg->weights || cfg->weights_len != P.blob_len) {
    set_error("weights blob has %zu floats, model needs %zu", cfg->weights_len, P.blob_len);
    return PCPP_ERR_INVALID;
  }
  int dev = 0;
  CKS(cudaGetDevice(&dev));
  cudaDeviceProp prop;
  CKS(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10) { set_error("libpcpp needs an sm_100 (B200) device, found sm_%d%d", prop.major, prop.minor); return PCPP_ERR_UNSUPPORTED; }
  kernels_init();
  P.use_tc = P.dtype == DT_BF16 && cfg->kernels == PCPP_KERNELS_AUTO && tc_available();
  if ((st = plan_allocate(P)) != PCPP_OK) return st;
  if ((st = plan_upload_weights(P, cfg->weights)) != PCPP_OK) return st;
  if ((st = plan_build_exchanges(P)) != PCPP_OK) return st;
  CKS(cudaStreamCreateWithFlags(&P.s0, cudaStreamNonBlocking)); P.own_s0 = true;
  CKS(cudaStreamCreateWithFlags(&P.s1, cudaStreamNonBlocking));
  CKS(cudaEventCreateWithFlags(&P.ev_fork, cudaEventDisableTiming));
  CKS(cudaEventCreateWithFlags(&P.ev_x, cudaEventDisableTiming));
  CKS(cudaEventCreateWithFlags(&P.ev_join, cudaEventDisableTiming));
  CKS(cudaEventCreate(&P.ev_t0)); CKS(cudaEventCreate(&P.ev_t1));
  CKS(cudaEventCreateWithFlags(&h->ev_in, cudaEventDisableTiming));
  CKS(cudaEventCreateWithFlags(&h->ev_out, cudaEventDisableTiming));
  if ((st = plan_init_comm(P)) != PCPP_OK) return st;
  if ((st = temb_precompute(P)) != PCPP_OK) return st;
  if ((st = plan_autotune(P)) != PCPP_OK) return st;
  CKS(cudaDeviceSynchronize());
  *out = h.release();
  return PCPP_OK;
  GUARD_END
}

static pcpp_status step_internal(pcpp_plan_s* h, float* latent, int t) {
  Plan& P = *h->P;
  if (P.poisoned) { set_error("plan is poisoned by an earlier CUDA/NCCL error"); return PCPP_ERR_STATE; }
  if (t != P.k || t >= P.S) { set_error("pcpp_step(t=%d) but the plan is at step %d of %d", t, P.k, P.S); return PCPP_ERR_STATE; }
  if (P.xf && !P.ctx_set) { set_error("_XF model: pcpp_set_context has not been called"); return PCPP_ERR_STATE; }
  const int sync = (P.n > 1 && (P.cfg.scheme == PCPP_SCHEME_SYNC || t < P.warmup)) ? 1 : 0;
  const int par = t & 1;
  const bool fork = (!P.loopback || P.xasync) && P.n > 1;
  pcpp_status st = PCPP_OK;
  cudaError_t e;
  if (P.cfg.use_graphs) {
    if (P.graph_latent != latent) {
      for (auto& g : P.graphs) for (auto& x : g) if (x) { cudaGraphExecDestroy(x); x = nullptr; }
      P.graph_latent = latent;
    }
    if (!P.graphs[sync][par]) {
      cudaGraph_t g = nullptr;
      e = cudaStreamBeginCapture(P.s0, cudaStreamCaptureModeRelaxed);
      if (e != cudaSuccess) { P.poisoned = true; set_error("capture: %s", cudaGetErrorString(e)); return PCPP_ERR_CUDA; }
      if (fork) { cudaEventRecord(P.ev_fork, P.s0); cudaStreamWaitEvent(P.s1, P.ev_fork, 0); }
      st = run_step(P, latent, sync, par);
      if (fork) { cudaEventRecord(P.ev_join, P.s1); cudaStreamWaitEvent(P.s0, P.ev_join, 0); }
      e = cudaStreamEndCapture(P.s0, &g);
      if (st != PCPP_OK) { if (g) cudaGraphDestroy(g); P.poisoned = true; return st; }
      if (e != cudaSuccess) { P.poisoned = true; set_error("end capture: %s", cudaGetErrorString(e)); return PCPP_ERR_CUDA; }
      e = cudaGraphInstantiate(&P.graphs[sync][par], g, 0);
      cudaGraphDestroy(g);
      if (e != cudaSuccess) { P.poisoned = true; set_error("instantiate: %s", cudaGetErrorString(e)); return PCPP_ERR_CUDA; }
    }
    cudaEventRecord(P.ev_t0, P.s0);
    e = cudaGraphLaunch(P.graphs[sync][par], P.s0);
    cudaEventRecord(P.ev_t1, P.s0);
    if (e != cudaSuccess) { P.poisoned = true; set_error("graph launch: %s", cudaGetErrorString(e)); return PCPP_ERR_CUDA; }
  } else {
    cudaEventRecord(P.ev_t0, P.s0);
    if (fork) { cudaEventRecord(P.ev_fork, P.s0); cudaStreamWaitEvent(P.s1, P.ev_fork, 0); }
    st = run_step(P, latent, sync, par);
    if (fork) { cudaEventRecord(P.ev_join, P.s1); cudaStreamWaitEvent(P.s0, P.ev_join, 0); }
    cudaEventRecord(P.ev_t1, P.s0);
    if (st != PCPP_OK) { P.poisoned = true; return st; }
  }
  P.k++;
  return PCPP_OK;
}

pcpp_status pcpp_step(pcpp_plan_t h, float* latent, int t) {
  GUARD_BEGIN
  if (!h || !latent) { set_error("NULL argument"); return PCPP_ERR_INVALID; }
  Plan& P = *h->P;
  cudaStream_t us = reinterpret_cast<cudaStream_t>(P.cfg.stream);
  CKS(cudaEventRecord(h->ev_in, us));
  CKS(cudaStreamWaitEvent(P.s0, h->ev_in, 0));
  pcpp_status st = step_internal(h, latent, t);
  if (st != PCPP_OK) return st;
  CKS(cudaEventRecord(h->ev_out, P.s0));
  CKS(cudaStreamWaitEvent(us, h->ev_out, 0));
  return PCPP_OK;
  GUARD_END
}

pcpp_status pcpp_reset(pcpp_plan_t h) {
  if (!h) { set_error("NULL plan"); return PCPP_ERR_INVALID; }
  Plan& P = *h->P;
  if (P.poisoned) { set_error("plan is poisoned"); return PCPP_ERR_STATE; }
  CKS(cudaMemsetAsync(P.k_dev, 0, sizeof(int), P.s0));
  P.k = 0;
  return PCPP_OK;
}

pcpp_status pcpp_set_cond(pcpp_plan_t h, const float* cond) {
  if (!h || !cond) { set_error("NULL argument"); return PCPP_ERR_INVALID; }
  Plan& P = *h->P;
  CKS(cudaMemcpyAsync(P.cond, cond, (size_t)P.T * 4, cudaMemcpyHostToDevice, P.s0));
  pcpp_status st = temb_precompute(P);
  if (st != PCPP_OK) return st;
  CKS(cudaStreamSynchronize(P.s0));
  return PCPP_OK;
}

pcpp_status pcpp_set_context(pcpp_plan_t h, const float* ctx) {
  GUARD_BEGIN
  if (!h || !ctx) { set_error("NULL argument"); return PCPP_ERR_INVALID; }
  Plan& P = *h->P;
  if (!P.xf) { set_error("pcpp_set_context: the plan's model has no cross-attention (use an _XF model)"); return PCPP_ERR_INVALID; }
  if (P.poisoned) { set_error("plan is poisoned"); return PCPP_ERR_STATE; }
  pcpp_status st = context_setup(P, ctx);
  if (st != PCPP_OK) P.poisoned = true;
  return st;
  GUARD_END
}

pcpp_status pcpp_sample(pcpp_plan_t h, const float* xT, const float* cond, float* x0) {
  GUARD_BEGIN
  if (!h || !xT || !cond || !x0) { set_error("NULL argument"); return PCPP_ERR_INVALID; }
  Plan& P = *h->P;
  const size_t patch = (size_t)(P.loopback ? P.H : P.H / P.n) * P.W * 4;
  const size_t full = (size_t)P.H * P.W * 4;
  const bool peer = P.backend == PCPP_COMM_PEER;
  if (peer && !P.peer_connected) { set_error("PEER backend: pcpp_peer_connect has not been called"); return PCPP_ERR_STATE; }
  if (peer) h->lat_dev = reinterpret_cast<float*>(P.rm[0].arena + P.off_lat);   // the gather source lives in the arena
  if (!h->lat_dev) CKS(cudaMalloc(&h->lat_dev, patch * 4));
  if (!P.loopback && !peer && !h->full_dev) CKS(cudaMalloc(&h->full_dev, full * 4));
  pcpp_status st = pcpp_reset(h);
  if (st != PCPP_OK) return st;
  if ((st = pcpp_set_cond(h, cond)) != PCPP_OK) return st;
  CKS(cudaMemcpyAsync(h->lat_dev, xT, patch * 4, cudaMemcpyHostToDevice, P.s0));
  for (int k = 0; k < P.S; ++k) if ((st = step_internal(h, h->lat_dev, k)) != PCPP_OK) return st;
  const float* src = h->lat_dev;
  if (peer) {                  // push the patch into every rank's x0g, then a barrier
    launch_copy_segments(P.push_dev + P.seg_x0.first, P.seg_x0.count, P.seg_x0.maxb, P.s0);
    peer_barrier(P, P.s0);
    src = reinterpret_cast<const float*>(P.rm[0].arena + P.off_x0g);
  } else if (!P.loopback) {
    if (P.nccl->AllGather(h->lat_dev, h->full_dev, patch, nccl_float32, reinterpret_cast<ncclComm_t>(P.comm), P.s0) != 0) {
      set_error("final ncclAllGather failed"); return PCPP_ERR_NCCL;
    }
    src = h->full_dev;
  }
  CKS(cudaMemcpyAsync(x0, src, full * 4, cudaMemcpyDeviceToHost, P.s0));
  CKS(cudaStreamSynchronize(P.s0));
  return PCPP_OK;
  GUARD_END
}

pcpp_status pcpp_peer_handle(pcpp_plan_t h, void* out64) {
  GUARD_BEGIN
  if (!h || !out64) { set_error("NULL argument"); return PCPP_ERR_INVALID; }
  Plan& P = *h->P;
  if (P.backend != PCPP_COMM_PEER) { set_error("pcpp_peer_handle: plan does not use the PEER backend"); return PCPP_ERR_STATE; }
  cudaIpcMemHandle_t mh;
  CKS(cudaIpcGetMemHandle(&mh, P.rm[0].arena));
  std::memcpy(out64, &mh, sizeof mh);
  return PCPP_OK;
  GUARD_END
}

pcpp_status pcpp_peer_connect(pcpp_plan_t h, const void* handles) {
  GUARD_BEGIN
  if (!h || !handles) { set_error("NULL argument"); return PCPP_ERR_INVALID; }
  pcpp_status st = plan_peer_connect(*h->P, handles);
  if (st == PCPP_ERR_CUDA) h->P->poisoned = true;
  return st;
  GUARD_END
}

pcpp_status pcpp_query(pcpp_plan_t h, pcpp_info* info) {
  GUARD_BEGIN
  if (!h || !info) { set_error("NULL argument"); return PCPP_ERR_INVALID; }
  Plan& P = *h->P;
  fill_info(P, info);
  float ms = 0.f;
  if (P.k > 0 && cudaEventSynchronize(P.ev_t1) == cudaSuccess && cudaEventElapsedTime(&ms, P.ev_t0, P.ev_t1) == cudaSuccess)
    info->last_step_ms = ms;
  info->device_bytes = (long long)P.rank_bytes * P.nr + (long long)P.wmat_len * (long long)dtype_size(P.dtype) + P.wf32_len * 4;
  info->graphs = P.cfg.use_graphs;
  info->tc_kernels = P.use_tc;
  info->simt_fallbacks = P.simt_fallbacks;
  std::snprintf(info->comm_lib, sizeof info->comm_lib, "%s", P.backend == PCPP_COMM_NCCL ? comm_lib_path() : "");
  return PCPP_OK;
  GUARD_END
}

pcpp_status pcpp_profile(pcpp_plan_t h, float* latent, int kind, int sync, int iters, pcpp_prof* out) {
  GUARD_BEGIN
  if (!h || !latent || !out || iters < 1 || kind <= 0 || (kind & ~31)) { set_error("pcpp_profile: bad arguments"); return PCPP_ERR_INVALID; }
  Plan& P = *h->P;
  if (P.poisoned) { set_error("plan is poisoned"); return PCPP_ERR_STATE; }
  sync = (P.n > 1 && sync) ? 1 : 0;
  const bool fork = (!P.loopback || P.xasync) && P.n > 1;
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ge = nullptr;
  CKS(cudaStreamSynchronize(P.s0));
  static const int op_timing = getenv("PCPP_OP_TIMING") ? atoi(getenv("PCPP_OP_TIMING")) : 0;
  if (op_timing && kind == 31 && !fork) { print_op_timing(P, latent, sync, P.k & 1); CKS(cudaStreamSynchronize(P.s0)); }
  CKS(cudaStreamBeginCapture(P.s0, cudaStreamCaptureModeRelaxed));
  if (fork) { cudaEventRecord(P.ev_fork, P.s0); cudaStreamWaitEvent(P.s1, P.ev_fork, 0); }
  pcpp_status st = run_step(P, latent, sync, P.k & 1, (unsigned)kind);
  if (fork) { cudaEventRecord(P.ev_join, P.s1); cudaStreamWaitEvent(P.s0, P.ev_join, 0); }
  cudaError_t e = cudaStreamEndCapture(P.s0, &g);
  if (st != PCPP_OK) { if (g) cudaGraphDestroy(g); return st; }
  CKS(e);
  CKS(cudaGraphInstantiate(&ge, g, 0));
  cudaGraphDestroy(g);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaGraphLaunch(ge, P.s0);
  cudaEventRecord(a, P.s0);
  for (int i = 0; i < iters; ++i) cudaGraphLaunch(ge, P.s0);
  cudaEventRecord(b, P.s0);
  e = cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a); cudaEventDestroy(b);
  cudaGraphExecDestroy(ge);
  CKS(e);
  out->ms = ms / iters;
  op_work(P, (unsigned)kind, sync, &out->flops, &out->bytes, &out->launches);
  return PCPP_OK;
  GUARD_END
}

int pcpp_debug_gemm_trace(unsigned long long* out) {
  if (!out) return -1;
  return gemm_trace_copy(out, 32);
}

pcpp_status pcpp_debug_comm_off(pcpp_plan_t h, int on) {
  GUARD_BEGIN
  if (!h) { set_error("NULL plan"); return PCPP_ERR_INVALID; }
  Plan& P = *h->P;
  if (P.comm_off != (on != 0)) {
    CKS(cudaStreamSynchronize(P.s0));
    for (auto& g : P.graphs) for (auto& x : g) if (x) { cudaGraphExecDestroy(x); x = nullptr; }
    P.comm_off = on != 0;
  }
  return PCPP_OK;
  GUARD_END
}

void pcpp_destroy(pcpp_plan_t h) {
  if (!h) return;
  if (h->P && h->P->s0) cudaStreamSynchronize(h->P->s0);
  if (h->P && h->P->backend == PCPP_COMM_PEER && h->P->peer_connected && !h->P->poisoned) {
    // collective: no peer may still push into this arena when it is unmapped and freed
    peer_barrier(*h->P, h->P->s0);
    cudaStreamSynchronize(h->P->s0);
  }
  if (h->lat_dev && !(h->P && h->P->backend == PCPP_COMM_PEER)) cudaFree(h->lat_dev);
  if (h->full_dev) cudaFree(h->full_dev);
  if (h->ev_in) cudaEventDestroy(h->ev_in);
  if (h->ev_out) cudaEventDestroy(h->ev_out);
  delete h;
}

// Workspaces of the kernel-level entry points: one per (device, purpose), grown on demand (the old
// buffer is freed with cudaFree, which waits for work still using it).  Calls on several host
// threads / streams at once would share them: the entry points are a test and benchmark surface.
enum { WS_CONV = 0, WS_ATTN = 1, WS_GN = 2, WS_SEG = 3, WS_COEF = 4 };
static void* op_scratch(int slot, size_t bytes, bool zero) {
  static std::mutex mu;
  static std::map<std::pair<int, int>, std::pair<void*, size_t>> pool;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  auto& e = pool[{dev, slot}];
  if (bytes > e.second) {
    if (e.first) cudaFree(e.first);
    e = {nullptr, 0};
    if (cudaMalloc(&e.first, bytes) != cudaSuccess) { e.first = nullptr; return nullptr; }
    if (zero && cudaMemset(e.first, 0, bytes) != cudaSuccess) return nullptr;
    e.second = bytes;
  }
  return e.first;
}

// ---- kernel-level entry points ------------------------------------------------------------------
pcpp_status pcpp_op_conv(const void* x, int rows_in, int B, int W_in, int Cin, int taps, int stride,
                         const void* w, const float* bias, const float* temb, const void* res, void* y,
                         int Cout, int dtype, int impl, void* stream) {
  GUARD_BEGIN
  if (!x || !w || !y || (taps != 1 && taps != 9) || (stride != 1 && stride != 2) || (taps == 1 && stride != 1) ||
      rows_in <= 0 || B <= 0 || W_in <= 0 || Cin <= 0 || Cout <= 0 || (dtype != PCPP_FP32 && dtype != PCPP_BF16)) {
    set_error("pcpp_op_conv: bad arguments"); return PCPP_ERR_INVALID;
  }
  if (stride == 2 && (rows_in % 2 || W_in % 2)) { set_error("stride 2 needs even rows/W"); return PCPP_ERR_INVALID; }
  kernels_init();
  const int dt = dtype == PCPP_FP32 ? DT_F32 : DT_BF16;
  GemmArgs g;
  const size_t rowb = (size_t)B * W_in * Cin * dtype_size(dt);
  g.a0.base = const_cast<char*>(reinterpret_cast<const char*>(x)) + (taps == 9 ? rowb : 0);
  g.a0.rows = rows_in; g.a0.B = B; g.a0.W = W_in; g.a0.C = Cin; g.a0.dtype = dt;
  g.c0 = Cin; g.cin = Cin; g.taps = taps; g.stride = stride;
  g.rows_out = rows_in / stride; g.w_out = W_in / stride; g.B = B;
  g.w = w; g.wdtype = dt; g.N = Cout; g.bias = bias; g.temb = temb; g.temb_ld = Cout;
  g.out.base = y; g.out.rows = g.rows_out; g.out.B = B; g.out.W = g.w_out; g.out.C = Cout; g.out.dtype = dt;
  if (res) { g.res = g.out; g.res.base = const_cast<void*>(res); }
  const size_t need = 8ull * g.rows_out * B * g.w_out * Cout;     // split-K partials (fp32)
  float* ws = dt == DT_BF16 ? reinterpret_cast<float*>(op_scratch(WS_CONV, need * 4, false)) : nullptr;
  g.ws = ws; g.ws_elems = ws ? need : 0;
  launch_gemm_auto(g, impl == PCPP_KERNELS_AUTO, reinterpret_cast<cudaStream_t>(stream));
  CKS(cudaGetLastError());
  return PCPP_OK;
  GUARD_END
}

pcpp_status pcpp_op_attention(const void* q, const void* const* kv, const int* kv_rows, int nsrc, int h, int B,
                              int W, int C, void* out, int dtype, int impl, void* stream) {
  GUARD_BEGIN
  if (!q || !kv || !kv_rows || !out || nsrc < 1 || nsrc > 3 || C % 64 || h <= 0 || W <= 0 || B <= 0) {
    set_error("pcpp_op_attention: bad arguments"); return PCPP_ERR_INVALID;
  }
  kernels_init();
  AttnArgs a;
  a.q = q; a.h = h; a.B = B; a.W = W; a.C = C; a.out = out; a.dtype = dtype == PCPP_FP32 ? DT_F32 : DT_BF16;
  a.nsrc = nsrc;
  for (int i = 0; i < nsrc; ++i) { a.src[i].kv = kv[i]; a.src[i].rows = kv_rows[i]; }
  const size_t need = 8ull * B * (C / 64) * h * W * 66;          // split-KV partials (fp32)
  float* ws = a.dtype == DT_BF16 ? reinterpret_cast<float*>(op_scratch(WS_ATTN, need * 4, false)) : nullptr;
  a.ws = ws; a.ws_elems = ws ? need : 0;
  launch_attn_auto(a, impl == PCPP_KERNELS_AUTO, reinterpret_cast<cudaStream_t>(stream));
  CKS(cudaGetLastError());
  return PCPP_OK;
  GUARD_END
}

pcpp_status pcpp_op_groupnorm(const void* x, int rows, int B, int W, int C, const float* gamma, const float* beta,
                              int silu, void* y, double* m_out, int dtype, void* stream) {
  GUARD_BEGIN
  if (!x || !gamma || !beta || !y || !m_out || C % 32 || (C / 32) % 1 || C % 8 || C > 2560 || B > 2 || rows <= 0 || W <= 0) {
    set_error("pcpp_op_groupnorm: bad arguments"); return PCPP_ERR_INVALID;
  }
  kernels_init();
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int dt = dtype == PCPP_FP32 ? DT_F32 : DT_BF16;
  GnStatsArgs a;
  a.x0.base = const_cast<void*>(x); a.x0.rows = rows; a.x0.B = B; a.x0.W = W; a.x0.C = C; a.x0.dtype = dt;
  a.c0 = C; a.C = C; a.nchunk = gn_stats_chunks(rows, W, C);
  char* sc = reinterpret_cast<char*>(op_scratch(WS_GN, (size_t)a.nchunk * 128 * 8, true));
  if (!sc) { set_error("scratch alloc"); return PCPP_ERR_OOM; }
  a.partial = reinterpret_cast<double*>(sc);
  a.m_out = m_out;
  launch_gn_stats(a, s);
  GnApplyArgs p;
  p.x0 = a.x0; p.c0 = C; p.C = C; p.out = a.x0; p.out.base = y;
  p.gamma = gamma; p.beta = beta; p.silu = silu; p.mode = 0; p.nranks = 1; p.m_fresh = m_out;
  p.count = (double)rows * W * (C / 32);
  launch_gn_apply(p, s);
  CKS(cudaGetLastError());
  return PCPP_OK;
  GUARD_END
}

pcpp_status pcpp_op_pack_rows(const void* src, long long row_bytes, int r0, int nrows, void* dst, void* stream) {
  GUARD_BEGIN
  if (!src || !dst || row_bytes <= 0 || row_bytes % 16 || r0 < 0 || nrows < 0) { set_error("pcpp_op_pack_rows: bad arguments"); return PCPP_ERR_INVALID; }
  if (nrows == 0) return PCPP_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  CopySeg* dseg = reinterpret_cast<CopySeg*>(op_scratch(WS_SEG, sizeof(CopySeg), false));
  if (!dseg) { set_error("scratch alloc"); return PCPP_ERR_OOM; }
  CopySeg h{reinterpret_cast<const char*>(src) + (size_t)r0 * row_bytes, dst, (unsigned long long)row_bytes * nrows};
  CKS(cudaMemcpyAsync(dseg, &h, sizeof h, cudaMemcpyHostToDevice, s));
  CKS(cudaStreamSynchronize(s));
  launch_copy_segments(dseg, 1, h.bytes, s);
  CKS(cudaGetLastError());
  return PCPP_OK;
  GUARD_END
}

pcpp_status pcpp_op_cfg_ddim(const float* eps, float* latent, int h, int W, float guidance, int S, int k, void* stream) {
  GUARD_BEGIN
  if (!eps || !latent || h <= 0 || W <= 0 || S < 1 || S > 1000 || k < 0 || k >= S) { set_error("pcpp_op_cfg_ddim: bad arguments"); return PCPP_ERR_INVALID; }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const double b0 = std::sqrt(0.00085), b1 = std::sqrt(0.012);
  double acc = 1.0; std::vector<double> ab(1000);
  for (int t = 0; t < 1000; ++t) { const double bt = b0 + (b1 - b0) * (double)t / 999.0; acc *= (1.0 - bt * bt); ab[t] = acc; }
  const int ratio = 1000 / S, tau = (S - 1 - k) * ratio + 1, prev = tau - ratio;
  const double at = ab[tau], ap = prev >= 0 ? ab[prev] : ab[0];
  struct { double c[4]; int k; int pad[3]; } hb = {{std::sqrt(at), std::sqrt(1 - at), std::sqrt(ap), std::sqrt(1 - ap)}, 0, {0, 0, 0}};
  char* d = reinterpret_cast<char*>(op_scratch(WS_COEF, sizeof hb, false));
  if (!d) { set_error("scratch alloc"); return PCPP_ERR_OOM; }
  CKS(cudaMemcpyAsync(d, &hb, sizeof hb, cudaMemcpyHostToDevice, s));
  CKS(cudaStreamSynchronize(s));
  launch_cfg_ddim(eps, latent, h, W, guidance, reinterpret_cast<const double*>(d), reinterpret_cast<const int*>(d + 32), s);
  CKS(cudaGetLastError());
  return PCPP_OK;
  GUARD_END
}

}  // extern "C"
