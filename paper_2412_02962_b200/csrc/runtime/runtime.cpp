// Plan memory layout, weight upload, exchange descriptors and the step executor.
//
// Exchange protocol (§3.2, reading D6): every buffer whose rows are sent is double-buffered by
// step parity q = k mod 2.  At async step k a rank sends its fresh rows of parity q and receives
// its neighbours' rows into parity q buffers that the SAME layer reads at step k+1 (conv halos go
// to the 1-q copy of the conv-input tensor, bands to recv_{top,bot}[q], GN sums to mall[q]).
// Reads at step k use what step k-1 received, so the transfer has a whole step of slack
// ("issued one step ahead") and nothing waits on it inside the step.  Warm-up (sync) steps
// exchange this step's data and wait for it ("synchronous AllGather").
#include <algorithm>
#include <stdexcept>
#include <cmath>
#include <cstring>
#include <dlfcn.h>
#include <cstdlib>
#include "runtime.h"
#include "nccl_api.h"

namespace pcpp {

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { set_error("CUDA %s at %s:%d: %s", #x, __FILE__, __LINE__, cudaGetErrorString(e_)); return PCPP_ERR_CUDA; } } while (0)

static char g_comm_lib[512] = "";
const char* comm_lib_path() { return g_comm_lib; }

// libnccl is dlopen'd: PCPP_NCCL_LIB (the Python binding sets it to the NCCL that torch ships) or,
// failing that, the loader's libnccl.so.2 (an NCCL already loaded by the process is reused)
NcclApi* nccl_api() {
  static NcclApi api;
  static bool tried = false;
  if (api.handle) return &api;
  if (tried) { set_error("NCCL could not be loaded"); return nullptr; }
  tried = true;
  const char* env = getenv("PCPP_NCCL_LIB");
  const char* cands[] = {env && *env ? env : nullptr, "libnccl.so.2"};
  for (const char* c : cands) {
    if (!c) continue;
    api.handle = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
    if (api.handle) break;
  }
  if (!api.handle) { set_error("dlopen(libnccl.so.2) failed (set PCPP_NCCL_LIB)"); return nullptr; }
#define SYM(f, n) api.f = reinterpret_cast<decltype(api.f)>(dlsym(api.handle, n)); if (!api.f) { set_error("missing %s", n); api.handle = nullptr; return nullptr; }
  SYM(GetUniqueId, "ncclGetUniqueId"); SYM(CommInitRank, "ncclCommInitRank"); SYM(CommDestroy, "ncclCommDestroy");
  SYM(CommAbort, "ncclCommAbort"); SYM(Send, "ncclSend"); SYM(Recv, "ncclRecv"); SYM(AllGather, "ncclAllGather");
  SYM(GroupStart, "ncclGroupStart"); SYM(GroupEnd, "ncclGroupEnd"); SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
  Dl_info di;
  if (dladdr(reinterpret_cast<void*>(api.GetUniqueId), &di) && di.dli_fname)
    snprintf(g_comm_lib, sizeof g_comm_lib, "%s", di.dli_fname);
  return &api;
}

Plan::~Plan() {
  for (auto& g : graphs) for (auto& x : g) if (x) cudaGraphExecDestroy(x);
  if (comm && nccl) nccl->CommDestroy(reinterpret_cast<ncclComm_t>(comm));
  for (int j = 0; j < 8; ++j)
    if (peer_base[j] && (rm.empty() || peer_base[j] != rm[0].arena)) cudaIpcCloseMemHandle(peer_base[j]);
  if (push_dev) cudaFree(push_dev);
  for (auto& r : rm) if (r.arena) cudaFree(r.arena);
  for (void* p : gallocs) cudaFree(p);
  if (segs_dev) cudaFree(segs_dev);
  cudaEvent_t evs[] = {ev_fork, ev_x, ev_join, ev_t0, ev_t1};
  for (auto e : evs) if (e) cudaEventDestroy(e);
  if (s1) cudaStreamDestroy(s1);
  if (own_s0 && s0) cudaStreamDestroy(s0);
}

// ---------------------------------------------------------------------------------------------
// memory layout
// ---------------------------------------------------------------------------------------------
static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// Rank-arena memory plan.  Pinned tensors (one buffer per step parity, halo-padded, or read by an
// exchange: their rows outlive the op that consumes them) get their own ranges.  Every other tensor
// lives from the op that first touches it to the op that last reads it within one step (ops run in
// order on the compute stream, and every kernel orders its global accesses after the previous
// kernel's completion -- stream order, or griddepcontrol.wait under PDL), so tensors whose live
// intervals are disjoint share memory: greedy first fit, largest first.  PCPP_MEMPLAN=0 disables it.
size_t plan_memory(Plan& P) {
  const int nt = (int)P.td.size();
  std::vector<int> first(nt, 1 << 30), last(nt, -1);
  for (int i = 0; i < (int)P.ops.size(); ++i) {
    const Op& o = P.ops[i];
    for (int r : {o.in0, o.in1, o.out, o.out2, o.res, o.tmp})
      if (r >= 0) { first[r] = std::min(first[r], i); last[r] = std::max(last[r], i); }
  }
  std::vector<char> pinned(nt, 0);
  for (int t = 0; t < nt; ++t) pinned[t] = P.td[t].dbl || P.td[t].pad || P.td[t].xdst || last[t] < 0;
  for (const HaloX& h : P.halos) pinned[h.t] = 1;
  for (const AttnX& a : P.attns) pinned[a.kv] = 1;
  size_t off = 0;
  for (int t = 0; t < nt; ++t) {
    if (!pinned[t]) continue;
    TDesc& d = P.td[t];
    d.off[0] = off; off = align256(off + d.bytes);
    if (d.dbl) { d.off[1] = off; off = align256(off + d.bytes); } else d.off[1] = d.off[0];
  }
  const size_t base = off;
  std::vector<int> order;
  for (int t = 0; t < nt; ++t) if (!pinned[t]) order.push_back(t);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return P.td[a].bytes > P.td[b].bytes; });
  std::vector<int> placed;
  size_t top = base;
  for (int t : order) {
    const size_t sz = align256(P.td[t].bytes);
    std::vector<std::pair<size_t, size_t>> busy;   // address ranges of time-overlapping placed tensors
    for (int u : placed)
      if (!(last[u] < first[t] || last[t] < first[u])) busy.push_back({P.td[u].off[0], P.td[u].off[0] + align256(P.td[u].bytes)});
    std::sort(busy.begin(), busy.end());
    size_t at = base;
    for (auto& r : busy) {
      if (at + sz <= r.first) break;
      at = std::max(at, r.second);
    }
    P.td[t].off[0] = P.td[t].off[1] = at;
    top = std::max(top, at + sz);
    placed.push_back(t);
  }
  // invariant: no two tensors that are live at the same op share an address
  for (size_t i = 0; i < placed.size(); ++i)
    for (size_t j = i + 1; j < placed.size(); ++j) {
      const int a = placed[i], b = placed[j];
      if (last[a] < first[b] || last[b] < first[a]) continue;
      const size_t a0 = P.td[a].off[0], a1 = a0 + P.td[a].bytes, b0 = P.td[b].off[0], b1 = b0 + P.td[b].bytes;
      if (a0 < b1 && b0 < a1) throw std::logic_error("memory plan overlap");
    }
  P.arena_tensor_bytes = top;
  return top;
}

pcpp_status plan_allocate(Plan& P) {
  size_t off = align256(plan_memory(P));
  const size_t mb = (size_t)P.B * GN_G * 2 * sizeof(double);
  for (auto& g : P.gns) {
    for (int q = 0; q < 2; ++q) { g.off_m[q] = off; off = align256(off + mb); }
    for (int q = 0; q < 2; ++q) { g.off_mall[q] = off; off = align256(off + mb * P.n); }
    g.off_part = off; off = align256(off + (size_t)g.nchunk * 128 * sizeof(double));
  }
  // GN statistics fused into the producing GEMM's epilogue (bf16 tensor-core path): the GN reads
  // x0 only, and x0's last writer is a CONV/GEMM that writes nothing else
  for (size_t i = 0; i < P.ops.size(); ++i) {
    Op& o = P.ops[i];
    if (o.k != OP_GN || o.in1 >= 0 || P.dtype != DT_BF16) continue;
    for (size_t j = i; j-- > 0;) {
      Op& pr = P.ops[j];
      if (pr.out != o.in0 && pr.out2 != o.in0) continue;
      if ((pr.k == OP_CONV || pr.k == OP_GEMM) && pr.out == o.in0 && pr.out2 < 0 && pr.gn_fuse < 0) pr.gn_fuse = o.xid;
      break;
    }
  }
  P.off_epart = off; off = align256(off + (size_t)148 * 4 * 128 * sizeof(double));
  P.gn_slots.assign((size_t)P.nr * P.gns.size(), 0);
  const size_t es = dtype_size(P.dtype);
  size_t gat_level[3] = {0, 0, 0};
  bool have_level[3] = {false, false, false};
  for (auto& a : P.attns) {
    const size_t rowb = (size_t)P.B * a.W * 2 * a.C * es;
    for (int q = 0; q < 2; ++q) {
      a.off_top[q] = off; off = align256(off + std::max<size_t>(16, (size_t)a.r * rowb));
      a.off_bot[q] = off; off = align256(off + std::max<size_t>(16, (size_t)a.r * rowb));
    }
    const size_t gb = (size_t)a.h * P.n * rowb;
    if (P.n > 1) {
      if (P.cfg.scheme == PCPP_SCHEME_FULLMAP) {
        for (int q = 0; q < 2; ++q) { a.off_gat[q] = off; off = align256(off + gb); }
      } else {
        if (!have_level[a.level]) { gat_level[a.level] = off; off = align256(off + gb); have_level[a.level] = true; }
        a.off_gat[0] = a.off_gat[1] = gat_level[a.level];
      }
    }
  }
  if (P.backend == PCPP_COMM_PEER) {    // flags [n] + epoch, gathered x_0, the latent patch (pcpp_sample)
    P.off_sig = off; off = align256(off + 16 * sizeof(unsigned long long));
    P.off_x0g = off; off = align256(off + (size_t)P.H * P.W * 4 * sizeof(float));
    P.off_lat = off; off = align256(off + (size_t)(P.H / P.n) * P.W * 4 * sizeof(float));
  }
  P.rank_bytes = off;
  P.rm.resize(P.nr);
  for (int i = 0; i < P.nr; ++i) {
    cudaError_t e = cudaMalloc(&P.rm[i].arena, P.rank_bytes);
    if (e != cudaSuccess) { set_error("cudaMalloc(%zu) for rank arena: %s", P.rank_bytes, cudaGetErrorString(e)); return PCPP_ERR_OOM; }
    P.rm[i].bytes = P.rank_bytes;
    CK(cudaMemset(P.rm[i].arena, 0, P.rank_bytes));   // zero halo rows at the image borders
  }
  auto galloc = [&](size_t bytes) -> void* {
    void* p = nullptr;
    if (cudaMalloc(&p, std::max<size_t>(bytes, 256)) != cudaSuccess) return nullptr;
    cudaMemset(p, 0, std::max<size_t>(bytes, 256));
    P.gallocs.push_back(p); return p;
  };
  P.wmat = galloc((size_t)P.wmat_len * es);
  P.wf32 = (float*)galloc((size_t)P.wf32_len * 4);
  P.emb = (float*)galloc(2 * P.T * 4); P.hid = (float*)galloc(P.T * 4);
  P.tproj = (float*)galloc((size_t)2 * P.J * 4); P.cond = (float*)galloc(P.T * 4);
  P.taus = (int*)galloc(P.S * 4); P.coef = (double*)galloc(P.S * 4 * 8); P.k_dev = (int*)galloc(16);
  P.coef_dpm = (double*)galloc(P.S * 6 * 8);
  P.tproj_all = (float*)galloc((size_t)P.S * 2 * P.J * 4); P.emb_all = (float*)galloc((size_t)8 * P.T * 4);
  P.kseq = (int*)galloc(P.S * 4);
  P.coef_anc = (double*)galloc(P.S * 5 * 8);
  if (P.cfg.scheduler == PCPP_SCHED_DPMPP2M) P.x0_hist = (float*)galloc((size_t)P.nr * (P.H / P.n) * P.W * 4 * 4);
  if (P.dtype == DT_BF16) {       // split-K workspace: up to 8 fp32 partial copies of the largest GEMM output
    size_t mx = 0;
    for (const Op& o : P.ops)
      if (o.k == OP_CONV || o.k == OP_GEMM) {
        const TDesc& t = P.td[o.out];
        mx = std::max(mx, (size_t)t.rows * P.B * t.W * (size_t)o.N);
      }
    P.ws_elems = std::min<size_t>(8 * mx, (size_t)1 << 28);
    P.ws = (float*)galloc(P.ws_elems * 4);
  }
  if (P.xf) {     // cross-attention context: as given, laid out per level, and every layer's keys/values
    P.ctx_f32 = (float*)galloc((size_t)2 * 77 * P.ctx_dim * 4);
    for (int l = 0; l < P.levels; ++l)
      P.ctx_level[l] = galloc((size_t)P.ctx_rows(l) * 2 * (P.W >> l) * P.ctx_dim * es);
    for (auto& xa : P.xattns) xa.kv = galloc((size_t)P.ctx_rows(xa.level) * 2 * (P.W >> xa.level) * 2 * xa.C * es);
  }
  for (void* p : P.gallocs) if (!p) { set_error("cudaMalloc failed for global buffers"); return PCPP_ERR_OOM; }
  // DDIM schedule (reading D2): scaled_linear betas, 'leading' spacing, offset 1, final ab_prev = ab[0]
  std::vector<double> ab(1000);
  {
    const double b0 = std::sqrt(0.00085), b1 = std::sqrt(0.012);
    double acc = 1.0;
    for (int t = 0; t < 1000; ++t) {
      const double bt = b0 + (b1 - b0) * (double)t / 999.0;
      acc *= (1.0 - bt * bt);
      ab[t] = acc;
    }
  }
  std::vector<int> taus(P.S); std::vector<double> coef(4 * P.S);
  const int ratio = 1000 / P.S;
  for (int k = 0; k < P.S; ++k) {
    const int tau = (P.S - 1 - k) * ratio + 1;
    const int prev = tau - ratio;
    const double at = ab[tau], ap = prev >= 0 ? ab[prev] : ab[0];
    taus[k] = tau;
    coef[4 * k + 0] = std::sqrt(at); coef[4 * k + 1] = std::sqrt(1.0 - at);
    coef[4 * k + 2] = std::sqrt(ap); coef[4 * k + 3] = std::sqrt(1.0 - ap);
  }
  // DPM-Solver++(2M) on the same ladder (reading D23): lambda = log(alpha / sigma); first order at
  // k = 0 and, for S < 15, at the final step; x' = A x + Bc (w0 x0_k + w1 x0_{k-1})
  std::vector<double> cd(6 * P.S);
  auto lam = [](double a) { return 0.5 * std::log(a) - 0.5 * std::log(1.0 - a); };
  for (int k = 0; k < P.S; ++k) {
    const int tau = (P.S - 1 - k) * ratio + 1;
    const int prev = tau - ratio;
    const double at = ab[tau], ap = prev >= 0 ? ab[prev] : ab[0];
    const double h = lam(ap) - lam(at);
    const bool second = k > 0 && !(P.S < 15 && k == P.S - 1);
    double w0 = 1.0, w1 = 0.0;
    if (second) {
      const double aq = ab[tau + ratio];                      // the previous ladder point
      const double r = (lam(at) - lam(aq)) / h;
      w0 = 1.0 + 1.0 / (2.0 * r); w1 = -1.0 / (2.0 * r);
    }
    cd[6 * k + 0] = 1.0 / std::sqrt(at); cd[6 * k + 1] = std::sqrt(1.0 - at);
    cd[6 * k + 2] = std::sqrt(1.0 - ap) / std::sqrt(1.0 - at);
    cd[6 * k + 3] = -std::sqrt(ap) * std::expm1(-h);
    cd[6 * k + 4] = w0; cd[6 * k + 5] = w1;
  }
  CK(cudaMemcpy(P.coef_dpm, cd.data(), P.S * 6 * 8, cudaMemcpyHostToDevice));
  // ancestral sampler (reading D24): eta = 1, sigma^2 = (1 - ab')/(1 - ab) (1 - ab/ab')
  std::vector<double> ca(5 * P.S);
  for (int k = 0; k < P.S; ++k) {
    const double at = coef[4 * k + 0] * coef[4 * k + 0], ap = coef[4 * k + 2] * coef[4 * k + 2];
    const double var = (1.0 - ap) / (1.0 - at) * (1.0 - at / ap);
    ca[5 * k + 0] = coef[4 * k + 0]; ca[5 * k + 1] = coef[4 * k + 1]; ca[5 * k + 2] = coef[4 * k + 2];
    ca[5 * k + 3] = std::sqrt(std::max(1.0 - ap - var, 0.0)); ca[5 * k + 4] = std::sqrt(var);
  }
  CK(cudaMemcpy(P.coef_anc, ca.data(), P.S * 5 * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(P.taus, taus.data(), P.S * 4, cudaMemcpyHostToDevice));
  {
    std::vector<int> ks(P.S);
    for (int k = 0; k < P.S; ++k) ks[k] = k;
    CK(cudaMemcpy(P.kseq, ks.data(), P.S * 4, cudaMemcpyHostToDevice));
  }
  CK(cudaMemcpy(P.coef, coef.data(), P.S * 4 * 8, cudaMemcpyHostToDevice));
  return PCPP_OK;
}

pcpp_status plan_upload_weights(Plan& P, const float* blob) {
  const size_t es = dtype_size(P.dtype);
  std::vector<float> f32((size_t)P.wf32_len, 0.f);
  std::vector<uint16_t> b16;
  std::vector<float> m32;
  if (P.dtype == DT_BF16) b16.assign((size_t)P.wmat_len, 0); else m32.assign((size_t)P.wmat_len, 0.f);
  for (const auto& u : P.uploads) {
    const float* src = blob + u.blob_off;
    if (u.f32) { std::memcpy(&f32[u.off], src, (size_t)u.numel * 4); continue; }
    if (P.dtype == DT_F32) { std::memcpy(&m32[u.off], src, (size_t)u.numel * 4); continue; }
    for (long long i = 0; i < u.numel; ++i) {   // round-to-nearest-even to bf16
      uint32_t x; std::memcpy(&x, &src[i], 4);
      const uint32_t lsb = (x >> 16) & 1u;
      b16[u.off + i] = (uint16_t)((x + 0x7FFFu + lsb) >> 16);
    }
  }
  CK(cudaMemcpy(P.wf32, f32.data(), f32.size() * 4, cudaMemcpyHostToDevice));
  if (P.dtype == DT_BF16) { CK(cudaMemcpy(P.wmat, b16.data(), b16.size() * es, cudaMemcpyHostToDevice)); }
  else { CK(cudaMemcpy(P.wmat, m32.data(), m32.size() * es, cudaMemcpyHostToDevice)); }
  return PCPP_OK;
}

// ---------------------------------------------------------------------------------------------
// views
// ---------------------------------------------------------------------------------------------
static ActView view(const Plan& P, int vr, int t, int par) {
  const TDesc& d = P.td[t];
  ActView v;
  const int B = d.B ? d.B : P.B;
  const size_t rowb = (size_t)B * d.W * d.C * dtype_size(d.dtype);
  v.base = P.rm[vr].arena + d.off[d.dbl ? par : 0] + (size_t)d.pad * rowb;
  v.rows = d.rows; v.B = B; v.W = d.W; v.C = d.C; v.dtype = d.dtype;
  return v;
}

static char* resolve(const Plan& P, int vr, const BufRef& r) {
  char* base = P.rm[vr].arena;
  switch (r.kind) {
    case BK_TENSOR: { const TDesc& d = P.td[r.id]; return base + d.off[d.dbl ? r.par : 0] + r.byte_off; }
    case BK_TOP: return base + P.attns[r.id].off_top[r.par] + r.byte_off;
    case BK_BOT: return base + P.attns[r.id].off_bot[r.par] + r.byte_off;
    case BK_GAT: return base + P.attns[r.id].off_gat[r.par] + r.byte_off;
    case BK_GNM: return base + P.gns[r.id].off_m[r.par] + r.byte_off;
    case BK_GNMALL: return base + P.gns[r.id].off_mall[r.par] + r.byte_off;
  }
  return nullptr;
}

// ---------------------------------------------------------------------------------------------
// exchange descriptors
// ---------------------------------------------------------------------------------------------
static BufRef tref(const Plan& P, int t, int par, int row) {
  const TDesc& d = P.td[t];
  const long long rowb = (long long)(d.B ? d.B : P.B) * d.W * d.C * dtype_size(d.dtype);
  return BufRef{BK_TENSOR, t, par, (long long)(row + d.pad) * rowb};
}

// Transfers of one exchange point.  Ranks are global (P.grank(branch, patch)); buffer offsets use
// the patch index within the branch group (a group exchanges only among its own patches).
static XGroup make_group(const Plan& P, const Op& op, int sync, int par, std::vector<Xfer>& lb) {
  XGroup G;
  const int n = P.n;
  G.wait = sync;
  lb.clear();
  if (op.k == OP_HALO) {
    const HaloX& hx = P.halos[op.xid];
    const TDesc& d = P.td[hx.t];
    const size_t rowb = (size_t)P.B * d.W * d.C * dtype_size(d.dtype);
    const int h = d.rows, pd = sync ? par : 1 - par;
    G.cls = 1;
    for (int bq = 0; bq < P.nb; ++bq)
      for (int i = 0; i < n; ++i) {
        const int me = P.grank(bq, i);
        if (i > 0) {   // my top halo <- patch i-1's last row
          const int src = P.grank(bq, i - 1);
          Xfer x{1, src, me, tref(P, hx.t, par, h - 1), tref(P, hx.t, pd, -1), rowb};
          G.remote.push_back(x); lb.push_back(x);
          if (sync) { G.local.push_back({1, me, me, tref(P, hx.t, par, -1), tref(P, hx.t, 1 - par, -1), rowb});
                      lb.push_back({1, src, me, tref(P, hx.t, par, h - 1), tref(P, hx.t, 1 - par, -1), rowb}); }
        }
        if (i < n - 1 && hx.stride == 1) {   // my bottom halo <- patch i+1's first row
          const int src = P.grank(bq, i + 1);
          Xfer x{1, src, me, tref(P, hx.t, par, 0), tref(P, hx.t, pd, h), rowb};
          G.remote.push_back(x); lb.push_back(x);
          if (sync) { G.local.push_back({1, me, me, tref(P, hx.t, par, h), tref(P, hx.t, 1 - par, h), rowb});
                      lb.push_back({1, src, me, tref(P, hx.t, par, 0), tref(P, hx.t, 1 - par, h), rowb}); }
        }
      }
  } else if (op.k == OP_GN) {
    const size_t mb = (size_t)P.B * GN_G * 2 * sizeof(double);
    G.cls = 2; G.allgather = 1;
    G.ag_send = BufRef{BK_GNM, op.xid, par, 0};
    G.ag_recv = BufRef{BK_GNMALL, op.xid, par, 0};
    G.ag_bytes = mb;
    for (int bq = 0; bq < P.nb; ++bq)
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
          Xfer x{2, P.grank(bq, j), P.grank(bq, i), BufRef{BK_GNM, op.xid, par, 0},
                 BufRef{BK_GNMALL, op.xid, par, (long long)(j * mb)}, mb};
          if (i != j) G.remote.push_back(x);
          lb.push_back(x);
        }
  } else if (op.k == OP_KVX) {
    const AttnX& a = P.attns[op.xid];
    const TDesc& d = P.td[a.kv];
    const size_t rowb = (size_t)P.B * d.W * d.C * dtype_size(d.dtype);
    const int h = a.h, r = a.r;
    G.cls = 0;
    const bool fullmap = P.cfg.scheme == PCPP_SCHEME_FULLMAP;
    for (int bq = 0; bq < P.nb; ++bq) {
      auto R = [&](int i) { return P.grank(bq, i); };
      if (!sync && !fullmap) {            // PCPP async: only the p-fraction bands, p2p to i +- 1
        for (int i = 0; i < n && r > 0; ++i) {
          if (i > 0) { Xfer x{0, R(i - 1), R(i), tref(P, a.kv, par, h - r), BufRef{BK_TOP, op.xid, par, 0}, r * rowb}; G.remote.push_back(x); lb.push_back(x); }
          if (i < n - 1) { Xfer x{0, R(i + 1), R(i), tref(P, a.kv, par, 0), BufRef{BK_BOT, op.xid, par, 0}, r * rowb}; G.remote.push_back(x); lb.push_back(x); }
        }
      } else {                            // all-gather of the full map (warm-up, or DistriFusion)
        const int gp = fullmap ? par : 0;
        G.allgather = 1;
        G.ag_send = tref(P, a.kv, par, 0);
        G.ag_recv = BufRef{BK_GAT, op.xid, gp, 0};
        G.ag_bytes = (size_t)h * rowb;
        for (int i = 0; i < n; ++i)
          for (int j = 0; j < n; ++j) {
            Xfer x{0, R(j), R(i), tref(P, a.kv, par, 0), BufRef{BK_GAT, op.xid, gp, (long long)((size_t)j * h * rowb)}, (size_t)h * rowb};
            if (i != j) { G.remote.push_back(x); lb.push_back(x); }
          }
        if (!fullmap && r > 0) {          // warm-up seeds the band buffers for step k+1 (unpack)
          for (int i = 0; i < n; ++i) {
            if (i > 0) {
              G.local.push_back({0, R(i), R(i), BufRef{BK_GAT, op.xid, 0, (long long)((size_t)(i * h - r) * rowb)}, BufRef{BK_TOP, op.xid, par, 0}, r * rowb});
              lb.push_back({0, R(i - 1), R(i), tref(P, a.kv, par, h - r), BufRef{BK_TOP, op.xid, par, 0}, r * rowb});
            }
            if (i < n - 1) {
              G.local.push_back({0, R(i), R(i), BufRef{BK_GAT, op.xid, 0, (long long)((size_t)((i + 1) * h) * rowb)}, BufRef{BK_BOT, op.xid, par, 0}, r * rowb});
              lb.push_back({0, R(i + 1), R(i), tref(P, a.kv, par, 0), BufRef{BK_BOT, op.xid, par, 0}, r * rowb});
            }
          }
        }
      }
    }
  } else if (op.k == OP_EPSX) {
    // CFG device split: the partner (same patch, other branch) sends its eps rows into my
    // two-branch buffer eps2 [h][2][W][4]; my own rows go to my slot.  Needed in the same step
    // (synchronous every step, like DistriFusion's), then every rank applies CFG + DDIM itself.
    const TDesc& e = P.td[op.in0];
    const size_t row1 = (size_t)e.W * 4 * sizeof(float);
    G.cls = 3; G.wait = 1;
    for (int bq = 0; bq < 2; ++bq)
      for (int i = 0; i < n; ++i) {
        const int me = P.grank(bq, i), pa = P.grank(1 - bq, i);
        for (int r = 0; r < e.rows; ++r) {
          const BufRef own{BK_TENSOR, op.in0, par, (long long)(r * row1)};
          Xfer x{3, pa, me, own, BufRef{BK_TENSOR, op.out, par, (long long)((2 * r + 1 - bq) * row1)}, row1};
          G.remote.push_back(x); lb.push_back(x);
          lb.push_back({3, me, me, own, BufRef{BK_TENSOR, op.out, par, (long long)((2 * r + bq) * row1)}, row1});
        }
      }
  }
  return G;
}

XGroup make_group_public(const Plan& P, const Op& op, int sync, int par, std::vector<Xfer>& lb) {
  return make_group(P, op, sync, par, lb);
}

pcpp_status plan_build_exchanges(Plan& P) {
  P.op_xord.assign(P.ops.size(), -1);
  int nx = 0;
  for (size_t i = 0; i < P.ops.size(); ++i) {
    const OpK k = P.ops[i].k;
    if (((k == OP_HALO || k == OP_KVX || k == OP_GN) && P.n > 1) || k == OP_EPSX) P.op_xord[i] = nx++;
  }
  std::vector<CopySeg> host;
  std::vector<Xfer> lb;
  for (int sync = 0; sync < 2; ++sync)
    for (int par = 0; par < 2; ++par) {
      P.xg[sync][par].assign(nx, XGroup{});
      P.seg_remote[sync][par].assign(nx, Plan::SegRange{});
      P.seg_local[sync][par].assign(nx, Plan::SegRange{});
      for (size_t i = 0; i < P.ops.size(); ++i) {
        const int xo = P.op_xord[i];
        if (xo < 0) continue;
        XGroup G = make_group(P, P.ops[i], sync, par, lb);
        // loopback: every transfer is a device copy (all ranks' arenas live here)
        if (P.loopback) {
          Plan::SegRange sr; sr.first = (int)host.size();
          for (auto& x : lb) {
            host.push_back(CopySeg{resolve(P, x.src_rank, x.src), resolve(P, x.dst_rank, x.dst), (unsigned long long)x.bytes});
            sr.maxb = std::max<unsigned long long>(sr.maxb, x.bytes);
          }
          sr.count = (int)host.size() - sr.first;
          P.seg_remote[sync][par][xo] = sr;
        } else {
          Plan::SegRange sr; sr.first = (int)host.size();
          for (auto& x : G.local) {
            if (x.dst_rank != P.rank0) continue;
            host.push_back(CopySeg{resolve(P, 0, x.src), resolve(P, 0, x.dst), (unsigned long long)x.bytes});
            sr.maxb = std::max<unsigned long long>(sr.maxb, x.bytes);
          }
          sr.count = (int)host.size() - sr.first;
          P.seg_local[sync][par][xo] = sr;
        }
        P.xg[sync][par][xo] = std::move(G);
      }
    }
  if (!host.empty()) {
    CK(cudaMalloc(&P.segs_dev, host.size() * sizeof(CopySeg)));
    CK(cudaMemcpy(P.segs_dev, host.data(), host.size() * sizeof(CopySeg), cudaMemcpyHostToDevice));
  }
  return PCPP_OK;
}

// counted ledger: bytes of all cross-rank transfers of one async / warm-up step
void compute_ledgers(Plan& P, pcpp_info* info) {
  std::vector<Xfer> lb;
  for (int c = 0; c < 3; ++c) { info->bytes_counted_async[c] = 0; info->bytes_counted_warmup[c] = 0; }
  info->bytes_eps = 0;
  if (P.world == 1) return;
  for (const Op& op : P.ops) {
    if (op.k == OP_EPSX) {
      XGroup G = make_group(P, op, 0, 0, lb);
      for (auto& x : G.remote) info->bytes_eps += (long long)x.bytes;
      continue;
    }
    if ((op.k != OP_HALO && op.k != OP_KVX && op.k != OP_GN) || P.n == 1) continue;
    for (int sync = 0; sync < 2; ++sync) {
      XGroup G = make_group(P, op, sync, 0, lb);
      for (auto& x : G.remote) (sync ? info->bytes_counted_warmup : info->bytes_counted_async)[x.cls] += (long long)x.bytes;
    }
  }
}

// ---------------------------------------------------------------------------------------------
// NCCL
// ---------------------------------------------------------------------------------------------
pcpp_status plan_init_comm(Plan& P) {
  if (P.loopback || P.n == 1 || P.backend == PCPP_COMM_PEER) return PCPP_OK;
  P.nccl = nccl_api();
  if (!P.nccl) return PCPP_ERR_NCCL;
  ncclUniqueId id; std::memcpy(&id, P.cfg.nccl_id, sizeof id);
  ncclComm_t c = nullptr;
  ncclResult_t r = P.nccl->CommInitRank(&c, P.n, id, P.cfg.rank);
  if (r != 0) { set_error("ncclCommInitRank: %s", P.nccl->GetErrorString(r)); return PCPP_ERR_NCCL; }
  P.comm = c;
  return PCPP_OK;
}

void peer_barrier(Plan& P, cudaStream_t s) { launch_peer_barrier(P.bar, s); }

// Open every peer's arena (IPC handles in rank order, from pcpp_peer_handle on each rank) and build
// this rank's push lists: the loopback transfer list of every exchange point restricted to
// src == me, source in the own arena, destination at the same offset in the peer's arena (every
// rank's plan has the same layout).
pcpp_status plan_peer_connect(Plan& P, const void* handles) {
  if (P.backend != PCPP_COMM_PEER) { set_error("pcpp_peer_connect: plan does not use the PEER backend"); return PCPP_ERR_STATE; }
  if (P.peer_connected) { set_error("pcpp_peer_connect: already connected"); return PCPP_ERR_STATE; }
  const int me = P.rank0, n = P.world;
  char* own = P.rm[0].arena;
  const cudaIpcMemHandle_t* hs = reinterpret_cast<const cudaIpcMemHandle_t*>(handles);
  for (int j = 0; j < n; ++j) {
    if (j == me) { P.peer_base[j] = own; continue; }
    void* ptr = nullptr;
    CK(cudaIpcOpenMemHandle(&ptr, hs[j], cudaIpcMemLazyEnablePeerAccess));
    P.peer_base[j] = reinterpret_cast<char*>(ptr);
  }
  auto remote = [&](int rank, const BufRef& r) { return P.peer_base[rank] + (resolve(P, 0, r) - own); };
  std::vector<CopySeg> host;
  std::vector<Xfer> lb;
  for (int sync = 0; sync < 2; ++sync)
    for (int par = 0; par < 2; ++par) {
      P.seg_push[sync][par].assign(P.xg[sync][par].size(), Plan::SegRange{});
      for (size_t i = 0; i < P.ops.size(); ++i) {
        const int xo = P.op_xord[i];
        if (xo < 0) continue;
        make_group(P, P.ops[i], sync, par, lb);
        Plan::SegRange sr; sr.first = (int)host.size();
        for (const Xfer& x : lb) {
          if (x.src_rank != me) continue;
          host.push_back(CopySeg{resolve(P, 0, x.src), remote(x.dst_rank, x.dst), (unsigned long long)x.bytes});
          sr.maxb = std::max<unsigned long long>(sr.maxb, x.bytes);
        }
        sr.count = (int)host.size() - sr.first;
        P.seg_push[sync][par][xo] = sr;
      }
    }
  {   // final gather: my latent patch into row block `patch` of every rank's x0g (with the CFG split
      // both branches hold the same patch; branch 0 sends it)
    const size_t pb = (size_t)(P.H / P.n) * P.W * 4 * sizeof(float);
    P.seg_x0.first = (int)host.size();
    if (P.branch_of(me) == 0)
      for (int j = 0; j < n; ++j)
        host.push_back(CopySeg{own + P.off_lat, P.peer_base[j] + P.off_x0g + (size_t)P.patch_of(me) * pb, (unsigned long long)pb});
    P.seg_x0.count = (int)host.size() - P.seg_x0.first; P.seg_x0.maxb = pb;
  }
  CK(cudaMalloc(&P.push_dev, std::max<size_t>(1, host.size()) * sizeof(CopySeg)));
  CK(cudaMemcpy(P.push_dev, host.data(), host.size() * sizeof(CopySeg), cudaMemcpyHostToDevice));
  P.bar.n = n; P.bar.me = me;
  P.bar.flags = reinterpret_cast<const unsigned long long*>(own + P.off_sig);
  P.bar.epoch = reinterpret_cast<unsigned long long*>(own + P.off_sig) + 8;
  for (int j = 0; j < n; ++j) P.bar.remote[j] = reinterpret_cast<unsigned long long*>(P.peer_base[j] + P.off_sig) + me;
  P.peer_connected = true;
  return PCPP_OK;
}

#define NK(x) do { ncclResult_t r_ = (x); if (r_ != 0) { set_error("NCCL %s: %s", #x, P.nccl->GetErrorString(r_)); return PCPP_ERR_NCCL; } } while (0)

static pcpp_status exchange(Plan& P, int xo, int sync, int par) {
  const XGroup& G = P.xg[sync][par][xo];
  const bool now = sync || G.wait;        // consumed in this step (warm-up, or the CFG-split eps exchange)
  if (P.comm_off && !now) return PCPP_OK;
  if (P.loopback && P.xasync) {     // the NCCL protocol with device copies (test mode)
    const auto& sr = P.seg_remote[sync][par][xo];
    CK(cudaEventRecord(P.ev_x, P.s0));
    CK(cudaStreamWaitEvent(P.s1, P.ev_x, 0));
    if (P.xdelay) launch_spin(P.xdelay * 1000 * (1 + (xo * 7919 + par * 31 + sync) % 5), P.s1);
    launch_copy_segments(P.segs_dev + sr.first, sr.count, sr.maxb, P.s1);
    if (G.wait) {
      CK(cudaEventRecord(P.ev_x, P.s1));
      CK(cudaStreamWaitEvent(P.s0, P.ev_x, 0));
    }
    return PCPP_OK;
  }
  if (P.loopback) {
    const auto& sr = P.seg_remote[sync][par][xo];
    launch_copy_segments(P.segs_dev + sr.first, sr.count, sr.maxb, P.s0);
    P.launches_per_step += sr.count > 0;
    return PCPP_OK;
  }
  if (P.backend == PCPP_COMM_PEER) {
    // one-sided pushes of this rank's data into the peers' buffers (the loopback transfer list
    // restricted to src == me).  Async: on the comm stream behind the producer, consumed one step
    // later (the step-start barrier orders it).  Warm-up: on the compute stream, then a barrier;
    // an all-gather of attention K/V first waits until every peer has left the previous attention
    // layer (the gather buffer is shared by the layers of a level).
    const auto& sr = P.seg_push[sync][par][xo];
    if (!now) {
      CK(cudaEventRecord(P.ev_x, P.s0));
      CK(cudaStreamWaitEvent(P.s1, P.ev_x, 0));
      launch_copy_segments(P.push_dev + sr.first, sr.count, sr.maxb, P.s1);
      P.launches_per_step += sr.count > 0;
    } else {
      if (G.allgather && G.cls == 0) { peer_barrier(P, P.s0); P.launches_per_step += 1; }
      launch_copy_segments(P.push_dev + sr.first, sr.count, sr.maxb, P.s0);
      peer_barrier(P, P.s0);
      P.launches_per_step += (sr.count > 0) + 1;
    }
    return PCPP_OK;
  }
  ncclComm_t comm = reinterpret_cast<ncclComm_t>(P.comm);
  const int me = P.rank0;
  CK(cudaEventRecord(P.ev_x, P.s0));
  CK(cudaStreamWaitEvent(P.s1, P.ev_x, 0));
  if (G.allgather) {
    NK(P.nccl->AllGather(resolve(P, 0, G.ag_send), resolve(P, 0, G.ag_recv), G.ag_bytes, nccl_int8, comm, P.s1));
  } else {
    NK(P.nccl->GroupStart());
    for (const Xfer& x : G.remote) {
      if (x.src_rank == me) NK(P.nccl->Send(resolve(P, 0, x.src), x.bytes, nccl_int8, x.dst_rank, comm, P.s1));
      if (x.dst_rank == me) NK(P.nccl->Recv(resolve(P, 0, x.dst), x.bytes, nccl_int8, x.src_rank, comm, P.s1));
    }
    NK(P.nccl->GroupEnd());
  }
  if (G.wait) {
    CK(cudaEventRecord(P.ev_x, P.s1));
    CK(cudaStreamWaitEvent(P.s0, P.ev_x, 0));
    const auto& sr = P.seg_local[sync][par][xo];
    launch_copy_segments(P.segs_dev + sr.first, sr.count, sr.maxb, P.s0);
  }
  return PCPP_OK;
}

// ---------------------------------------------------------------------------------------------
// the step
// ---------------------------------------------------------------------------------------------
// temb for all S steps (reading D19; SURVEY §8(a) a9 "precomputed for all S steps"): per step the
// sinusoid -> Linear -> SiLU -> Linear (+ cond for the conditional branch), then the ResBlock
// projections of 4 steps (8 embedding vectors) per pass over the [J][T] matrix.  Enqueued on s0;
// called at plan time and whenever the cond vector changes.
pcpp_status temb_precompute(Plan& P) {
  cudaStream_t s = P.s0;
  for (int k0 = 0; k0 < P.S; k0 += 4) {
    const int cs = std::min(4, P.S - k0);
    for (int kk = 0; kk < cs; ++kk)
      launch_temb(P.wf32 + P.t_w1, P.wf32 + P.t_b1, P.wf32 + P.t_w2, P.wf32 + P.t_b2, P.cond, P.taus, P.kseq + k0 + kk,
                  P.T, P.SIN, P.hid, P.emb_all + (size_t)kk * 2 * P.T, s);
    launch_temb_proj_multi(P.wf32 + P.t_wt, P.wf32 + P.t_bt, P.emb_all, P.T, P.J, 2 * cs,
                           P.tproj_all + (size_t)k0 * 2 * P.J, s);
  }
  CK(cudaGetLastError());
  return PCPP_OK;
}

void launch_gemm_tc_or_simt(const Plan& P, const GemmArgs& g, cudaStream_t s);
void launch_attn_tc_or_simt(const Plan& P, const AttnArgs& a, cudaStream_t s);

static unsigned op_kind(OpK k) {
  switch (k) {
    case OP_CONV: case OP_GEMM: return K_GEMM;
    case OP_ATTN: return K_ATTN;
    case OP_GN: return K_GN;
    case OP_HALO: case OP_KVX: case OP_EPSX: return K_XCH;
    case OP_XATTN: return K_ATTN;
    case OP_END: return K_END;
    default: return K_MISC;
  }
}

void gemm_tc_autotune(const GemmArgs& g, cudaStream_t s);
bool gemm_tc_supported(const GemmArgs& g);

// Per-shape GEMM configuration search on the plan's own buffers (before any graph capture).
void gemm_tune_load(const char* path);
void gemm_tune_save(const char* path);

pcpp_status plan_autotune(Plan& P) {
  if (!P.use_tc) return PCPP_OK;
  static const int env = getenv("PCPP_AUTOTUNE") ? atoi(getenv("PCPP_AUTOTUNE")) : 1;
  if (!env) return PCPP_OK;
  static bool loaded = false;
  if (!loaded && getenv("PCPP_TUNE_FILE")) { gemm_tune_load(getenv("PCPP_TUNE_FILE")); loaded = true; }
  const size_t es = dtype_size(P.dtype);
  const char* wm = reinterpret_cast<const char*>(P.wmat);
  for (const Op& op : P.ops) {
    if (op.k != OP_CONV && op.k != OP_GEMM) continue;
    GemmArgs g;
    g.a0 = view(P, 0, op.in0, 0);
    g.c0 = g.a0.C; g.cin = g.a0.C;
    if (op.in1 >= 0) { g.a1 = view(P, 0, op.in1, 0); g.cin += g.a1.C; }
    g.taps = op.k == OP_CONV ? 9 : 1;
    g.stride = op.stride;
    const ActView o = view(P, 0, op.out, 0);
    g.rows_out = o.rows; g.w_out = o.W; g.B = P.B;
    g.w = op.w_f32 ? (const void*)(P.wf32 + op.w) : (const void*)(wm + (size_t)op.w * es);
    g.wdtype = op.w_f32 ? DT_F32 : P.dtype;
    g.N = op.N;
    g.bias = op.b >= 0 ? P.wf32 + op.b : nullptr;
    if (op.temb_off >= 0) { g.temb = P.tproj + op.temb_off; g.temb_ld = P.J; }
    if (op.res >= 0) g.res = view(P, 0, op.res, 0);
    g.out = o;
    if (op.out2 >= 0) { g.out2 = view(P, 0, op.out2, 0); g.n_split = op.n_split; }
    g.geglu = op.geglu;
    g.ws = P.ws; g.ws_elems = P.ws_elems;
    int slots = 0;
    if (op.gn_fuse >= 0) { g.gn_part = reinterpret_cast<double*>(P.rm[0].arena + P.off_epart); g.gn_slots = &slots; }
    if (gemm_tc_supported(g)) gemm_tc_autotune(g, P.s0);
  }
  if (getenv("PCPP_TUNE_SAVE")) gemm_tune_save(getenv("PCPP_TUNE_SAVE"));
  CK(cudaStreamSynchronize(P.s0));
  CK(cudaGetLastError());
  return PCPP_OK;
}

// _XF models: lay the context out per level and compute every layer's context keys/values
// [ctx W_k ; ctx W_v] with the plan's GEMM kernels (once per context; reading D26)
pcpp_status context_setup(Plan& P, const float* ctx_host) {
  const size_t es = dtype_size(P.dtype);
  CK(cudaMemcpyAsync(P.ctx_f32, ctx_host, (size_t)2 * 77 * P.ctx_dim * 4, cudaMemcpyHostToDevice, P.s0));
  for (int l = 0; l < P.levels; ++l) {
    ActView v; v.base = P.ctx_level[l]; v.rows = P.ctx_rows(l); v.B = B_CFG; v.W = P.W >> l; v.C = P.ctx_dim; v.dtype = P.dtype;
    launch_ctx_layout(P.ctx_f32, v, 77, P.s0);
  }
  const char* wm = reinterpret_cast<const char*>(P.wmat);
  for (const XAttnX& xa : P.xattns) {
    GemmArgs g;
    g.a0.base = P.ctx_level[xa.level]; g.a0.rows = P.ctx_rows(xa.level); g.a0.B = B_CFG; g.a0.W = P.W >> xa.level;
    g.a0.C = P.ctx_dim; g.a0.dtype = P.dtype;
    g.c0 = g.cin = P.ctx_dim; g.taps = 1; g.stride = 1;
    g.rows_out = g.a0.rows; g.w_out = g.a0.W; g.B = B_CFG;
    g.w = wm + (size_t)xa.w * es; g.wdtype = P.dtype; g.N = 2 * xa.C;
    g.out = g.a0; g.out.base = xa.kv; g.out.C = 2 * xa.C;
    g.ws = P.ws; g.ws_elems = P.ws_elems;
    launch_gemm_tc_or_simt(P, g, P.s0);
  }
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(P.s0));
  P.ctx_set = true;
  return PCPP_OK;
}

pcpp_status run_step(Plan& P, float* latent, int sync, int par, unsigned mask) {
  const int n = P.n, nr = P.nr;
  cudaStream_t s = P.s0;
  const int lps_prev = P.launches_per_step;
  P.launches_per_step = 0;
  const long long fb0 = simt_fallback_count(), lc0 = launch_count();
  // PEER: every peer has finished step k-1 (its compute and its pushes) before this step reads what
  // they pushed during k-1 and before this step pushes into the buffers they read during k-1
  if (P.backend == PCPP_COMM_PEER && P.world > 1 && (mask & K_XCH)) {
    if (!P.peer_connected) { set_error("PEER backend: pcpp_peer_connect has not been called"); return PCPP_ERR_STATE; }
    peer_barrier(P, s);
    P.launches_per_step += 1;
  }
  const size_t es = dtype_size(P.dtype);
  const char* wm = reinterpret_cast<const char*>(P.wmat);
  for (size_t oi = 0; oi < P.ops.size(); ++oi) {
    if (P.op_ev_on) cudaEventRecord(P.op_ev[oi], s);
    const Op& op = P.ops[oi];
    const int xo_all = P.op_xord[oi];
    const unsigned kind = op_kind(op.k);
    if (!(mask & kind) && !(op.k == OP_GN && (mask & K_XCH))) continue;
    const int xo = (mask & K_XCH) ? xo_all : -1;
    const bool do_op = (mask & kind) != 0;
    if (!do_op && op.k != OP_GN) continue;
    switch (op.k) {
      case OP_TEMB:
        // the temb MLP and every ResBlock's projection depend only on (tau_k, cond): precomputed for
        // all S steps (temb_precompute); the step selects its row by the device step counter
        launch_temb_select(P.tproj_all, P.k_dev, 2 * P.J, P.tproj, s);
        P.launches_per_step += 1;
        break;
      case OP_PREP: {
        const int h = P.H / n;
        for (int vr = 0; vr < nr; ++vr) {
          const float* lat = latent + (P.loopback ? (size_t)P.patch_of(vr) * h * P.W * 4 : 0);
          launch_prep_latent(lat, view(P, vr, op.out, par), s);
        }
        P.launches_per_step += nr;
        break;
      }
      case OP_HALO:
      case OP_KVX:
      case OP_EPSX:
        if (xo >= 0) { pcpp_status st = exchange(P, xo, sync, par); if (st != PCPP_OK) return st; }
        break;
      case OP_CONV:
      case OP_GEMM:
        for (int vr = 0; vr < nr; ++vr) {
          GemmArgs g;
          g.a0 = view(P, vr, op.in0, par);
          g.c0 = g.a0.C; g.cin = g.a0.C;
          if (op.in1 >= 0) { g.a1 = view(P, vr, op.in1, par); g.cin += g.a1.C; }
          g.taps = op.k == OP_CONV ? 9 : 1;
          g.stride = op.stride;
          const ActView o = view(P, vr, op.out, par);
          g.rows_out = o.rows; g.w_out = o.W; g.B = P.B;
          g.w = op.w_f32 ? (const void*)(P.wf32 + op.w) : (const void*)(wm + (size_t)op.w * es);
          g.wdtype = op.w_f32 ? DT_F32 : P.dtype;
          g.N = op.N;
          g.bias = op.b >= 0 ? P.wf32 + op.b : nullptr;
          // temb rows [2][J]: batch b of this rank is CFG branch b, or the rank's branch with the split
          if (op.temb_off >= 0) { g.temb = P.tproj + op.temb_off + (size_t)P.branch_of(P.rank0 + vr) * P.J; g.temb_ld = P.J; }
          if (op.res >= 0) g.res = view(P, vr, op.res, par);
          g.out = o;
          if (op.out2 >= 0) { g.out2 = view(P, vr, op.out2, par); g.n_split = op.n_split; }
          g.ws = P.ws; g.ws_elems = P.ws_elems;
          if (op.gn_fuse >= 0) {
            g.gn_part = reinterpret_cast<double*>(P.rm[vr].arena + P.off_epart);
            g.gn_slots = &P.gn_slots[(size_t)vr * P.gns.size() + op.gn_fuse];
          }
          if (op.geglu) {    // fused GEGLU epilogue on the tensor-core path, else GEMM into tmp + GEGLU kernel
            g.geglu = 1;
            if (!(P.use_tc && gemm_tc_supported(g))) {
              g.geglu = 0;
              g.out = view(P, vr, op.tmp, par);
              launch_gemm_tc_or_simt(P, g, s);
              launch_geglu(g.out, o, s);
              continue;
            }
          }
          launch_gemm_tc_or_simt(P, g, s);
        }
        P.launches_per_step += nr;
        break;
      case OP_GN: {
        const GnX& gx = P.gns[op.xid];
        auto stats_args = [&](int vr) {
          GnStatsArgs a;
          a.x0 = view(P, vr, op.in0, par); a.c0 = a.x0.C; a.C = gx.C;
          if (op.in1 >= 0) a.x1 = view(P, vr, op.in1, par);
          char* base = P.rm[vr].arena;
          a.partial = reinterpret_cast<double*>(base + gx.off_part);
          a.m_out = reinterpret_cast<double*>(base + gx.off_m[par]);
          a.nchunk = gx.nchunk;
          return a;
        };
        auto apply_args = [&](int vr) {
          GnApplyArgs a;
          a.x0 = view(P, vr, op.in0, par); a.c0 = a.x0.C; a.C = gx.C;
          if (op.in1 >= 0) a.x1 = view(P, vr, op.in1, par);
          a.out = view(P, vr, op.out, par);
          a.gamma = P.wf32 + op.g; a.beta = P.wf32 + op.be; a.silu = op.silu;
          char* base = P.rm[vr].arena;
          a.nranks = n; a.count = gx.count;
          a.m_fresh = reinterpret_cast<const double*>(base + gx.off_m[par]);
          if (n == 1) a.mode = 0;
          else if (sync) { a.mode = 1; a.mall = reinterpret_cast<const double*>(base + gx.off_mall[par]); }
          else {
            a.mode = 2;
            a.mall = reinterpret_cast<const double*>(base + gx.off_mall[1 - par]);
            a.m_prev = reinterpret_cast<const double*>(base + gx.off_m[1 - par]);
          }
          return a;
        };
        {
          // no synchronous exchange of this step's sums: the apply kernel sums the producer's partial
          // slots itself (no finalize launch) and publishes m[par]; the asynchronous exchange of m[par]
          // then follows the apply
          const bool can_merge = n == 1 || !sync;
          std::vector<int> merged(nr, 0);
          for (int vr = 0; vr < nr && do_op; ++vr) {
            const int slots = P.gn_slots[(size_t)vr * P.gns.size() + op.xid];
            if (slots > 0 && can_merge) { merged[vr] = slots; continue; }
            if (slots > 0)
              launch_gn_finalize(reinterpret_cast<const double*>(P.rm[vr].arena + P.off_epart), slots, P.B,
                                 reinterpret_cast<double*>(P.rm[vr].arena + gx.off_m[par]), s);
            else if (can_merge) {
              launch_gn_stats(stats_args(vr), s, false);
              merged[vr] = -gx.nchunk;              // slots of the stats kernel
            } else
              launch_gn_stats(stats_args(vr), s);
          }
          if (xo >= 0 && !can_merge) { pcpp_status st = exchange(P, xo, sync, par); if (st != PCPP_OK) return st; }
          for (int vr = 0; vr < nr && do_op; ++vr) {
            GnApplyArgs a = apply_args(vr);
            char* base = P.rm[vr].arena;
            if (merged[vr] > 0) {
              a.part = reinterpret_cast<const double*>(base + P.off_epart); a.nslots = merged[vr];
            } else if (merged[vr] < 0) {
              a.part = reinterpret_cast<const double*>(base + gx.off_part); a.nslots = -merged[vr];
            }
            if (a.nslots) a.m_write = reinterpret_cast<double*>(base + gx.off_m[par]);
            launch_gn_apply(a, s);
          }
          if (xo >= 0 && can_merge) { pcpp_status st = exchange(P, xo, sync, par); if (st != PCPP_OK) return st; }
        }
        break;
      }
      case OP_ATTN: {
        const AttnX& ax = P.attns[op.xid];
        const TDesc& kvd = P.td[ax.kv];
        const size_t rowb = (size_t)P.B * kvd.W * kvd.C * es;
        const bool fullmap = P.cfg.scheme == PCPP_SCHEME_FULLMAP;
        for (int vr = 0; vr < nr; ++vr) {
          const int i = P.patch_of(P.rank0 + vr);
          char* base = P.rm[vr].arena;
          AttnArgs a;
          a.q = view(P, vr, op.in0, par).base;
          a.h = ax.h; a.B = P.B; a.W = ax.W; a.C = ax.C; a.dtype = P.dtype;
          a.out = view(P, vr, op.out, par).base;
          const void* local = view(P, vr, op.in1, par).base;
          int ns = 0;
          if (n == 1) {
            a.src[ns++] = AttnSrc{local, ax.h};
          } else if (sync || fullmap) {
            const int gp = fullmap ? (sync ? par : 1 - par) : 0;
            const char* gat = base + ax.off_gat[gp];
            if (i > 0) a.src[ns++] = AttnSrc{gat, i * ax.h};
            a.src[ns++] = AttnSrc{local, ax.h};
            if (i < n - 1) a.src[ns++] = AttnSrc{gat + (size_t)(i + 1) * ax.h * rowb, (n - 1 - i) * ax.h};
          } else {
            if (i > 0 && ax.r > 0) a.src[ns++] = AttnSrc{base + ax.off_top[1 - par], ax.r};
            a.src[ns++] = AttnSrc{local, ax.h};
            if (i < n - 1 && ax.r > 0) a.src[ns++] = AttnSrc{base + ax.off_bot[1 - par], ax.r};
          }
          a.nsrc = ns;
          a.ws = P.ws; a.ws_elems = P.ws_elems;
          launch_attn_tc_or_simt(P, a, s);
        }
        P.launches_per_step += nr;
        break;
      }
      case OP_LN:
        for (int vr = 0; vr < nr; ++vr)
          if (!launch_layernorm(view(P, vr, op.in0, par), view(P, vr, op.out, par), P.wf32 + op.g, P.wf32 + op.be, s)) {
            set_error("LayerNorm: unsupported channel count %d", P.td[op.in0].C); return PCPP_ERR_UNSUPPORTED;
          }
        P.launches_per_step += nr;
        break;
      case OP_XATTN: {     // cross-attention: queries of the patch, keys/values of the 77-token context
        const XAttnX& xa = P.xattns[op.xid];
        for (int vr = 0; vr < nr; ++vr) {
          const ActView q = view(P, vr, op.in0, par);
          AttnArgs a;
          a.q = q.base; a.h = q.rows; a.B = P.B; a.W = q.W; a.C = xa.C; a.dtype = P.dtype;
          a.out = view(P, vr, op.out, par).base;
          a.src[0] = AttnSrc{xa.kv, P.ctx_rows(xa.level), 77};
          a.nsrc = 1;
          a.ws = P.ws; a.ws_elems = P.ws_elems;
          launch_attn_tc_or_simt(P, a, s);
        }
        P.launches_per_step += nr;
        break;
      }
      case OP_UPS:
        for (int vr = 0; vr < nr; ++vr) launch_upsample2(view(P, vr, op.in0, par), view(P, vr, op.out, par), s);
        P.launches_per_step += nr;
        break;
      case OP_CONVOUT:
        for (int vr = 0; vr < nr; ++vr)
          launch_conv_out(view(P, vr, op.in0, par), P.wf32 + op.w, P.wf32 + op.b, view(P, vr, op.out, par), s);
        P.launches_per_step += nr;
        break;
      case OP_CFGDDIM: {
        const int h = P.H / n;
        for (int vr = 0; vr < nr; ++vr) {
          // CFG split in one process: both branches of a patch compute the same update; branch 0 writes it
          if (P.loopback && P.branch_of(vr) == 1) continue;
          float* lat = latent + (P.loopback ? (size_t)P.patch_of(vr) * h * P.W * 4 : 0);
          if (P.cfg.scheduler == PCPP_SCHED_ANCESTRAL)
            launch_cfg_ancestral(reinterpret_cast<const float*>(view(P, vr, op.in0, par).base), lat, h, P.W,
                                 P.patch_of(P.rank0 + vr) * h, P.cfg.guidance_scale, P.coef_anc, P.cfg.noise_seed, P.k_dev, s);
          else if (P.cfg.scheduler == PCPP_SCHED_DPMPP2M)
            launch_cfg_dpmpp(reinterpret_cast<const float*>(view(P, vr, op.in0, par).base), lat,
                             P.x0_hist + (size_t)vr * h * P.W * 4, h, P.W, P.cfg.guidance_scale, P.coef_dpm, P.k_dev, s);
          else
            launch_cfg_ddim(reinterpret_cast<const float*>(view(P, vr, op.in0, par).base), lat, h, P.W,
                            P.cfg.guidance_scale, P.coef, P.k_dev, s);
        }
        P.launches_per_step += nr;
        break;
      }
      case OP_END:
        launch_step_end(P.k_dev, s);
        P.launches_per_step += 1;
        break;
    }
  }
  if (P.op_ev_on) cudaEventRecord(P.op_ev[P.ops.size()], s);
  P.simt_fallbacks = std::max<int>(P.simt_fallbacks, (int)(simt_fallback_count() - fb0));
  // every kernel a whole step enqueued (exact); partial (profiling) steps leave the record alone
  P.launches_per_step = mask == K_ALL ? (int)(launch_count() - lc0) : lps_prev;
  CK(cudaGetLastError());
  return PCPP_OK;
}

// Per-op device time of one eager step (events between ops; the host runs ahead of the device for
// every op longer than the launch latency), printed to stderr.  Debug / tuning aid only.  The
// step-end op (device step counter) is excluded, so the plan's step bookkeeping is unchanged.
void print_op_timing(Plan& P, float* latent, int sync, int par) {
  const size_t n = P.ops.size() + 1;
  P.op_ev.resize(n);
  for (auto& e : P.op_ev) cudaEventCreate(&e);
  P.op_ev_on = true;
  for (int rep = 0; rep < 2; ++rep) run_step(P, latent, sync, par, K_ALL & ~K_END);   // k_dev untouched
  cudaStreamSynchronize(P.s0);
  P.op_ev_on = false;
  static const char* names[] = {"TEMB", "PREP", "HALO", "CONV", "GEMM", "GN", "KVX", "ATTN", "UPS", "COUT", "CFG", "END"};
  double tot = 0;
  for (size_t oi = 0; oi + 1 < n; ++oi) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, P.op_ev[oi], P.op_ev[oi + 1]);
    tot += ms;
    const Op& op = P.ops[oi];
    const int k = (int)op.k;
    if (op.k == OP_CONV || op.k == OP_GEMM) {
      const TDesc& o = P.td[op.out];
      const int cin = P.td[op.in0].C + (op.in1 >= 0 ? P.td[op.in1].C : 0);
      const double fl = 2.0 * o.rows * P.B * o.W * op.N * (op.k == OP_CONV ? 9 : 1) * cin * P.nr;
      fprintf(stderr, "op %3zu %-4s rows=%3d W=%3d N=%4d cin=%4d s=%d res=%d gn=%d out2=%d %8.1f us %6.0f TF/s\n", oi,
              names[k], o.rows, o.W, op.N, cin, op.stride, op.res >= 0, op.gn_fuse >= 0, op.out2 >= 0, ms * 1e3,
              fl / (ms * 1e-3) / 1e12);
    } else {
      fprintf(stderr, "op %3zu %-4s %8.1f us\n", oi, k >= 0 && k < 12 ? names[k] : "?", ms * 1e3);
    }
  }
  fprintf(stderr, "op-timing total %.3f ms\n", tot);
  for (auto& e : P.op_ev) cudaEventDestroy(e);
  P.op_ev.clear();
}

void op_work(const Plan& P, unsigned kind, int sync, double* flops, double* bytes, int* launches) {
  double f = 0, by = 0; int nl = 0;
  const int n = P.n;
  const double es = (double)dtype_size(P.dtype);
  for (size_t oi = 0; oi < P.ops.size(); ++oi) {
    const Op& op = P.ops[oi];
    if (!(op_kind(op.k) & kind)) continue;
    switch (op.k) {
      case OP_CONV: case OP_GEMM: {
        const TDesc& o = P.td[op.geglu ? op.tmp : op.out];
        double cin = P.td[op.in0].C + (op.in1 >= 0 ? P.td[op.in1].C : 0);
        const double M = (double)o.rows * P.B * o.W;
        f += 2.0 * M * op.N * (op.k == OP_CONV ? 9 : 1) * cin * P.nr;
        nl += P.nr;
        break;
      }
      case OP_ATTN: {
        const AttnX& a = P.attns[op.xid];
        for (int vr = 0; vr < P.nr; ++vr) {
          const int i = P.patch_of(P.rank0 + vr);
          int kv = a.h;
          if (n > 1) {
            if (sync || P.cfg.scheme == PCPP_SCHEME_FULLMAP) kv = a.h * n;
            else kv = a.h + (i > 0 ? a.r : 0) + (i < n - 1 ? a.r : 0);
          }
          f += 4.0 * ((double)a.h * a.W) * ((double)kv * a.W) * a.C * P.B;
          by += ((double)a.h * a.W * a.C * 2 + (double)kv * a.W * 2 * a.C) * P.B * es;   // Q + O + K/V
        }
        nl += P.nr;
        break;
      }
      case OP_XATTN: {
        const XAttnX& xa = P.xattns[op.xid];
        const TDesc& q = P.td[op.in0];
        f += 4.0 * ((double)q.rows * q.W) * 77.0 * xa.C * P.B * P.nr;
        by += ((double)q.rows * q.W * xa.C * 2 + 77.0 * 2 * xa.C) * P.B * es * P.nr;
        nl += P.nr;
        break;
      }
      case OP_GN: {
        const TDesc& x = P.td[op.in0];
        double C = x.C + (op.in1 >= 0 ? P.td[op.in1].C : 0);
        by += 3.0 * x.rows * P.B * x.W * C * es * P.nr;     // stats read + apply read/write
        nl += 2 * P.nr;
        break;
      }
      default:
        nl += 1;
        break;
    }
  }
  if (kind & K_XCH) {
    pcpp_info info;
    compute_ledgers(const_cast<Plan&>(P), &info);
    for (int c = 0; c < 3; ++c) by += (double)(sync ? info.bytes_counted_warmup[c] : info.bytes_counted_async[c]);
  }
  *flops = f; *bytes = by; *launches = nl;
}

}  // namespace pcpp
