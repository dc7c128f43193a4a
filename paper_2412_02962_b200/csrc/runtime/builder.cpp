// Layer-program builder: walks the SDXL-shaped or TINY stack once at plan time and
// emits the op list, tensor table, exchange points and weight manifest.  Independent of the
// oracle: this is the product's own transcription of the stack.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include "runtime.h"

namespace pcpp {

static thread_local char g_err[512];
const char* set_error(const char* fmt, ...) {
  va_list ap; va_start(ap, fmt); vsnprintf(g_err, sizeof g_err, fmt, ap); va_end(ap);
  return g_err;
}
const char* last_error_msg() { return g_err; }

// Eq. 1 "p h" rows; reading D1: floor(p h + 1e-9), >= 1 if p > 0, <= h.
int band_rows(double p, int h) {
  if (p <= 0.0) return 0;
  long long r = (long long)std::floor(p * (double)h + 1e-9);
  if (r < 1) r = 1;
  if (r > h) r = h;
  return (int)r;
}

pcpp_status validate(int H, int W, int C, int n, double p, int w, const pcpp_config* cfg) {
  if (!cfg) { set_error("cfg is NULL"); return PCPP_ERR_INVALID; }
  if (cfg->model < PCPP_MODEL_TINY || cfg->model > PCPP_MODEL_SDXL_XF) { set_error("unknown model %d", cfg->model); return PCPP_ERR_INVALID; }
  const bool sdxl_like = cfg->model == PCPP_MODEL_SDXL || cfg->model == PCPP_MODEL_SDXL_XF;
  const int levels = sdxl_like ? 3 : 1;
  const int div = 1 << (levels - 1);
  if (n < 1 || n > 8) { set_error("n_patches must be in [1, 8], got %d", n); return PCPP_ERR_INVALID; }
  if (C != 4) { set_error("latent channels must be 4, got %d", C); return PCPP_ERR_INVALID; }
  if (H <= 0 || W <= 0 || H % (n * div) != 0) { set_error("H=%d must be a positive multiple of n*%d=%d", H, div, n * div); return PCPP_ERR_INVALID; }
  const int wq = sdxl_like ? 32 : 8;
  if (W % wq != 0) { set_error("W=%d must be a multiple of %d", W, wq); return PCPP_ERR_INVALID; }
  if (!(p >= 0.0 && p <= 1.0)) { set_error("cond_fraction must be in [0, 1] (p > 1 undefined, P:209), got %g", p); return PCPP_ERR_INVALID; }
  if (cfg->num_steps < 1 || cfg->num_steps > 1000) { set_error("num_steps must be in [1, 1000]"); return PCPP_ERR_INVALID; }
  if (n > 1 && w < 1) { set_error("warmup_steps must be >= 1 when n > 1 (reading D20)"); return PCPP_ERR_INVALID; }
  if (w < 0 || w > cfg->num_steps) { set_error("warmup_steps must be in [0, num_steps]"); return PCPP_ERR_INVALID; }
  if (cfg->guidance_scale < 1.0f) { set_error("guidance_scale must be >= 1 (Eq. 2, P:39)"); return PCPP_ERR_INVALID; }
  if (cfg->scheduler != PCPP_SCHED_DDIM && cfg->scheduler != PCPP_SCHED_DPMPP2M && cfg->scheduler != PCPP_SCHED_ANCESTRAL) {
    set_error("scheduler must be PCPP_SCHED_DDIM, PCPP_SCHED_DPMPP2M or PCPP_SCHED_ANCESTRAL"); return PCPP_ERR_INVALID;
  }
  if (cfg->precision != PCPP_FP32 && cfg->precision != PCPP_BF16) { set_error("bad precision"); return PCPP_ERR_INVALID; }
  if (cfg->scheme < 0 || cfg->scheme > 2) { set_error("bad scheme"); return PCPP_ERR_INVALID; }
  if (cfg->cfg_split != 0 && cfg->cfg_split != 1) { set_error("cfg_split must be 0 or 1"); return PCPP_ERR_INVALID; }
  if (cfg->cfg_split && (cfg->model == PCPP_MODEL_TINY_XF || cfg->model == PCPP_MODEL_SDXL_XF)) {
    set_error("cfg_split with the _XF models is not supported"); return PCPP_ERR_UNSUPPORTED;
  }
  if (cfg->cfg_split && cfg->comm_backend == PCPP_COMM_NCCL) {
    set_error("cfg_split needs the PEER or LOOPBACK backend (NCCL would need per-branch communicators)"); return PCPP_ERR_UNSUPPORTED;
  }
  if (cfg->comm_backend == PCPP_COMM_NCCL) {
    if (cfg->world != n) { set_error("world (%d) must equal n_patches (%d)", cfg->world, n); return PCPP_ERR_INVALID; }
    if (cfg->rank < 0 || cfg->rank >= n) { set_error("rank out of range"); return PCPP_ERR_INVALID; }
    if (n > 1 && !cfg->nccl_id) { set_error("nccl_id required for the NCCL backend"); return PCPP_ERR_INVALID; }
  } else if (cfg->comm_backend == PCPP_COMM_PEER) {
    const int world = cfg->cfg_split ? 2 * n : n;
    if (cfg->world != world) { set_error("world (%d) must equal n_patches%s (%d)", cfg->world, cfg->cfg_split ? " x 2 (cfg_split)" : "", world); return PCPP_ERR_INVALID; }
    if (cfg->rank < 0 || cfg->rank >= world) { set_error("rank out of range"); return PCPP_ERR_INVALID; }
    if (world > 8) { set_error("PEER backend: at most 8 ranks"); return PCPP_ERR_INVALID; }
  } else if (cfg->comm_backend != PCPP_COMM_LOOPBACK) { set_error("bad comm_backend"); return PCPP_ERR_INVALID; }
  return PCPP_OK;
}

namespace {

struct Builder {
  Plan& P;
  int act;   // activation dtype
  explicit Builder(Plan& p) : P(p), act(p.dtype) {}

  long long take(const std::string& name, std::vector<long long> shape) {
    long long nume = 1;
    for (long long d : shape) nume *= d;
    P.man_name.push_back(name);
    P.man_shape.push_back(shape);
    P.man_off.push_back((long long)P.blob_len);
    long long off = (long long)P.blob_len;
    P.blob_len += (size_t)nume;
    return off;
  }
  long long numel(const std::vector<long long>& s) { long long x = 1; for (auto d : s) x *= d; return x; }
  // upload a manifest tensor into an arena; returns arena offset
  long long up_mat(long long blob_off, long long nume) {
    long long o = P.wmat_len; P.uploads.push_back({blob_off, nume, 0, o}); P.wmat_len += nume;
    P.wmat_len = (P.wmat_len + 63) & ~63LL; return o;
  }
  long long up_f32(long long blob_off, long long nume) {
    long long o = P.wf32_len; P.uploads.push_back({blob_off, nume, 1, o}); P.wf32_len += nume;
    P.wf32_len = (P.wf32_len + 63) & ~63LL; return o;
  }
  long long vec(const std::string& name, int C) { return up_f32(take(name, {C}), C); }

  int rows_at(int level) const { return (P.H >> level) / P.n; }
  int w_at(int level) const { return P.W >> level; }

  int tensor(const std::string& name, int level, int C, int dtype, int pad, int dbl, int B = 0) {
    TDesc t;
    t.name = name; t.level = level; t.rows = rows_at(level); t.W = w_at(level); t.C = C; t.dtype = dtype;
    t.pad = pad; t.dbl = dbl; t.B = B;
    t.bytes = (size_t)(t.rows + 2 * pad) * (B ? B : P.B) * t.W * C * dtype_size(dtype);
    P.td.push_back(t);
    return (int)P.td.size() - 1;
  }
  int conv_in_tensor(const std::string& name, int level, int C) { return tensor(name, level, C, act, 1, 1); }

  Op& op(OpK k) { P.ops.push_back(Op{}); P.ops.back().k = k; return P.ops.back(); }

  void halo(int t, int stride) {
    if (P.n == 1) return;
    P.halos.push_back({t, stride});
    Op& o = op(OP_HALO); o.in0 = t; o.stride = stride; o.xid = (int)P.halos.size() - 1;
  }

  void gn(int x0, int x1, int out, const std::string& pre, int silu) {
    const TDesc& a = P.td[x0];
    int C = a.C + (x1 >= 0 ? P.td[x1].C : 0);
    GnX g{}; g.C = C; g.rows = a.rows; g.W = a.W;
    g.nchunk = gn_stats_chunks(a.rows, a.W, C);
    g.count = (double)(a.rows * P.n) * a.W * (C / GN_G);
    P.gns.push_back(g);
    Op& o = op(OP_GN); o.in0 = x0; o.in1 = x1; o.out = out; o.silu = silu;
    o.g = vec(pre + ".g", C); o.be = vec(pre + ".b", C);
    o.xid = (int)P.gns.size() - 1;
  }

  // conv3x3 from padded input t_in
  int conv(int t_in, const std::string& wname, int cout, int stride, int out_t, int temb_off, int res) {
    const TDesc& a = P.td[t_in];
    long long wo = take(wname + ".w", {cout, 3, 3, a.C});
    long long bo = take(wname + ".b", {cout});
    Op& o = op(OP_CONV); o.in0 = t_in; o.out = out_t; o.taps = 9; o.stride = stride; o.N = cout;
    if (a.dtype == DT_F32 && act != DT_F32) { o.w = up_f32(wo, (long long)cout * 9 * a.C); o.w_f32 = 1; }
    else o.w = up_mat(wo, (long long)cout * 9 * a.C);
    o.b = up_f32(bo, cout); o.temb_off = temb_off; o.res = res;
    return out_t;
  }

  int resblock(int x0, int x1, int cin, int cout, const std::string& pre, int level, bool out_pad) {
    int tg1 = conv_in_tensor(pre + ".g1", level, cin);
    gn(x0, x1, tg1, pre + ".gn1", 1);
    halo(tg1, 1);
    int th1 = tensor(pre + ".h1", level, cout, act, 0, 0);
    // conv1 + bias + temb (parameter order: conv1.w, conv1.b, temb.w, temb.b)
    const TDesc& a = P.td[tg1];
    long long wo = take(pre + ".conv1.w", {cout, 3, 3, cin});
    long long bo = take(pre + ".conv1.b", {cout});
    long long two = take(pre + ".temb.w", {cout, P.T});
    long long tbo = take(pre + ".temb.b", {cout});
    temb_rows.push_back({two, tbo, cout, P.J});
    int toff = P.J; P.J += cout;
    {
      Op& o = op(OP_CONV); o.in0 = tg1; o.out = th1; o.taps = 9; o.stride = 1; o.N = cout;
      o.w = up_mat(wo, (long long)cout * 9 * a.C); o.b = up_f32(bo, cout); o.temb_off = toff;
    }
    int tg2 = conv_in_tensor(pre + ".g2", level, cout);
    gn(th1, -1, tg2, pre + ".gn2", 1);
    halo(tg2, 1);
    long long w2 = take(pre + ".conv2.w", {cout, 3, 3, cout});
    long long b2 = take(pre + ".conv2.b", {cout});
    int res = x0;
    if (cin != cout) {
      long long sw = take(pre + ".skip.w", {cout, cin});
      long long sb = take(pre + ".skip.b", {cout});
      int ts = tensor(pre + ".skip", level, cout, act, 0, 0);
      Op& o = op(OP_GEMM); o.in0 = x0; o.in1 = x1; o.out = ts; o.taps = 1; o.N = cout;
      o.w = up_mat(sw, (long long)cout * cin); o.b = up_f32(sb, cout);
      res = ts;
    }
    int tout = tensor(pre + ".out", level, cout, act, out_pad ? 1 : 0, out_pad ? 1 : 0);
    Op& o = op(OP_CONV); o.in0 = tg2; o.out = tout; o.taps = 9; o.stride = 1; o.N = cout;
    o.w = up_mat(w2, (long long)cout * 9 * cout); o.b = up_f32(b2, cout); o.res = res;
    return tout;
  }

  int attn_stack(int x, int C, int depth, const std::string& pre, int level, bool out_pad) {
    int tg = tensor(pre + ".gn", level, C, act, 0, 0);
    gn(x, -1, tg, pre + ".gn", 0);
    int th = tensor(pre + ".pin", level, C, act, 0, 0);
    {
      long long w = take(pre + ".proj_in.w", {C, C}); long long b = take(pre + ".proj_in.b", {C});
      Op& o = op(OP_GEMM); o.in0 = tg; o.out = th; o.N = C; o.w = up_mat(w, (long long)C * C); o.b = up_f32(b, C);
    }
    for (int d = 0; d < depth; ++d) {
      std::string a = pre + ".attn" + std::to_string(d);
      int tin = th;                          // the self-attention input: h, or LN1(h) in the _XF models
      if (P.xf) tin = layernorm(th, a + ".ln1", level, C);
      long long wq = take(a + ".wq", {C, C}), wk = take(a + ".wk", {C, C}), wv = take(a + ".wv", {C, C});
      long long wo = take(a + ".wo", {C, C}), bo = take(a + ".bo", {C});
      int tq = tensor(a + ".q", level, C, act, 0, 0);
      int tkv = tensor(a + ".kv", level, 2 * C, act, 0, 1);
      {
        Op& o = op(OP_GEMM); o.in0 = tin; o.out = tq; o.out2 = tkv; o.n_split = C; o.N = 3 * C;
        o.w = up_mat(wq, (long long)C * C); up_mat(wk, (long long)C * C); up_mat(wv, (long long)C * C);
      }
      AttnX ax{}; ax.kv = tkv; ax.level = level; ax.h = rows_at(level); ax.W = w_at(level); ax.C = C;
      ax.r = band_rows(P.p, ax.h);
      P.attns.push_back(ax);
      int aid = (int)P.attns.size() - 1;
      if (P.n > 1) { Op& o = op(OP_KVX); o.in0 = tkv; o.xid = aid; }
      int to = tensor(a + ".o", level, C, act, 0, 0);
      { Op& o = op(OP_ATTN); o.in0 = tq; o.in1 = tkv; o.out = to; o.xid = aid; }
      int th2 = tensor(a + ".h", level, C, act, 0, 0);
      { Op& o = op(OP_GEMM); o.in0 = to; o.out = th2; o.N = C; o.w = up_mat(wo, (long long)C * C); o.b = up_f32(bo, C); o.res = th; }
      th = th2;
      if (P.xf) th = xf_tail(th, a, level, C);
    }
    int tout = tensor(pre + ".out", level, C, act, out_pad ? 1 : 0, out_pad ? 1 : 0);
    long long w = take(pre + ".proj_out.w", {C, C}); long long b = take(pre + ".proj_out.b", {C});
    Op& o = op(OP_GEMM); o.in0 = th; o.out = tout; o.N = C; o.w = up_mat(w, (long long)C * C); o.b = up_f32(b, C); o.res = x;
    return tout;
  }

  // LayerNorm(C) of x into a new tensor (parameters <pre>.g, <pre>.b)
  int layernorm(int x, const std::string& pre, int level, int C) {
    int t = tensor(pre, level, C, act, 0, 0);
    Op& o = op(OP_LN); o.in0 = x; o.out = t;
    o.g = vec(pre + ".g", C); o.be = vec(pre + ".b", C);
    return t;
  }
  // the rest of SDXL's transformer block after the self-attention (reading D25):
  // h += W_xo CA(LN2 h, ctx) + b_xo;  h += W_ff2 (a * gelu(g)) + b_ff2, [a | g] = LN3(h) W_ff1 + b_ff1
  int xf_tail(int th, const std::string& a, int level, int C) {
    int tl2 = layernorm(th, a + ".ln2", level, C);
    long long xq = take(a + ".xq", {C, C});
    long long xk = take(a + ".xk", {C, P.ctx_dim}), xv = take(a + ".xv", {C, P.ctx_dim});
    long long xo = take(a + ".xo", {C, C}), xbo = take(a + ".xbo", {C});
    int tq = tensor(a + ".xq", level, C, act, 0, 0);
    { Op& o = op(OP_GEMM); o.in0 = tl2; o.out = tq; o.N = C; o.w = up_mat(xq, (long long)C * C); }
    XAttnX xa; xa.level = level; xa.C = C;
    xa.w = up_mat(xk, (long long)C * P.ctx_dim); up_mat(xv, (long long)C * P.ctx_dim);   // [W_k; W_v] = [2C][ctx_dim]
    P.xattns.push_back(xa);
    int to = tensor(a + ".xo_in", level, C, act, 0, 0);
    { Op& o = op(OP_XATTN); o.in0 = tq; o.out = to; o.xid = (int)P.xattns.size() - 1; }
    int th2 = tensor(a + ".xh", level, C, act, 0, 0);
    { Op& o = op(OP_GEMM); o.in0 = to; o.out = th2; o.N = C; o.w = up_mat(xo, (long long)C * C); o.b = up_f32(xbo, C); o.res = th; }
    int tl3 = layernorm(th2, a + ".ln3", level, C);
    long long f1 = take(a + ".ff1.w", {8 * C, C}), f1b = take(a + ".ff1.b", {8 * C});
    long long f2 = take(a + ".ff2.w", {C, 4 * C}), f2b = take(a + ".ff2.b", {C});
    // W_ff1 = [W_value (4C rows); W_gate (4C rows)] is uploaded in 64-row blocks [value k | gate k], so a
    // 128-column GEMM tile holds a value column and its gate: the tcgen05 epilogue applies the GEGLU
    // and writes 4C channels; other paths write the 8C blocked product to tu and run the GEGLU kernel
    int tu = tensor(a + ".ff_u", level, 8 * C, act, 0, 0);
    int tg = tensor(a + ".ff_g", level, 4 * C, act, 0, 0);
    {
      Op& o = op(OP_GEMM); o.in0 = tl3; o.out = tg; o.tmp = tu; o.geglu = 1; o.N = 8 * C;
      o.w = P.wmat_len; o.b = P.wf32_len;
      for (int k = 0; k < 4 * C / 64; ++k)
        for (int half = 0; half < 2; ++half) {            // value block k, then gate block k
          const long long row0 = (long long)half * 4 * C + 64LL * k;
          P.uploads.push_back({f1 + row0 * C, 64LL * C, 0, P.wmat_len + (128LL * k + 64 * half) * C});
          P.uploads.push_back({f1b + row0, 64, 1, P.wf32_len + 128LL * k + 64 * half});
        }
      P.wmat_len = (P.wmat_len + 8LL * C * C + 63) & ~63LL;
      P.wf32_len = (P.wf32_len + 8LL * C + 63) & ~63LL;
    }
    int th3 = tensor(a + ".fh", level, C, act, 0, 0);
    { Op& o = op(OP_GEMM); o.in0 = tg; o.out = th3; o.N = C; o.w = up_mat(f2, 4LL * C * C); o.b = up_f32(f2b, C); o.res = th2; }
    return th3;
  }

  struct TembRow { long long w, b; int cout, col; };
  std::vector<TembRow> temb_rows;

  void build(int model) {
    const bool sdxl = model == PCPP_MODEL_SDXL || model == PCPP_MODEL_SDXL_XF;
    P.xf = model == PCPP_MODEL_TINY_XF || model == PCPP_MODEL_SDXL_XF;
    P.ctx_dim = P.xf ? (sdxl ? 2048 : 256) : 0;
    P.levels = sdxl ? 3 : 1; P.C0 = sdxl ? 320 : 128; P.T = 4 * P.C0; P.SIN = P.C0;
    long long w1 = take("time.lin1.w", {P.T, P.SIN}), b1 = take("time.lin1.b", {P.T});
    long long w2 = take("time.lin2.w", {P.T, P.T}), b2 = take("time.lin2.b", {P.T});
    P.t_w1 = up_f32(w1, (long long)P.T * P.SIN); P.t_b1 = up_f32(b1, P.T);
    P.t_w2 = up_f32(w2, (long long)P.T * P.T); P.t_b2 = up_f32(b2, P.T);
    op(OP_TEMB);
    // conv_in (latent stays fp32: reading of the latent precision, SURVEY §8(c) tolerances)
    int xin = tensor("xin", 0, 4, DT_F32, 1, 1);
    { Op& o = op(OP_PREP); o.out = xin; }
    halo(xin, 1);
    int h = tensor("conv_in.out", 0, P.C0, act, 0, 0);
    conv(xin, "conv_in", P.C0, 1, h, -1, -1);
    if (!sdxl) {
      for (int j = 0; j < 2; ++j) {
        h = resblock(h, -1, P.C0, P.C0, "blk" + std::to_string(j) + ".rb", 0, false);
        h = attn_stack(h, P.C0, 1, "blk" + std::to_string(j) + ".as", 0, false);
      }
    } else {
      const int ch[3] = {320, 640, 1280}, dep[3] = {0, 2, 10};
      std::vector<int> skips;
      skips.push_back(h);
      int cin = 320;
      for (int lvl = 0; lvl < 3; ++lvl) {
        for (int j = 0; j < 2; ++j) {
          const bool last_pad = (lvl < 2 && j == 1);
          const std::string pre = "down" + std::to_string(lvl) + "." + std::to_string(j);
          h = resblock(h, -1, cin, ch[lvl], pre + ".rb", lvl, last_pad && !dep[lvl]);
          cin = ch[lvl];
          if (dep[lvl]) h = attn_stack(h, ch[lvl], dep[lvl], pre + ".as", lvl, last_pad);
          skips.push_back(h);
        }
        if (lvl < 2) {
          halo(h, 2);
          int t = tensor("down" + std::to_string(lvl) + ".ds.out", lvl + 1, ch[lvl], act, 0, 0);
          conv(h, "down" + std::to_string(lvl) + ".ds.conv", ch[lvl], 2, t, -1, -1);
          h = t;
          skips.push_back(h);
        }
      }
      h = resblock(h, -1, 1280, 1280, "mid.rb0", 2, false);
      h = attn_stack(h, 1280, 10, "mid.as", 2, false);
      h = resblock(h, -1, 1280, 1280, "mid.rb1", 2, false);
      int cur = 1280;
      for (int lvl = 2; lvl >= 0; --lvl) {
        for (int j = 0; j < 3; ++j) {
          int sk = skips.back(); skips.pop_back();
          const std::string pre = "up" + std::to_string(lvl) + "." + std::to_string(j);
          h = resblock(h, sk, cur + P.td[sk].C, ch[lvl], pre + ".rb", lvl, false);
          cur = ch[lvl];
          if (dep[lvl]) h = attn_stack(h, ch[lvl], dep[lvl], pre + ".as", lvl, false);
        }
        if (lvl > 0) {
          int tu = tensor("up" + std::to_string(lvl) + ".us.in", lvl - 1, ch[lvl], act, 1, 1);
          { Op& o = op(OP_UPS); o.in0 = h; o.out = tu; }
          halo(tu, 1);
          int t = tensor("up" + std::to_string(lvl) + ".us.out", lvl - 1, ch[lvl], act, 0, 0);
          conv(tu, "up" + std::to_string(lvl) + ".us.conv", ch[lvl], 1, t, -1, -1);
          h = t;
        }
      }
    }
    // out: GN -> SiLU -> conv3x3 -> eps (fp32), then CFG + DDIM
    int tg = conv_in_tensor("out.g", 0, P.C0);
    gn(h, -1, tg, "out.gn", 1);
    halo(tg, 1);
    int teps = tensor("eps", 0, 4, DT_F32, 0, 0);
    {
      long long wo = take("conv_out.w", {4, 3, 3, P.C0}), bo = take("conv_out.b", {4});
      Op& o = op(OP_CONVOUT); o.in0 = tg; o.out = teps; o.N = 4;
      o.w = up_f32(wo, 4LL * 9 * P.C0); o.w_f32 = 1; o.b = up_f32(bo, 4);
    }
    if (P.split) {   // CFG device split: both branches' eps of this patch side by side (the partner's by exchange)
      int teps2 = tensor("eps2", 0, 4, DT_F32, 0, 0, 2);
      P.td[teps2].xdst = 1;
      Op& o = op(OP_EPSX); o.in0 = teps; o.out = teps2;
      teps = teps2;
    }
    { Op& o = op(OP_CFGDDIM); o.in0 = teps; }
    op(OP_END);
    // temb projections: one [J][T] matrix (fp32) in ResBlock order
    P.t_wt = P.wf32_len;
    for (auto& tr : temb_rows) { P.uploads.push_back({tr.w, (long long)tr.cout * P.T, 1, P.wf32_len + (long long)tr.col * P.T}); }
    P.wf32_len += (long long)P.J * P.T; P.wf32_len = (P.wf32_len + 63) & ~63LL;
    P.t_bt = P.wf32_len;
    for (auto& tr : temb_rows) { P.uploads.push_back({tr.b, tr.cout, 1, P.wf32_len + tr.col}); }
    P.wf32_len += P.J; P.wf32_len = (P.wf32_len + 63) & ~63LL;
  }
};

}  // namespace

pcpp_status build_program(Plan& P, int model) {
  Builder b(P);
  b.build(model);
  return PCPP_OK;
}

}  // namespace pcpp
