"""Thin ctypes binding of libpcpp (include/pcpp.h).  Argument marshalling only: every step of
the path runs in libpcpp's CUDA kernels.  There is no CPU or PyTorch fallback -- if the library
is missing, loading fails loudly."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpcpp.so")

OK, ERR_INVALID, ERR_STATE, ERR_CUDA, ERR_NCCL, ERR_OOM, ERR_UNSUPPORTED = range(7)
FP32, BF16 = 0, 1
SCHEME_PCPP, SCHEME_FULLMAP, SCHEME_SYNC = 0, 1, 2
MODEL_TINY, MODEL_SDXL, MODEL_TINY_XF, MODEL_SDXL_XF = 0, 1, 2, 3
CTX_LEN = 77
COMM_NCCL, COMM_LOOPBACK, COMM_PEER = 0, 1, 2
BACKENDS = {"nccl": COMM_NCCL, "loopback": COMM_LOOPBACK, "peer": COMM_PEER}
PEER_HANDLE_BYTES = 64
KERNELS_AUTO, KERNELS_SIMT = 0, 1
MAX_LAYERS = 128
MODELS = {"tiny": MODEL_TINY, "sdxl": MODEL_SDXL, "tiny_xf": MODEL_TINY_XF, "sdxl_xf": MODEL_SDXL_XF}
SCHEMES = {"pcpp": SCHEME_PCPP, "fullmap": SCHEME_FULLMAP, "sync": SCHEME_SYNC}


SCHEDULERS = {"ddim": 0, "dpmpp2m": 1, "ancestral": 2}   # PCPP_SCHED_* (include/pcpp.h)


class pcpp_config(C.Structure):
    _fields_ = [("rank", C.c_int), ("world", C.c_int), ("num_steps", C.c_int),
                ("guidance_scale", C.c_float), ("precision", C.c_int), ("scheme", C.c_int),
                ("model", C.c_int), ("weights", C.POINTER(C.c_float)), ("weights_len", C.c_size_t),
                ("nccl_id", C.c_void_p), ("stream", C.c_void_p), ("comm_backend", C.c_int),
                ("kernels", C.c_int), ("use_graphs", C.c_int), ("scheduler", C.c_int),
                ("noise_seed", C.c_ulonglong), ("cfg_split", C.c_int)]


class pcpp_info(C.Structure):
    _fields_ = [("n_conv", C.c_int), ("n_gn", C.c_int), ("n_attn", C.c_int), ("h_latent", C.c_int),
                ("attn_h", C.c_int * MAX_LAYERS), ("attn_r", C.c_int * MAX_LAYERS),
                ("bytes_async", C.c_longlong * 3), ("bytes_warmup", C.c_longlong * 3),
                ("bytes_fullmap", C.c_longlong * 3), ("bytes_counted_async", C.c_longlong * 3),
                ("bytes_counted_warmup", C.c_longlong * 3), ("last_step_ms", C.c_double),
                ("device_bytes", C.c_longlong), ("n_kernels_per_step", C.c_int), ("graphs", C.c_int),
                ("tc_kernels", C.c_int), ("step_flops", C.c_double), ("step_flops_rank_max", C.c_double),
                ("arena_bytes_per_rank", C.c_longlong), ("arena_bytes_unplanned", C.c_longlong),
                ("simt_fallbacks", C.c_int), ("backend", C.c_int), ("comm_lib", C.c_char * 192),
                ("bytes_eps", C.c_longlong)]

    def as_dict(self):
        d = {}
        for name, _ in self._fields_:
            v = getattr(self, name)
            if name in ("attn_h", "attn_r"):
                v = list(v)[: self.n_attn]
            elif name == "comm_lib":
                v = v.decode()
            elif hasattr(v, "__len__"):
                v = list(v)
            d[name] = v
        return d


class pcpp_prof(C.Structure):
    _fields_ = [("ms", C.c_double), ("flops", C.c_double), ("bytes", C.c_double), ("launches", C.c_int)]


SYMBOLS = ["pcpp_plan_schedule", "pcpp_profile", "pcpp_config_default", "pcpp_get_unique_id", "pcpp_weights_len", "pcpp_manifest_count",
           "pcpp_manifest_entry", "pcpp_plan", "pcpp_plan_info", "pcpp_set_cond", "pcpp_step",
           "pcpp_sample", "pcpp_reset", "pcpp_query", "pcpp_debug_comm_off", "pcpp_destroy", "pcpp_last_error",
           "pcpp_op_conv", "pcpp_op_attention", "pcpp_op_groupnorm", "pcpp_op_pack_rows",
           "pcpp_op_cfg_ddim", "pcpp_peer_handle", "pcpp_peer_connect", "pcpp_set_context", "pcpp_debug_gemm_trace"]

_lib = None


def lib():
    """Load libpcpp.so (built in-tree by build.py / __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"libpcpp.so not built ({LIB_PATH}); run python paper_2412_02962_b200/build.py")
    if "PCPP_NCCL_LIB" not in os.environ:        # the NCCL torch ships (used by the NCCL backend only)
        try:
            import nvidia.nccl
            cand = os.path.join(list(nvidia.nccl.__path__)[0], "lib", "libnccl.so.2")
            if os.path.exists(cand):
                os.environ["PCPP_NCCL_LIB"] = cand
        except Exception:
            pass
    L = C.CDLL(LIB_PATH)
    V, P, I, D, S = C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_size_t
    L.pcpp_config_default.argtypes = [C.POINTER(pcpp_config)]; L.pcpp_config_default.restype = None
    L.pcpp_get_unique_id.argtypes = [V]; L.pcpp_get_unique_id.restype = I
    L.pcpp_weights_len.argtypes = [I]; L.pcpp_weights_len.restype = S
    L.pcpp_manifest_count.argtypes = [I]; L.pcpp_manifest_count.restype = I
    L.pcpp_manifest_entry.argtypes = [I, I, C.c_char_p, I, C.POINTER(C.c_longlong)]; L.pcpp_manifest_entry.restype = I
    L.pcpp_plan.argtypes = [I, I, I, I, D, I, C.POINTER(pcpp_config), C.POINTER(P)]; L.pcpp_plan.restype = I
    L.pcpp_plan_info.argtypes = [I, I, I, I, D, I, C.POINTER(pcpp_config), C.POINTER(pcpp_info)]; L.pcpp_plan_info.restype = I
    L.pcpp_set_cond.argtypes = [P, V]; L.pcpp_set_cond.restype = I
    L.pcpp_set_context.argtypes = [P, V]; L.pcpp_set_context.restype = I
    L.pcpp_step.argtypes = [P, V, I]; L.pcpp_step.restype = I
    L.pcpp_sample.argtypes = [P, V, V, V]; L.pcpp_sample.restype = I
    L.pcpp_reset.argtypes = [P]; L.pcpp_reset.restype = I
    L.pcpp_query.argtypes = [P, C.POINTER(pcpp_info)]; L.pcpp_query.restype = I
    L.pcpp_destroy.argtypes = [P]; L.pcpp_destroy.restype = None
    L.pcpp_plan_schedule.argtypes = [I, I, I, I, D, I, C.POINTER(pcpp_config), I, C.POINTER(C.c_int), I]
    L.pcpp_plan_schedule.restype = I
    L.pcpp_profile.argtypes = [P, V, I, I, I, C.POINTER(pcpp_prof)]; L.pcpp_profile.restype = I
    L.pcpp_debug_comm_off.argtypes = [P, I]; L.pcpp_debug_comm_off.restype = I
    L.pcpp_debug_gemm_trace.argtypes = [P]; L.pcpp_debug_gemm_trace.restype = I
    L.pcpp_last_error.argtypes = []; L.pcpp_last_error.restype = C.c_char_p
    L.pcpp_op_conv.argtypes = [V, I, I, I, I, I, I, V, V, V, V, V, I, I, I, V]; L.pcpp_op_conv.restype = I
    L.pcpp_op_attention.argtypes = [V, C.POINTER(C.c_void_p), C.POINTER(C.c_int), I, I, I, I, I, V, I, I, V]
    L.pcpp_op_attention.restype = I
    L.pcpp_op_groupnorm.argtypes = [V, I, I, I, I, V, V, I, V, V, I, V]; L.pcpp_op_groupnorm.restype = I
    L.pcpp_op_pack_rows.argtypes = [V, C.c_longlong, I, I, V, V]; L.pcpp_op_pack_rows.restype = I
    L.pcpp_op_cfg_ddim.argtypes = [V, V, I, I, C.c_float, I, I, V]; L.pcpp_op_cfg_ddim.restype = I
    L.pcpp_peer_handle.argtypes = [P, V]; L.pcpp_peer_handle.restype = I
    L.pcpp_peer_connect.argtypes = [P, V]; L.pcpp_peer_connect.restype = I
    _lib = L
    return L


class PcppError(RuntimeError):
    def __init__(self, status, where):
        msg = lib().pcpp_last_error()
        super().__init__(f"{where} -> status {status}: {msg.decode() if msg else ''}")
        self.status = status


def _chk(st, where):
    if st != OK:
        raise PcppError(st, where)


def _ptr(x):
    """Device or host address of a torch tensor / numpy array / int."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return x.data_ptr()


# ---- manifest -----------------------------------------------------------------------------------
def pcpp_weights_len(model: str) -> int:
    return int(lib().pcpp_weights_len(MODELS[model]))


def manifest(model: str):
    """[(name, shape)] in blob order, as libpcpp's own builder defines it."""
    L = lib()
    m = MODELS[model]
    out = []
    buf = C.create_string_buffer(256)
    shape = (C.c_longlong * 4)()
    for i in range(L.pcpp_manifest_count(m)):
        nd = L.pcpp_manifest_entry(m, i, buf, 256, shape)
        out.append((buf.value.decode(), tuple(int(shape[d]) for d in range(nd))))
    return out


def pcpp_get_unique_id() -> bytes:
    b = C.create_string_buffer(128)
    _chk(lib().pcpp_get_unique_id(b), "pcpp_get_unique_id")
    return b.raw


def make_config(model="sdxl", num_steps=50, guidance=5.0, precision="bf16", scheme="pcpp",
                backend="loopback", rank=0, world=1, weights=None, nccl_id=None, stream=None,
                kernels="auto", graphs=True, scheduler="ddim", noise_seed=0, cfg_split=False):
    cfg = pcpp_config()
    lib().pcpp_config_default(C.byref(cfg))
    cfg.model = MODELS[model]
    cfg.num_steps = num_steps
    cfg.guidance_scale = guidance
    cfg.precision = BF16 if precision == "bf16" else FP32
    cfg.scheme = SCHEMES[scheme]
    cfg.comm_backend = BACKENDS[backend]
    cfg.rank, cfg.world = rank, world
    cfg.kernels = KERNELS_AUTO if kernels == "auto" else KERNELS_SIMT
    cfg.use_graphs = 1 if graphs else 0
    cfg.scheduler = SCHEDULERS[scheduler]
    cfg.noise_seed = noise_seed
    cfg.cfg_split = 1 if cfg_split else 0
    if weights is not None:
        cfg.weights = weights.ctypes.data_as(C.POINTER(C.c_float))
        cfg.weights_len = weights.size
    if nccl_id is not None:
        cfg._id_buf = C.create_string_buffer(nccl_id, 128)
        cfg.nccl_id = C.cast(cfg._id_buf, C.c_void_p)
    cfg.stream = stream
    return cfg


def pcpp_plan_schedule(H, W, Cl, n, p, warmup, cfg, sync: int):
    """This rank's NCCL issue schedule for one step: [(op, peer, bytes, cls, group)]."""
    L = lib()
    cnt = L.pcpp_plan_schedule(H, W, Cl, n, float(p), warmup, C.byref(cfg), int(sync), None, 0)
    if cnt < 0:
        raise PcppError(ERR_INVALID, "pcpp_plan_schedule")
    buf = (C.c_int * (5 * max(cnt, 1)))()
    L.pcpp_plan_schedule(H, W, Cl, n, float(p), warmup, C.byref(cfg), int(sync), buf, cnt)
    return [tuple(buf[5 * i:5 * i + 5]) for i in range(cnt)]


def pcpp_plan_info(H, W, Cl, n, p, warmup, cfg) -> dict:
    info = pcpp_info()
    _chk(lib().pcpp_plan_info(H, W, Cl, n, float(p), warmup, C.byref(cfg), C.byref(info)), "pcpp_plan_info")
    return info.as_dict()


class Plan:
    """Owns one pcpp_plan_t.  Methods mirror the C calls (pcpp_step, pcpp_sample, ...)."""

    def __init__(self, H, W, Cl, n, p, warmup, cfg, weights):
        self._w = np.ascontiguousarray(weights, dtype=np.float32)   # keep alive during pcpp_plan
        cfg.weights = self._w.ctypes.data_as(C.POINTER(C.c_float))
        cfg.weights_len = self._w.size
        self.cfg = cfg
        self.H, self.W, self.n = H, W, n
        self.h = C.c_void_p()
        _chk(lib().pcpp_plan(H, W, Cl, n, float(p), warmup, C.byref(cfg), C.byref(self.h)), "pcpp_plan")
        self._w = None

    def pcpp_set_cond(self, cond: np.ndarray):
        c = np.ascontiguousarray(cond, dtype=np.float32)
        _chk(lib().pcpp_set_cond(self.h, c.ctypes.data), "pcpp_set_cond")

    def pcpp_set_context(self, ctx: np.ndarray):
        """_xf models: the cross-attention context [2, 77, ctx_dim] (b = 0 uncond, 1 cond)."""
        c = np.ascontiguousarray(ctx, dtype=np.float32)
        _chk(lib().pcpp_set_context(self.h, c.ctypes.data), "pcpp_set_context")

    def pcpp_step(self, latent, t: int):
        _chk(lib().pcpp_step(self.h, _ptr(latent), int(t)), "pcpp_step")

    def pcpp_sample(self, xT: np.ndarray, cond: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(xT, dtype=np.float32)
        c = np.ascontiguousarray(cond, dtype=np.float32)
        out = np.empty((self.H, self.W, 4), dtype=np.float32)
        _chk(lib().pcpp_sample(self.h, x.ctypes.data, c.ctypes.data, out.ctypes.data), "pcpp_sample")
        return out

    def pcpp_sample_into(self, xT_ptr: int, cond_ptr: int, out_ptr: int):
        """Host pointers (e.g. pinned torch tensors)."""
        _chk(lib().pcpp_sample(self.h, xT_ptr, cond_ptr, out_ptr), "pcpp_sample")

    def pcpp_peer_handle(self) -> bytes:
        """PEER backend: this rank's 64-byte CUDA IPC handle of its arena."""
        b = C.create_string_buffer(PEER_HANDLE_BYTES)
        _chk(lib().pcpp_peer_handle(self.h, b), "pcpp_peer_handle")
        return b.raw

    def pcpp_peer_connect(self, handles: list[bytes]):
        """PEER backend: open every rank's arena (handles in rank order)."""
        buf = C.create_string_buffer(b"".join(handles), PEER_HANDLE_BYTES * len(handles))
        _chk(lib().pcpp_peer_connect(self.h, buf), "pcpp_peer_connect")

    def pcpp_reset(self):
        _chk(lib().pcpp_reset(self.h), "pcpp_reset")

    def pcpp_query(self) -> dict:
        info = pcpp_info()
        _chk(lib().pcpp_query(self.h, C.byref(info)), "pcpp_query")
        return info.as_dict()

    def pcpp_profile(self, latent, kind_mask: int, sync: int = 0, iters: int = 5) -> dict:
        """Device ms per step of the ops in kind_mask (1 GEMM/conv, 2 attention, 4 GN, 8 exchange,
        16 other), measured in isolation, plus their algorithmic flops/bytes."""
        pr = pcpp_prof()
        _chk(lib().pcpp_profile(self.h, _ptr(latent), kind_mask, sync, iters, C.byref(pr)), "pcpp_profile")
        return dict(ms=pr.ms, flops=pr.flops, bytes=pr.bytes, launches=pr.launches)

    def pcpp_debug_comm_off(self, on: bool = True):
        """COMM_OFF timing mode: asynchronous steps skip their exchanges (results not the method's)."""
        _chk(lib().pcpp_debug_comm_off(self.h, 1 if on else 0), "pcpp_debug_comm_off")

    def close(self):
        if self.h:
            lib().pcpp_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- kernel-level entry points ---------------------------------------------------------------------
def _dt(t):
    import torch
    return FP32 if t.dtype == torch.float32 else BF16


def pcpp_op_conv(x, rows_in, B, W_in, Cin, taps, stride, w, bias, temb, res, y, Cout, impl="auto", stream=None):
    _chk(lib().pcpp_op_conv(_ptr(x), rows_in, B, W_in, Cin, taps, stride, _ptr(w), _ptr(bias), _ptr(temb),
                            _ptr(res), _ptr(y), Cout, _dt(x), KERNELS_AUTO if impl == "auto" else KERNELS_SIMT,
                            stream), "pcpp_op_conv")


def pcpp_op_attention(q, kvs, kv_rows, h, B, W, Cm, out, impl="auto", stream=None):
    arr = (C.c_void_p * len(kvs))(*[_ptr(k) for k in kvs])
    rows = (C.c_int * len(kvs))(*kv_rows)
    _chk(lib().pcpp_op_attention(_ptr(q), arr, rows, len(kvs), h, B, W, Cm, _ptr(out), _dt(q),
                                 KERNELS_AUTO if impl == "auto" else KERNELS_SIMT, stream), "pcpp_op_attention")


def pcpp_op_groupnorm(x, rows, B, W, Cm, gamma, beta, silu, y, m_out, stream=None):
    _chk(lib().pcpp_op_groupnorm(_ptr(x), rows, B, W, Cm, _ptr(gamma), _ptr(beta), int(silu), _ptr(y),
                                 _ptr(m_out), _dt(x), stream), "pcpp_op_groupnorm")


def pcpp_op_pack_rows(src, row_bytes, r0, nrows, dst, stream=None):
    _chk(lib().pcpp_op_pack_rows(_ptr(src), row_bytes, r0, nrows, _ptr(dst), stream), "pcpp_op_pack_rows")


def pcpp_op_cfg_ddim(eps, latent, h, W, guidance, num_steps, k, stream=None):
    _chk(lib().pcpp_op_cfg_ddim(_ptr(eps), _ptr(latent), h, W, float(guidance), num_steps, k, stream),
         "pcpp_op_cfg_ddim")


def pcpp_debug_gemm_trace():
    """GEMM timeline ring (PCPP_GEMM_TRACE=1): returns (launches recorded, uint64 array [32][148][8])."""
    import numpy as np
    buf = np.zeros(32 * 148 * 8, dtype=np.uint64)
    n = lib().pcpp_debug_gemm_trace(buf.ctypes.data)
    return n, buf.reshape(32, 148, 8)
