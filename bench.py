#!/usr/bin/env python
"""bench.py -- PCPP denoising-step latency on B200 (SDXL-shaped 1024^2, CFG batch 2, 50-step DDIM).

  python bench.py [--gpus N --steps K --warmup W]             # libpcpp arm (one process per GPU)
  python bench.py --impl reference [--gpus N ...]              # the fp64 CPU oracle arm

Metric (BASELINE.json): per-step latency (and, across N, speed-up) of the PCPP denoising step plus
bytes exchanged per step.  One "step" = one UNet forward over both CFG branches on this rank's
patch + the neighbour exchanges + CFG + DDIM (pcpp_step).  N = 1 is the single-device baseline
(one patch); N > 1 splits the latent into N patches (p = 0.3 at 2, 0.8 at 4 and 8: the paper's
Fig. 4 settings), warm-up 4, exchanges by one-sided peer stores (PEER backend; NCCL
with --backend nccl).  Timed steps are post-warm-up (async) steps.  Device time: CUDA events around
K pcpp_step calls, max over ranks.  The per-step working set (1.57 GB of bf16 weights +
activations) exceeds the 126 MB L2, so no explicit flush is needed.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

P_BY_N = {1: 0.0, 2: 0.3, 4: 0.8, 8: 0.8}
METRIC = "PCPP denoising step latency (SDXL-shaped UNet, 1024x1024 / 128x128x4 latent, CFG batch 2)"
T_START = time.time()


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="pcpp", choices=["pcpp", "reference"])
    ap.add_argument("--res", type=int, default=128, help="latent H = W (128 -> 1024^2 image)")
    ap.add_argument("--scheme", default="pcpp", choices=["pcpp", "fullmap", "sync"])
    ap.add_argument("--p", type=float, default=None)
    ap.add_argument("--backend", default="peer", choices=["peer", "nccl"],
                    help="N > 1 exchange transport: one-sided peer stores (default) or NCCL send/recv")
    ap.add_argument("--e2e-samples", type=int, default=5)
    ap.add_argument("--cfg-split", action="store_true",
                    help="the paper's CFG device split (P:24): N GPUs = 2 branch groups x N/2 patches")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--no-comm-off", action="store_true", help="N > 1: skip the COMM_OFF re-timing")
    ap.add_argument("--no-loopback", action="store_true", help="skip the n = 2/4/8 loopback projections (N = 1)")
    ap.add_argument("--no-large", action="store_true", help="skip the 2048^2 / 3840^2 lines (N = 1)")
    ap.add_argument("--no-xf", action="store_true", help="skip the SDXL-transformer-block (sdxl_xf) line (N = 1)")
    ap.add_argument("--kernels", default="auto", choices=["auto", "simt"])
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class Clocks:
    """nvidia-smi sampling during the timed region (clock + throttle reasons)."""

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = sorted(float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit())
        mx = max((float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------------------------
# the oracle (reference / cpu_baseline) -- imports only oracle/ and the seeded generators
# ---------------------------------------------------------------------------------------------
def _host_info():
    """Host threads / CPU model / BLAS of the oracle timing."""
    cpu = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                cpu = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    threads, blas = os.cpu_count(), "unknown"
    try:
        from threadpoolctl import threadpool_info
        infos = [i for i in threadpool_info() if i.get("user_api") == "blas"]
        if infos:
            threads = max(i.get("num_threads", 0) for i in infos)
            blas = f"{infos[0].get('internal_api')} {infos[0].get('version')}"
    except Exception:
        pass
    return threads, cpu, blas


def oracle_step_times(n, p, S, w, res, steps):
    """Wall time of `steps` full fp64 oracle PCPP steps (k = 0 .. steps-1; the first w synchronous) of
    the SDXL-shaped stack at the bench's own res x res latent, n ranks simulated in one process."""
    from oracle import model as M
    from oracle import pcpp as OP
    from paper_2412_02962_b200 import inputs
    blob = inputs.make_weight_blob(M.weight_specs("sdxl"))
    xT = inputs.make_latent(res, res)
    c = inputs.make_cond(M.arch("sdxl")["temb"])
    cfg = OP.Config(model="sdxl", H=res, W=res, n=n, p=p, warmup=w, steps=S)
    times = []
    t_prev = [time.perf_counter()]

    def tick(_k):
        t = time.perf_counter()
        times.append(t - t_prev[0])
        t_prev[0] = t
    OP.sample(cfg, blob, xT, c, max_steps=steps, record=False, on_step=tick)
    return times


def run_reference(args):
    """The oracle arm: the fp64 CPU oracle, as it stands, on the host cores at the bench's own
    workload.  A full 128^2 oracle step takes about a minute, so the arm's K "steps" are a bounded
    sample: ceil(K / 10) full steps, reported as the mean ms per full step (no extrapolation)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    n = args.gpus
    p = P_BY_N.get(n, 0.8) if args.p is None else args.p
    w = 4 if n > 1 else 0
    S = 50
    m = max(1, -(-args.steps // 10))
    times = oracle_step_times(n, p, S, w, args.res, m)
    ms = 1000.0 * sum(times) / len(times)
    cores, cpu, blas = _host_info()
    sample = (f"{len(times)} full fp64 oracle PCPP step(s) (UNet forward over both CFG branches, n={n} simulated "
              f"ranks, CFG + DDIM) of the SDXL-shaped stack measured at the {args.res}x{args.res} latent itself "
              f"(no extrapolation); per-step s: {[round(t, 2) for t in times]}")
    out = {"impl": "reference", "metric": METRIC, "value": ms, "unit": "ms/step", "n_gpus": n,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"sdxl-{args.res * 8} ({args.res}x{args.res}x4 latent)", "n_patches": n,
                      "cond_fraction": p, "warmup_steps": w, "num_steps": S},
           "cpu_baseline": {"value": ms, "unit": "ms/step", "cores": cores, "kind": "oracle", "sample": sample,
                            "cpu_model": cpu, "blas": blas},
           "e2e": {"value": ms, "unit": "ms/step", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


def _progress(msg):
    """Phase marker on stderr (the JSON line stays the only stdout line)."""
    if os.environ.get("PCPP_BENCH_QUIET") is None:
        print(f"[bench {time.strftime('%H:%M:%S')} +{time.time() - T_START:.0f}s] {msg}", file=sys.stderr, flush=True)


TUNE_FILE = os.path.join(ROOT, "profiles", "gemm_tune_b200.txt")
DIST_DEV = "cuda"          # device of the small tensors of the process-group collectives (cpu under gloo)


def _comm_off_timing(plan, lat, pre, steps, ms, dist, torch):
    """COMM_OFF re-timing at N > 1: the same async steps with every exchange skipped
    (pcpp_debug_comm_off); step - COMM_OFF step = the communication the overlap did not hide.
    Every rank takes the same branch: a local failure is all-reduced before any rank returns, and the
    plan always leaves COMM_OFF mode (finally) before anything else is measured."""
    err, ms_off = None, 0.0
    try:
        plan.pcpp_debug_comm_off(True)
        plan.pcpp_reset()
        for k in range(pre):
            plan.pcpp_step(lat, k)
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for k in range(pre, pre + steps):
            plan.pcpp_step(lat, k)
        ev1.record()
        torch.cuda.synchronize()
        ms_off = ev0.elapsed_time(ev1) / steps
    except Exception as e:  # the headline line must survive a failure of this diagnostic
        err = repr(e)[:200]
    finally:
        try:
            plan.pcpp_debug_comm_off(False)
        except Exception as e:
            err = err or repr(e)[:200]
    t = torch.tensor([ms_off, 1.0 if err else 0.0], dtype=torch.float64, device=DIST_DEV)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)        # outside the try: every rank gets here
    if t[1].item() > 0:
        return {"error": err or "failed on another rank"}
    ms_off = float(t[0].item())
    _progress("COMM_OFF steps done")
    return {"ms_per_step": round(ms_off, 4), "exposed_comm_ms": round(ms - ms_off, 4),
            "note": "pcpp_debug_comm_off: async steps without their exchanges (max over ranks)"}


def time_steps(plan, lat, first, count, torch):
    """Device ms per step of pcpp_step k = first .. first+count-1 (CUDA events on the current stream,
    which pcpp_step orders its work against)."""
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(first, first + count):
        plan.pcpp_step(lat, k)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / count


def loopback_line(pcpp, torch, np, inputs, res, nv, pv, scheme, S, cond, kernels, blob, comm_off=True, split=False):
    """All virtual ranks of an n-patch plan back to back on this GPU (LOOPBACK: exchanges are device
    copies of exactly the bytes the transports move); ms/step of all ranks / ranks = the mean per-rank
    step -- a projection of one rank on its own GPU, not a multi-GPU measurement.  split: the CFG
    device split, 2 x n ranks of batch 1."""
    wv = 4 if nv > 1 else 0
    ranks = 2 * nv if split else nv
    cfg = pcpp.make_config(model="sdxl", num_steps=S, precision="bf16", scheme=scheme, backend="loopback",
                           kernels=kernels, cfg_split=split)
    pl = pcpp.Plan(res, res, 4, nv, pv, wv, cfg, blob)
    pl.pcpp_set_cond(cond)
    lat = torch.from_numpy(np.ascontiguousarray(inputs.make_latent(res, res))).cuda()
    pl.pcpp_reset()
    for k in range(wv + 2):
        pl.pcpp_step(lat, k)
    t = time_steps(pl, lat, wv + 2, 5, torch)
    info = pl.pcpp_query()                    # launches of an async step (before any COMM_OFF re-timing)
    t_off = None
    if comm_off and nv > 1 and scheme == "pcpp":        # the same steps with the exchange copies skipped
        pl.pcpp_debug_comm_off(True)
        pl.pcpp_reset()
        for k in range(wv + 2):
            pl.pcpp_step(lat, k)
        t_off = round(time_steps(pl, lat, wv + 2, 5, torch), 4)
        pl.pcpp_debug_comm_off(False)
    pl.close()
    return {"scheme": scheme + ("+cfg_split" if split else ""), "n_patches": nv, "gpus": ranks, "p": pv,
            "ms_per_step_all_ranks": round(t, 4), "ms_per_rank": round(t / ranks, 4),
            "ms_per_step_all_ranks_comm_off": t_off, "step_flops_rank_max": info["step_flops_rank_max"],
            "launches_per_step_all_ranks": info["n_kernels_per_step"],
            "bytes_exchanged_per_step": sum(info["bytes_counted_async"]) + info["bytes_eps"],
            "bytes_by_class": dict(zip(("attn", "conv", "gn", "eps"), info["bytes_counted_async"] + [info["bytes_eps"]]))}


def main():
    # GEMM configurations: the committed per-shape table (deterministic across runs and identical
    # under ncu); shapes it lacks are tuned at plan time
    if os.path.exists(TUNE_FILE):
        os.environ.setdefault("PCPP_TUNE_FILE", TUNE_FILE)
    import faulthandler
    # a wedged run dumps every thread's stack and exits instead of hanging the caller
    faulthandler.dump_traceback_later(int(os.environ.get("PCPP_BENCH_WATCHDOG_S", "1500")), exit=True)
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch
    from paper_2412_02962_b200 import inputs, pcpp

    rank, world, local = dist_env()
    N = args.gpus
    if world > 1 and world != N:
        raise SystemExit(f"WORLD_SIZE={world} but --gpus {N}")
    if world == 1 and N > 1:
        raise SystemExit("--gpus N > 1 must be launched with torchrun (one process per GPU)")
    # PCPP_BENCH_ONE_GPU=1 (test mode): every rank on cuda:0 with a gloo process group -- exercises the
    # N > 1 code path (PEER exchanges between processes, COMM_OFF, profiles, e2e) on a one-GPU box;
    # its timings are of ranks sharing one GPU and mean nothing
    one_gpu = os.environ.get("PCPP_BENCH_ONE_GPU") == "1"
    dev = "cpu" if one_gpu else "cuda"
    globals()["DIST_DEV"] = dev
    torch.cuda.set_device(0 if one_gpu else local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    split = args.cfg_split and N > 1
    if split and N % 2:
        raise SystemExit("--cfg-split needs an even number of GPUs")
    n = N // 2 if split else N          # patches (per branch group with the split)
    p = P_BY_N.get(n, 0.8) if args.p is None else args.p
    w = 4 if n > 1 else 0
    H = W = args.res
    h = H // n
    patch_id = rank % n
    pre = max(args.warmup, w)
    S = max(50, pre + args.steps)

    blob = inputs.make_weight_blob(inputs.init_specs(pcpp.manifest("sdxl")))
    cond = inputs.make_cond(1280)
    xT = inputs.make_latent(H, W)

    def make_plan(backend):
        nccl_id = None
        if backend == "nccl":
            idt = torch.zeros(128, dtype=torch.uint8, device=DIST_DEV)
            if rank == 0:
                idt.copy_(torch.frombuffer(bytearray(pcpp.pcpp_get_unique_id()), dtype=torch.uint8))
            dist.broadcast(idt, 0)
            nccl_id = bytes(idt.cpu().numpy().tobytes())
        cfg = pcpp.make_config(model="sdxl", num_steps=S, precision="bf16", scheme=args.scheme, backend=backend,
                               rank=rank, world=max(world, 1), nccl_id=nccl_id, kernels=args.kernels, cfg_split=split)
        pl = pcpp.Plan(H, W, 4, n, p, w, cfg, blob)
        if backend == "peer":
            handles = [None] * world
            dist.all_gather_object(handles, pl.pcpp_peer_handle())
            pl.pcpp_peer_connect(handles)
        return pl

    backend = args.backend if world > 1 else "loopback"
    plan, backend_note, ok = None, None, 1.0
    try:
        plan = make_plan(backend)
    except Exception as e:        # e.g. CUDA IPC unavailable: every rank switches to NCCL together
        backend_note, ok = f"{backend} backend failed ({repr(e)[:160]})", 0.0
    if world > 1:
        t = torch.tensor([ok], device=DIST_DEV)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        ok = float(t.item())
    if ok < 1.0:
        if world == 1 or backend == "nccl":
            raise SystemExit(backend_note or "plan creation failed")
        if plan is not None:
            plan.close()
        backend = "nccl"
        backend_note = (backend_note or "peer backend failed on another rank") + "; fell back to nccl"
        plan = make_plan(backend)
    _progress(f"plan built ({backend}; weights uploaded, GEMMs autotuned, graphs pending)")
    plan.pcpp_set_cond(cond)
    patch = xT[patch_id * h:(patch_id + 1) * h] if world > 1 else xT
    lat = torch.from_numpy(np.ascontiguousarray(patch)).cuda()

    def barrier():
        if dist is not None:
            dist.barrier()

    # warm-up: the first w steps are the synchronous warm-up of the method, plus W untimed
    plan.pcpp_reset()
    for k in range(pre):
        plan.pcpp_step(lat, k)
    torch.cuda.synchronize()
    _progress("warm-up steps done")
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        ev0.record()
        for k in range(pre, pre + args.steps):
            plan.pcpp_step(lat, k)
        ev1.record()
        torch.cuda.synchronize()
    barrier()
    _progress("timed steps done")
    ms = ev0.elapsed_time(ev1) / args.steps
    if dist is not None:
        t = torch.tensor([ms], device=DIST_DEV)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    info = plan.pcpp_query()
    if args.kernels == "auto" and info["simt_fallbacks"]:
        raise SystemExit(f"{info['simt_fallbacks']} launches per step fell back to SIMT kernels")

    # COMM_OFF: the same async steps with every exchange skipped; the difference is
    # the communication the overlap failed to hide behind the compute
    comm_off = None
    if world > 1 and not args.no_comm_off:
        comm_off = _comm_off_timing(plan, lat, pre, args.steps, ms, dist, torch)

    # per-kind breakdown of one async step, each kind captured alone (pcpp_profile; collective for
    # the PEER backend -- every rank runs the same sequence)
    prof = {}
    if os.environ.get("PCPP_OP_TIMING") and world == 1:       # per-op device-time table on stderr
        plan.pcpp_profile(lat, 31, 0, 1)
    if not args.no_profile:
        for name, mask in (("conv_gemm", 1), ("attention", 2), ("groupnorm", 4), ("exchange", 8), ("other", 16)):
            prof[name] = plan.pcpp_profile(lat, mask, 0, 5)
    peaks = measured_peaks()
    roof = roof_attn = roof_gn = None
    if prof:
        g = prof["conv_gemm"]
        peak = peaks.get("bf16_tflops", 1590.0)
        ach = g["flops"] / (g["ms"] * 1e-3) / 1e12
        traffic, tsrc = None, None
        tfile = next((f for f in (os.path.join(ROOT, "profiles", f"r{r}_gemm_traffic_step.json") for r in (2, 1))
                      if os.path.exists(f)), "")
        if tfile and args.res == 128 and world == 1 and args.scheme == "pcpp":
            tj = json.load(open(tfile))
            traffic, tsrc = tj["gemm_dram_bytes_per_launch"], tj["source"]
        roof = {"kernel": "gemm_tc_kernel / gemm_tc2_kernel (implicit-GEMM conv3x3 / 1x1, tcgen05)",
                "bound": "tensor", "achieved": round(ach, 1), "peak": peak, "unit": "TFLOP/s",
                "frac": round(ach / peak, 4), "traffic": traffic, "traffic_unit": "bytes/launch (DRAM read+write)",
                "traffic_source": tsrc,
                "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst; kernel timed alone)" if peaks else "fallback",
                "per_launch_flops": g["flops"] / max(g["launches"], 1),
                "avg_launch_ms": g["ms"] / max(g["launches"], 1)}
        # the attention is bound by exp2 on the MUFU (16/clk/SM measured, tools/ubench/mufu.cu ->
        # 4.63e12/s at 1965 MHz), one exp2 per score = flops / (4 * 64)
        a = prof["attention"]
        if a["launches"]:
            ex = a["flops"] / 256.0 / (a["ms"] * 1e-3)
            roof_attn = {"kernel": "attn_tc_kernel (partially conditioned flash attention, tcgen05)", "bound": "alu",
                         "what": "exp2 on the MUFU (d = 64: 2 exp-bound clk per 1 tensor clk)",
                         "achieved": round(ex / 1e12, 3), "peak": 4.63, "unit": "Texp2/s",
                         "frac": round(ex / 4.63e12, 4), "tensor_tflops": round(a["flops"] / (a["ms"] * 1e-3) / 1e12, 1),
                         "peak_source": "measured 16 ex2/clk/SM x 148 SMs x 1.965 GHz (profiles/r1_ubench.txt)"}
        gn = prof["groupnorm"]
        if gn["launches"]:
            hbm = peaks.get("hbm_gbs", 6551.7)
            gbs = gn["bytes"] / (gn["ms"] * 1e-3) / 1e9
            roof_gn = {"kernel": "gn_stats / gn_finalize / gn_apply_wide (GroupNorm, fresh local + stale global)",
                       "bound": "hbm", "achieved": round(gbs, 1), "peak": hbm, "unit": "GB/s", "frac": round(gbs / hbm, 4),
                       "algorithmic_bytes_per_step": gn["bytes"],
                       "bytes_rule": "stats read of x (unless fused into the producer GEMM) + apply read x + write y",
                       "peak_source": "MEASURED_PEAKS.json hbm_gbs"}

    # end to end through the public API: pcpp_sample with pinned host buffers (x_T in, x_0 out)
    e2e = None
    if not args.no_e2e:
        xT_h = torch.from_numpy(np.ascontiguousarray(patch)).pin_memory()
        c_h = torch.from_numpy(cond).pin_memory()
        x0_h = torch.empty((H, W, 4), dtype=torch.float32).pin_memory()
        plan.pcpp_sample_into(xT_h.data_ptr(), c_h.data_ptr(), x0_h.data_ptr())     # warm (graphs exist)
        dts = []
        for _ in range(max(1, args.e2e_samples)):       # mean over samples after warm-up
            barrier()
            t0 = time.perf_counter()
            plan.pcpp_sample_into(xT_h.data_ptr(), c_h.data_ptr(), x0_h.data_ptr())
            dts.append(time.perf_counter() - t0)
        dt = sum(dts) / len(dts)
        if dist is not None:
            t = torch.tensor([dt], device=DIST_DEV)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        e2e = {"value": dt * 1000.0 / S, "unit": "ms/step", "sample_ms": dt * 1000.0, "num_steps": S,
               "samples": len(dts), "sample_ms_each": [round(x * 1000.0, 2) for x in dts],
               "h2d_bytes_per_step": (xT_h.numel() * 4 + c_h.numel() * 4) / S,
               "d2h_bytes_per_step": x0_h.numel() * 4 / S,
               "note": "pcpp_sample (public API): x_T/cond H2D once, S steps (4 warm-up for n > 1), x_0 gathered + "
                       "D2H once; per-step = mean sample time / S over `samples` samples after one warm sample"}
        _progress("e2e samples done")
    plan.close()
    del blob

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        _progress("timing the fp64 oracle (one full step at the bench latent)")
        times = oracle_step_times(n, p, S, w, H, 1)
        cores, cpu_model, blas = _host_info()
        cpu = {"value": 1000.0 * times[0], "unit": "ms/step", "cores": cores, "kind": "oracle",
               "sample": f"one full fp64 oracle PCPP step (both CFG branches, CFG + DDIM) of the SDXL-shaped "
                         f"stack, measured at the {H}x{W} latent itself ({times[0]:.1f} s; no extrapolation)",
               "cpu_model": cpu_model, "blas": blas}

    # single-GPU projections (LOOPBACK, N = 1 only): the n-patch PCPP / FULLMAP steps at 1024^2, the
    # conditioning-fraction sweep (config SW), and the 2048^2 / 3840^2 workloads (configs X2 / X3)
    loop, sweep, large = None, None, None
    if rank == 0 and world == 1 and args.scheme == "pcpp" and args.res == 128:
        blob2 = inputs.make_weight_blob(inputs.init_specs(pcpp.manifest("sdxl")))
        if not args.no_loopback:
            loop = {}
            for nv, sch in ((2, "pcpp"), (4, "pcpp"), (8, "pcpp"), (8, "fullmap")):
                r = loopback_line(pcpp, torch, np, inputs, H, nv, P_BY_N[nv], sch, S, cond, args.kernels, blob2)
                r["projected_speedup_vs_n1"] = round(ms / r["ms_per_rank"], 2)
                loop[f"n{nv}" + ("" if sch == "pcpp" else "_fullmap")] = r
            for gpus in (2, 4, 8):          # the paper's deployment: CFG split, gpus / 2 patches per branch
                nv = gpus // 2
                r = loopback_line(pcpp, torch, np, inputs, H, nv, P_BY_N.get(nv, 0.0), "pcpp", S, cond, args.kernels,
                                  blob2, comm_off=False, split=True)
                r["projected_speedup_vs_n1"] = round(ms / r["ms_per_rank"], 2)
                loop[f"gpus{gpus}_cfg_split"] = r
            loop["note"] = ("loopback: the n virtual ranks run sequentially on one GPU, exchanges are device copies; "
                            "ms_per_rank = all-rank time / n (a projection of one rank on its own GPU, not measured); "
                            "n8_fullmap = the DistriFusion-style full-map exchange (P:86) on the same kernels")
            _progress("1024^2 loopback projections done")
            sweep = {}
            for pv in (0.0, 0.125, 0.25, 0.5, 1.0):       # config SW: p sweep at 1024^2, n = 8
                r = loopback_line(pcpp, torch, np, inputs, H, 8, pv, "pcpp", S, cond, args.kernels, blob2, comm_off=False)
                sweep[str(pv)] = {k: r[k] for k in ("ms_per_rank", "ms_per_step_all_ranks", "bytes_exchanged_per_step",
                                                   "bytes_by_class")}
            sweep["note"] = "config SW (n = 8 at 1024^2, loopback projection); error vs oracle: tests/test_gpu_golden.py"
            _progress("SW sweep done")
        if not args.no_large:
            large = {}
            for res, nvs in ((256, (1, 4, 8)), (480, (1, 8))):     # configs X2 / X3
                base = None
                for nv in nvs:
                    schemes = ("pcpp", "fullmap") if (nv == 8 and res == 256) else ("pcpp",)
                    for sch in schemes:
                        r = loopback_line(pcpp, torch, np, inputs, res, nv, P_BY_N[nv], sch, S, cond, args.kernels,
                                          blob2, comm_off=False)
                        if nv == 1:
                            base = r["ms_per_rank"]
                        r["projected_speedup_vs_n1"] = round(base / r["ms_per_rank"], 2) if base else None
                        large[f"res{res * 8}_n{nv}" + ("" if sch == "pcpp" else "_fullmap")] = r
                _progress(f"{res * 8}^2 lines done")
            large["note"] = ("2048^2 (X2) and 3840^2 (X3) SDXL-shaped steps: n = 1 measured on this GPU, n > 1 as loopback "
                             "projections (ms_per_rank = all-rank time / n)")
        del blob2

    # the SDXL-faithful stack: every attention layer a full transformer block (LN,
    # self-attn, LN, cross-attn to 77 tokens, LN, GEGLU FF; 2.57 B parameters), N = 1 and an n = 8 projection
    xf = None
    if rank == 0 and world == 1 and args.scheme == "pcpp" and args.res == 128 and not args.no_xf:
        xf = {}
        blob3 = inputs.make_weight_blob(inputs.init_specs(pcpp.manifest("sdxl_xf")))
        ctxt = inputs.make_context(77, 2048)
        for nv in (1, 8):
            wv = 4 if nv > 1 else 0
            cfg3 = pcpp.make_config(model="sdxl_xf", num_steps=S, precision="bf16", backend="loopback", kernels=args.kernels)
            pl = pcpp.Plan(H, W, 4, nv, P_BY_N[nv], wv, cfg3, blob3)
            pl.pcpp_set_cond(cond)
            pl.pcpp_set_context(ctxt)
            lat3 = torch.from_numpy(np.ascontiguousarray(xT)).cuda()
            for k in range(wv + 2):
                pl.pcpp_step(lat3, k)
            t = time_steps(pl, lat3, wv + 2, 5, torch)
            inf3 = pl.pcpp_query()
            pl.close()
            xf[f"n{nv}"] = {"ms_per_step_all_ranks": round(t, 4), "ms_per_rank": round(t / nv, 4),
                            "step_flops_rank_max": inf3["step_flops_rank_max"],
                            "achieved_tflops_rank": round(inf3["step_flops_rank_max"] / (t / nv * 1e-3) / 1e12, 1),
                            "simt_fallbacks": inf3["simt_fallbacks"]}
        xf["projected_speedup_n8"] = round(xf["n1"]["ms_per_rank"] / xf["n8"]["ms_per_rank"], 2)
        xf["note"] = ("sdxl_xf = SDXL's transformer blocks (2.57 B parameters, SDXL's UNet size); n = 8 is a loopback "
                      "projection (all-rank time / 8)")
        del blob3
        _progress("sdxl_xf lines done")

    if rank == 0:
        cls = ("attn", "conv", "gn")
        out = {
            "metric": METRIC, "value": round(ms, 4), "unit": "ms/step", "n_gpus": N, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic: seeded N(0,1) latent and cond, random-init SDXL-shaped weights (no checkpoint offline)",
            "config": {"workload": f"sdxl-{H * 8} ({H}x{W}x4 latent, 50-step DDIM schedule, CFG s=5 "
                                   + ("split over 2 GPU groups)" if split else "as batch 2)"),
                       "model": "SDXL-shaped UNet stack (70 self-attn, 40 conv3x3, 46 GN; SURVEY App. A)",
                       "global_batch": 2, "seq_len": H * W,
                       "parallelism": f"pcpp-patch{n}" + ("-cfgsplit2" if split else ""), "cfg_split": split,
                       "n_patches": n, "cond_fraction": p, "warmup_steps": w, "num_steps": S,
                       "scheme": args.scheme, "step_flops_per_rank": info["step_flops_rank_max"],
                       "backend": ["nccl", "loopback", "peer"][info["backend"]], "backend_note": backend_note,
                       "simt_fallbacks_per_step": info["simt_fallbacks"],
                       "l2": "per-step working set (1.57 GB bf16 weights + activations) >> 126 MB L2; no flush"},
            "bytes_exchanged_per_step": {"async": dict(zip(cls, info["bytes_counted_async"])), "eps_cfg_split": info["bytes_eps"],
                                         "warmup": dict(zip(cls, info["bytes_counted_warmup"])),
                                         "fullmap_async": dict(zip(cls, info["bytes_fullmap"]))},
            "achieved_tflops_step": round(info["step_flops_rank_max"] / (ms * 1e-3) / 1e12, 1),
            "gpu_launches": info["n_kernels_per_step"] * args.steps,
            "clocks": clk.summary(),
            "e2e": e2e, "roofline": roof, "roofline_attention": roof_attn, "roofline_groupnorm": roof_gn,
            "cpu_baseline": cpu,
            "breakdown_ms": {k: round(v["ms"], 4) for k, v in prof.items()},
            "pcpp_loopback_1gpu": loop, "sw_sweep_1024_n8": sweep, "large_resolutions": large, "sdxl_xf_1024": xf,
            "comm_off": comm_off,
            "context": "paper: 2.36-8.02x speed-up on 4-8 A100-40GB, SDXL fp16 (P:5); not comparable hardware",
            "bench_wall_s": round(time.time() - T_START, 1),
        }
        print(json.dumps(out), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
