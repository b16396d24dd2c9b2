#!/usr/bin/env python
"""bench.py — RRS A4W4 linear layer on B200 (one JSON line on rank 0).

    python bench.py [--gpus N --steps K --warmup W] [--workload c2_llama2_7b_qo] [--out-dtype bf16]
    python bench.py --impl reference ...      # the CPU oracle as the reference arm (rank 0 only)
    torchrun --nproc-per-node N bench.py --gpus N ...   # column-parallel W over N GPUs + NCCL all-gather

A step is one pass of the whole hot path (a7 is the offline weight
preparation, timed once and reported separately) over one batch of synthetic input already resident in HBM:
    rrs_rotate_smooth_quant -> rrs_gemm (-> rrs_allgather_columns when N > 1).
L2 is flushed (256 MiB write + 256 MiB clean read, bench/l2flush.py) before every timed step; each step is timed with CUDA events on the launching
stream and the bracketing barrier + synchronize surround the whole timed loop.  Multi-GPU times are the max
over ranks.  Inputs: seeded synthetic LLaMA-like activations and N(0, 0.02^2) weights (rrs_synth).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "bench"))
from l2flush import L2Flush  # noqa: E402  (bench/l2flush.py)

from rrs_synth import WORKLOADS, make_layer, make_weights  # noqa: E402

METRIC = "RRS A4W4 linear TOPS"
INT8_OVER_BF16 = 2.0  # nominal dense int8 : bf16 tensor ratio (4.5 : 2.25 PFLOP/s, B200_PROFILING.md)


def peaks():
    p = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "src": "fallback (B200_PROFILING.md)"}
    f = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(f):
        with open(f) as fh:
            m = json.load(fh)
        p = {"hbm_gbs": float(m["hbm_gbs"]), "bf16_tflops": float(m["bf16_tflops"]),
             "bf16_tflops_sustained": float(m.get("bf16_tflops_sustained", m["bf16_tflops"])),
             "src": "measured (MEASURED_PEAKS.json)"}
    return p


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------------------------------ GPU arm

def max_over_ranks(vals, device, world: int) -> float:
    """Mean of this rank's per-step times, then the MAX over ranks (the slowest rank sets the job time)."""
    import torch
    import torch.distributed as dist
    v = torch.tensor([statistics.fmean(vals)], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
    return float(v.item())


def measure_workload(args, wname, dev, world, rank, comm, cpu_base: bool, i8: bool = False):
    """Time one workload on this rank; returns the rank-0 summary (other ranks: None).

    Prefill shapes run rrs_linear (fused prologue + tcgen05 pair GEMM).  Decode-sized T (<= 64, configs[3]) runs the
    decode regime: the small-T prologue (int8 activation codes) + the packed-4-bit W stream GEMM (RRS_W_PACKED4).
    i8: the int8 operand carrier (tcgen05 kind::i8, int32 group sums -- the north_star's contract path) instead of
    the default E4M3 carrier (kind::f8f6f4, exact f32 group sums)."""
    import torch
    import torch.distributed as dist

    import paper_2409_20361_b200 as rrs

    w = WORKLOADS[wname]
    T, K, N = w.T, w.K, w.N
    out_dtype = torch.bfloat16 if args.out_dtype == "bf16" else torch.float32
    esz = 2 if args.out_dtype == "bf16" else 4
    decode = T <= 64 and world == 1

    # ---- inputs (seeded, synthetic), resident in HBM before timing
    X_bits, W_bits, Xc_bits = make_layer(w, index=list(WORKLOADS).index(wname))

    def dev_bf16(b):
        return torch.from_numpy(np.ascontiguousarray(b).view(np.int16)).to(dev).view(torch.bfloat16)

    X, W_full, Xc = dev_bf16(X_bits), dev_bf16(W_bits), dev_bf16(Xc_bits)
    stream = torch.cuda.current_stream()
    perm = rrs.calibrate_perm(Xc)                      # offline reorder (R5), on the GPU
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    layer = rrs.RRSLinear(W_full, perm, comm=comm, world=world, rank=rank, i8=i8, decode=decode)  # a7, offline
    t1.record()
    torch.cuda.synchronize()
    prep_ms = t0.elapsed_time(t1)
    del W_full
    n_local = N // world
    ws = layer.workspace(T, dev)
    Xop = torch.empty((T, K), dtype=torch.uint8, device=dev)
    xs = torch.empty(T, dtype=torch.float32, device=dev)
    sg = torch.empty(K // 128, dtype=torch.float32, device=dev)
    pws = torch.empty(rrs.rrs_workspace_bytes(T, 1, K, 128, 1), dtype=torch.uint8, device=dev)
    Y_shard = torch.empty((T, n_local), dtype=out_dtype, device=dev)
    Y = torch.empty((T, N), dtype=out_dtype, device=dev)
    flush = L2Flush(dev)
    out_scale = 1.0 / K
    op_i8 = i8 or decode  # the decode GEMM takes int8 activation codes

    def new_events(n, k):
        return [[torch.cuda.Event(enable_timing=True) for _ in range(k)] for _ in range(n)]

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def linear(Xin=X):  # one whole hot-path step through the public C-ABI entry point (a1-a9, + e when world > 1)
        if decode:
            rrs.rrs_linear(Xin, perm, layer.Wp4, layer.w_scale, Y, ws, N_total=N, packed4=True, stream=stream)
        else:
            rrs.rrs_linear(Xin, perm, layer.Wop, layer.w_scale, Y, ws, N_total=N, comm=comm, i8=i8, stream=stream)

    # ---- headline: K timed steps of rrs_linear on HBM-resident inputs, L2 flushed before each step
    for _ in range(args.warmup):
        flush.zero_()
        linear()
    barrier()
    evs = new_events(args.steps, 2)
    with ClockSampler(dev.index) as clocks:
        barrier()
        wall0 = time.perf_counter()
        for i in range(args.steps):
            flush.zero_()
            evs[i][0].record(stream)
            linear()
            evs[i][1].record(stream)
        barrier()
        wall = time.perf_counter() - wall0
    per_step = [e[0].elapsed_time(e[1]) for e in evs]

    # ---- breakdown (separate pass, L2 flushed before each timed piece, events on the launching stream):
    #   prologue / GEMM / all-gather of the layer; baselines on the SAME codes: the plain per-channel A4W4 GEMM and
    #   the sub-channel A4W4 GEMM (P:322's two efficiency baselines; the sub-channel scales are arbitrary positive
    #   numbers -- its speed does not depend on their values), and the prologues of a QuaRot-style layer (online
    #   rotation + per-token RTN, RRS_NO_SMOOTH) and of a plain A4W4 layer (per-token RTN only) for O_quarot / O_plain
    sub_ok = n_local % 8 == 0 and not decode and not i8
    G = K // 128
    sub_xs = torch.rand((G, T), dtype=torch.float32, device=dev) + 0.5
    sub_ws = torch.rand((G, n_local), dtype=torch.float32, device=dev) + 0.5
    Xop_b, xs_b, sg_b = torch.empty_like(Xop), torch.empty_like(xs), torch.empty_like(sg)
    pieces = {
        "prologue": lambda: rrs.rrs_rotate_smooth_quant(X, perm, None, Xop, xs, sg, ws=pws, i8=op_i8, stream=stream),
        "rrs_gemm": (lambda: rrs.rrs_gemm(Xop, xs, sg, layer.Wp4, layer.w_scale, Y_shard, out_scale, packed4=True,
                                          stream=stream)) if decode else
                    (lambda: rrs.rrs_gemm(Xop, xs, sg, layer.Wop, layer.w_scale, Y_shard, out_scale, i8=i8,
                                          stream=stream)),
        "quarot_prologue": lambda: rrs.rrs_rotate_smooth_quant(X, perm, None, Xop_b, xs_b, sg_b, ws=pws, i8=op_i8,
                                                               no_smooth=True, stream=stream),
        "plain_prologue": lambda: rrs.rrs_rotate_smooth_quant(X, perm, None, Xop_b, xs_b, sg_b, ws=pws, i8=op_i8,
                                                              no_smooth=True, no_rotation=True, stream=stream),
    }
    if not decode:
        pieces["plain_gemm"] = lambda: rrs.rrs_gemm(Xop, xs, None, layer.Wop, layer.w_scale, Y_shard, out_scale,
                                                    plain=True, i8=i8, stream=stream)
    if sub_ok:
        pieces["subchannel_gemm"] = lambda: rrs.rrs_gemm(Xop, sub_xs, None, layer.Wop, sub_ws, Y_shard, out_scale,
                                                         subchannel=True, stream=stream)
    if world > 1:
        pieces["allgather"] = lambda: rrs.rrs_allgather_columns(Y_shard, Y, comm, ws, stream=stream)
    if decode:  # the round-1 decode path (one byte per W code, split-K GEMM) on the same layer, for comparison
        pieces["r1_byte_operand_layer"] = lambda: rrs.rrs_linear(X, perm, layer.Wop, layer.w_scale, Y, ws, N_total=N,
                                                                 stream=stream)
    times = {k: [] for k in pieces}
    rrs.rrs_rotate_smooth_quant(X, perm, None, Xop, xs, sg, ws=pws, i8=op_i8, stream=stream)
    for i in range(args.warmup + args.steps):
        evp = {k: new_events(1, 2)[0] for k in pieces}
        for k, fn in pieces.items():
            flush.zero_()
            evp[k][0].record(stream)
            fn()
            evp[k][1].record(stream)
        torch.cuda.synchronize()
        if i >= args.warmup:
            for k in pieces:
                times[k].append(evp[k][0].elapsed_time(evp[k][1]))

    # ---- end to end through the public API with host buffers: pinned H2D of X, rrs_linear, D2H of Y
    X_host = X.cpu().pin_memory()
    Y_host = torch.empty((T, N), dtype=out_dtype).pin_memory()
    X_dev = torch.empty_like(X)
    eev = new_events(args.steps, 2)
    for i in range(args.warmup + args.steps):
        flush.zero_()
        ev = eev[i - args.warmup] if i >= args.warmup else new_events(1, 2)[0]
        ev[0].record(stream)
        X_dev.copy_(X_host, non_blocking=True)
        linear(X_dev)
        Y_host.copy_(Y, non_blocking=True)
        ev[1].record(stream)
    torch.cuda.synchronize()
    e2e = [e[0].elapsed_time(e[1]) for e in eev]

    def mx(vals):
        return max_over_ranks(vals, dev, world)

    ms_step, ms_e2e = mx(per_step), mx(e2e)
    bd = {k: mx(v) for k, v in times.items()}
    ck = clocks.summary()
    if world > 1:
        dist.barrier()
    if rank != 0:
        return None
    ops = 2.0 * T * K * N
    gemm_tops = 2.0 * T * K * n_local / (bd["rrs_gemm"] * 1e-3) / 1e12
    bd["prepare_weights_offline"] = prep_ms
    res = {
        "workload": wname, "T": T, "K": K, "N": N, "ms_per_step": ms_step, "carrier": "int8" if op_i8 else "e4m3",
        "path": "decode (small-T prologue + packed-4-bit W stream GEMM)" if decode else "prefill",
        "tops": ops / (ms_step * 1e-3) / 1e12, "tokens_per_s": T / (ms_step * 1e-3),
        "breakdown_ms": bd, "gemm_tops": gemm_tops,
        "e2e_tops": ops / (ms_e2e * 1e-3) / 1e12, "h2d": T * K * 2, "d2h": T * N * esz,
        "clocks": ck, "wall_s_timed_region": wall,
    }
    if "plain_gemm" in bd:
        res["rrs_overhead_vs_plain_gemm"] = bd["rrs_gemm"] / bd["plain_gemm"] - 1.0  # O_gemm
        res["o_quarot"] = ms_step / (bd["quarot_prologue"] + bd["plain_gemm"]) - 1.0
        res["o_plain"] = ms_step / (bd["plain_prologue"] + bd["plain_gemm"]) - 1.0
    if decode:
        wbytes = layer.Wp4.numel()
        res["w_stream_gbs"] = wbytes / (bd["rrs_gemm"] * 1e-3) / 1e9
        res["w_bytes"] = wbytes
    if cpu_base:
        res["cpu_baseline"] = cpu_baseline(w, X_bits, W_bits, Xc_bits, budget_s=args.cpu_budget)
    return res


def measure_mlp(args, dev, prerotated: bool = False):
    """SURVEY §8 f1 on config C3 (LLaMA-3-8B MLP, 4096-token prefill, D = 4096, F = 14336), single GPU:
    h = SwiGLU fused into ONE RRS GEMM over the interleaved gate/up rows (one prologue on X), then the
    down_proj RRS layer on h.  Ops = 2 T D (2F) + 2 T F D.  prerotated: the up/gate input arrives already rotated
    (RRS_PREROTATED: its prologue skips the online FWHT; down_proj still rotates online)."""
    import torch

    import paper_2409_20361_b200 as rrs

    wu = WORKLOADS["c3_llama3_8b_up"]
    T, D, F = wu.T, wu.K, wu.N
    X_bits, _, Xc_bits = make_layer(wu, index=list(WORKLOADS).index("c3_llama3_8b_up"), N=8)

    def dev_bf16(b):
        return torch.from_numpy(np.ascontiguousarray(b).view(np.int16)).to(dev).view(torch.bfloat16)

    X, Xc = dev_bf16(X_bits), dev_bf16(Xc_bits)
    Wg, Wu_, Wd = (dev_bf16(make_weights(*shape, seed)) for shape, seed in
                   (((F, D), 7101), ((F, D), 7102), ((D, F), 7103)))
    perm_in = rrs.calibrate_perm(Xc)
    up_gate = rrs.RRSLinear(rrs.interleave_gate_up(Wg, Wu_), perm_in, swiglu=True, prerotated=prerotated)
    perm_mid = rrs.calibrate_perm(up_gate(Xc))  # offline reorder of the down_proj input (R5)
    down = rrs.RRSLinear(Wd, perm_mid)
    del Wg, Wu_, Wd
    stream = torch.cuda.current_stream()
    flush = L2Flush(dev)
    h = torch.empty((T, F), dtype=torch.bfloat16, device=dev)
    Y = torch.empty((T, D), dtype=torch.bfloat16, device=dev)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.warmup + args.steps)]
    for ev in evs:
        flush.zero_()
        ev[0].record(stream)
        up_gate(X, Y=h, stream=stream)
        ev[1].record(stream)
        down(h, Y=Y, stream=stream)
        ev[2].record(stream)
    torch.cuda.synchronize()
    evs = evs[args.warmup:]
    ug = float(np.median([e[0].elapsed_time(e[1]) for e in evs]))
    dn = float(np.median([e[1].elapsed_time(e[2]) for e in evs]))
    step = float(np.median([e[0].elapsed_time(e[2]) for e in evs]))
    ops = 2.0 * T * D * 2 * F + 2.0 * T * F * D
    return {"ms_per_step": step, "tops": ops / (step * 1e-3) / 1e12, "tokens_per_s": T / (step * 1e-3),
            "breakdown_ms": {"up_gate_swiglu (prologue + one GEMM over 2F rows)": ug,
                             "down_proj (K = 14336 prologue + GEMM)": dn},
            "note": "SURVEY 8 f1: LLaMA-3-8B MLP block, T=4096 D=4096 F=14336, bf16 h and Y, L2 flushed per step"
                    + ("; up/gate input pre-rotated (RRS_PREROTATED, P:138)" if prerotated else "")}


def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_2409_20361_b200 as rrs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    comm = rrs.make_comm()[0] if world > 1 else None

    head = measure_workload(args, args.workload, dev, world, rank, comm,
                            cpu_base=(world == 1 and not args.no_cpu_baseline))
    extras = {}
    keep = ("path", "carrier", "ms_per_step", "tops", "tokens_per_s", "breakdown_ms", "gemm_tops",
            "rrs_overhead_vs_plain_gemm", "o_quarot", "o_plain", "w_stream_gbs", "e2e_tops")
    for wn in (args.also.split(",") if args.also else []):
        if wn.startswith("c3_llama3_8b_mlp"):
            if world == 1:
                extras[wn] = measure_mlp(args, dev, prerotated=wn.endswith("_prerotated"))
            continue
        i8 = wn.endswith("_i8")
        r = measure_workload(args, wn[:-3] if i8 else wn, dev, world, rank, comm, cpu_base=False, i8=i8)
        if r is not None:
            extras[wn] = {k: r[k] for k in keep if k in r}
            if "w_stream_gbs" in r:  # decode: the W stream against the HBM roofline
                pk = peaks()
                extras[wn]["roofline"] = {
                    "bound": "hbm", "kernel": "rrs_decode_gemm_kernel", "achieved": r["w_stream_gbs"],
                    "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": r["w_stream_gbs"] / pk["hbm_gbs"],
                    "algorithmic": f"packed 4-bit W ({r['w_bytes']} B) per launch / decode GEMM CUDA-event time",
                    "step_frac": (r["w_bytes"] / (pk["hbm_gbs"] * 1e9)) / (r["ms_per_step"] * 1e-3),
                    "step_frac_note": "whole layer step vs its W-stream floor (W bytes / HBM peak)"}
    if world > 1:
        dist.barrier()
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return None

    pk = peaks()
    int8_peak = pk["bf16_tflops"] * INT8_OVER_BF16
    sm_mhz = (head["clocks"] or {}).get("sm_mhz") or 1965.0
    micro_peak = 8189.0 * 2 * 148 * sm_mhz * 1e6 / 1e12  # tcgen05 microbenchmark: 8189 MAC/clk/SM (profiles/micro_r1.txt)
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof):
        with open(prof) as fh:
            traffic = json.load(fh).get(args.workload, {}).get("gemm_dram_bytes_per_launch")
    w = WORKLOADS[args.workload]
    pow2 = (w.K & (w.K - 1)) == 0  # K = 2^m: the single-launch fused prologue
    # prologue rooflines: FP64 DADDs of the exact FWHT (K log2 K per token; 28*2^m: m + 14 per element)
    # against 64 DADD/clk/SM, and algorithmic HBM bytes (2K read + K operand bytes + 4 per token, 4K + 4G per call)
    a_k = (w.K.bit_length() - 1) if pow2 else ((w.K // 28).bit_length() - 1 + 14)
    t_pro = head["breakdown_ms"]["prologue"] * 1e-3
    dadd = float(w.T) * w.K * a_k
    fp64_peak = 64.0 * 148 * sm_mhz * 1e6
    pro_bytes = w.T * (3.0 * w.K + 4) + 4.0 * w.K + 4.0 * (w.K // 128)
    out = {
        "metric": METRIC,
        "value": head["tops"],
        "unit": "TOPS",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": head["ms_per_step"],
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "int4 codes (e4m3 carrier: tcgen05 kind::f8f6f4, exact f32 group sums; fp64 rotation, f32 scales)",
        "data": "synthetic (seeded LLaMA-like bf16 activations, N(0,0.02^2) bf16 weights; rrs_synth)",
        "config": {"workload": args.workload, "T": w.T, "K": w.K, "N": w.N, "group": 128,
                   "out_dtype": args.out_dtype, "note": w.note,
                   "parallelism": f"tp-columns x{world} (W column-sharded, X replicated, NCCL all-gather of Y)"
                   if world > 1 else "single GPU",
                   "l2": L2Flush.describe},
        "tokens_per_s": head["tokens_per_s"],
        "breakdown_ms": head["breakdown_ms"],
        "gemm_tops": head["gemm_tops"],
        "gemm_pct_int8_peak": 100.0 * head["gemm_tops"] / int8_peak,
        "rrs_overhead_vs_plain_gemm": head.get("rrs_overhead_vs_plain_gemm"),
        "o_quarot": head.get("o_quarot"),
        "o_plain": head.get("o_plain"),
        "roofline": {"bound": "tensor", "kernel": "rrs_gemm_kernel", "achieved": head["gemm_tops"],
                     "peak": int8_peak, "unit": "TFLOP/s", "frac": head["gemm_tops"] / int8_peak,
                     "traffic": traffic,
                     "peak_src": f"int8/fp8 = {INT8_OVER_BF16:g} x bf16 burst {pk['bf16_tflops']} TFLOP/s, {pk['src']}",
                     "frac_vs_tcgen05_microbench": head["gemm_tops"] / micro_peak,
                     "tcgen05_microbench_peak": micro_peak,
                     "frac_vs_nominal_4500": head["gemm_tops"] / 4500.0,
                     "algorithmic": "2*T*K*N_local int ops per launch / rrs_gemm CUDA-event time (SURVEY 8(d))"},
        "prologue_roofline": {"bound": "fp64", "kernel": "prologue_group_kernel" if pow2 else
                              "fwht_colmax_kernel + smooth_quant_kernel",
                              "achieved": dadd / t_pro / 1e12, "peak": fp64_peak / 1e12, "unit": "T DADD/s",
                              "frac": dadd / t_pro / fp64_peak,
                              "hbm_achieved_gbs": pro_bytes / t_pro / 1e9, "hbm_peak_gbs": pk["hbm_gbs"],
                              "hbm_frac": pro_bytes / t_pro / 1e9 / pk["hbm_gbs"],
                              "algorithmic": f"T*K*{a_k} DADD (exact FWHT) and T*(3K+4)+4K+4G bytes per call",
                              "note": "issue-bound, not FP64-bound: 34 executed instructions per element of which 12 "
                                      "DADD, 8 warps/SM at 255 registers (profiles/ncu_r2f3.txt, DESIGN.md 7)"},
        "headline_context": {k: {kk: extras[k].get(kk) for kk in ("tops", "ms_per_step", "rrs_overhead_vs_plain_gemm")}
                             for k in ("c3_llama3_8b_down", "c3_llama3_8b_mlp") if k in extras},
        "e2e": {"value": head["e2e_tops"], "unit": "TOPS", "h2d_bytes_per_step": head["h2d"],
                "d2h_bytes_per_step": head["d2h"],
                "api": "rrs_linear (pinned host X -> device -> host Y, copies inside the timed region)"},
        "gpu_launches": (2 if pow2 else 3) + (1 if world > 1 else 0),
        "gpu_launches_note": "per step: " + ("prologue_group_kernel" if pow2 else
                                             "fwht_colmax_kernel, smooth_quant_kernel (+ one cudaMemsetAsync of chan_max)")
                             + ", rrs_gemm_kernel"
                             + (", relayout_kernel (+ ncclAllGather)" if world > 1 else ""),
        "clocks": head["clocks"],
        "wall_s_timed_region": head["wall_s_timed_region"],
    }
    if "cpu_baseline" in head:
        out["cpu_baseline"] = head["cpu_baseline"]
    if extras:
        out["also"] = extras
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return out


# ------------------------------------------------------------------------------------------ CPU oracle

def _oracle_step(o, Xs, Wr_prepared, perm, K):
    Xr = o.rotate(Xs)
    c = o.channel_max(Xr)
    s = o.group_scales(c, perm, 128)
    q, a = o.smooth_quant(Xr, perm, s, 128)
    qw, beta = Wr_prepared
    return o.scale_accumulate_rows(q, qw, s, a, beta, 128, 1.0 / K)


def cpu_baseline(w, X_bits, W_bits, Xc_bits, budget_s=20.0, rows=None):
    """The oracle as it stands, timed on this host's cores on a bounded token sample of the workload."""
    from oracle import rrs_oracle as o
    from rrs_synth import bf16_bits_to_f64
    try:
        from threadpoolctl import threadpool_info
        threads = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        threads = os.cpu_count()
    perm = o.calibrate_perm(bf16_bits_to_f64(Xc_bits[:256]))
    qw, beta, _ = o.prepare_weights(bf16_bits_to_f64(W_bits), perm)  # offline, not timed
    T = rows or min(w.T, 256)
    Xs = bf16_bits_to_f64(X_bits[:T])
    t = time.perf_counter()
    n = 0
    while True:
        _oracle_step(o, Xs, (qw, beta), perm, w.K)
        n += 1
        if time.perf_counter() - t > budget_s / 2 or n >= 8:
            break
    dt = (time.perf_counter() - t) / n
    return {"value": 2.0 * T * w.K * w.N / dt / 1e12, "unit": "TOPS", "cores": threads, "kind": "oracle",
            "sample": f"{T} of {w.T} tokens of {w.name} (K={w.K}, N={w.N}), full layer forward a1-a9 "
                      f"(weights prepared offline, untimed), {n} repetitions, {dt:.2f} s each"}


def run_reference(args):
    """--impl reference: the CPU oracle as the reference arm (rank 0 only; other ranks exit 0)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    from oracle import rrs_oracle as o
    from rrs_synth import bf16_bits_to_f64
    w = WORKLOADS[args.workload]
    X_bits, W_bits, Xc_bits = make_layer(w, index=list(WORKLOADS).index(args.workload))
    perm = o.calibrate_perm(bf16_bits_to_f64(Xc_bits[:256]))
    qw, beta, _ = o.prepare_weights(bf16_bits_to_f64(W_bits), perm)
    T = min(w.T, args.ref_rows)
    Xs = bf16_bits_to_f64(X_bits[:T])
    for _ in range(args.warmup):
        _oracle_step(o, Xs, (qw, beta), perm, w.K)
    times = []
    for _ in range(args.steps):
        t = time.perf_counter()
        _oracle_step(o, Xs, (qw, beta), perm, w.K)
        times.append(time.perf_counter() - t)
    dt = statistics.fmean(times)
    try:
        from threadpoolctl import threadpool_info
        threads = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        threads = os.cpu_count()
    value = 2.0 * T * w.K * w.N / dt / 1e12
    sample = f"{T} of {w.T} tokens of {w.name} per step (K={w.K}, N={w.N}), layer forward a1-a9"
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": "TOPS", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (rrs_synth)",
           "config": {"workload": args.workload, "T": w.T, "K": w.K, "N": w.N, "group": 128,
                      "sample_tokens": T},
           "cpu_baseline": {"value": value, "unit": "TOPS", "cores": threads, "kind": "oracle", "sample": sample},
           "e2e": {"value": value, "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return out


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["rrs", "reference"], default="rrs")
    ap.add_argument("--workload", default="c3_llama3_8b_up", choices=sorted(WORKLOADS))
    ap.add_argument("--also", default="c3_llama3_8b_down,c3_llama3_8b_mlp,c3_llama3_8b_mlp_prerotated,c3_llama3_8b_up_i8,"
                                      "c2_llama2_7b_qo,c4_decode_t64,c4_decode_t1,c5_llama3_70b_up_rank8",
                    help="comma-separated extra workloads summarised under 'also' (empty: none)")
    ap.add_argument("--out-dtype", default="bf16", choices=["bf16", "f32"])
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--ref-rows", type=int, default=256)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    main()
