#!/usr/bin/env python
"""bench.py — GRAF ambiguity-function hot path on B200 (BASELINE.json metric:
"AF forward+loss+grad surfaces/sec (N x M cells/s) and % of HBM/FP32 roofline").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl graf|reference]

A step = one forward + loss + gradient pass of the whole hot path (SURVEY.md
§8(a) rows a0-a7, plus a8 when sharded) over one batch of seeded synthetic
waveforms of the chosen BASELINE.json config (default: configs[1] = c2, B=256,
N=M=256, masked ISL, fused single pass), called through the C ABI
(graf_af_loss_grad).  Inputs are resident in HBM before timing; each timed step
is a CUDA-graph replay of that call, timed with CUDA events on the launching
stream, with L2 flushed (256 MiB memset) between steps outside the events.
Multi-GPU (torchrun): batch sharding, every rank runs its own batch (weak
scaling, no data-path collective); time = max over ranks.

`--impl reference`: this build has no reference implementation (the paper
ships no code); the reference arm is the float64 CPU oracle (oracle/), timed on
the host cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from graf_inputs import CONFIGS, config_waveforms  # noqa: E402

FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12   # B200_PROFILING.md: 148 SMs, 1965 MHz; 128 FP32 lanes/SM


def workload(cid: int) -> dict:
    cfg = CONFIGS[cid]
    loss = dict(cfg["loss"])
    note = ""
    if cid in (1, 3):
        # DESIGN.md R12: normalised full-plane ISL is identically M-1 with a zero
        # gradient (volume identity); time the raw mode, whose gradient is real work.
        loss["normalize"] = 0
        note = "raw (unnormalised) full-plane ISL: the normalised one is constant (volume identity)"
    N, M, B = cfg["N"], cfg["M"], cfg["B"]
    rows = min(loss["k_max"], N - 1) + 1                       # folded delay rows k >= 0
    ffts = 2 if loss["lambda_psl"] == 0 else 3                  # fused ISL: fwd+inv; soft-PSL: fwd | fwd+inv
    single = False
    if ffts == 3 and not cfg["surface"]:
        # band cache (graf_api.cu make_plan): a band of <= M/4 bins (cache <= 1 GiB) is kept
        # from pass 1, so pass 2 runs only the inverse FFT -- count the FFTs actually executed
        nband = 2 * min(loss["d_max"], M // 2) + 1
        if nband <= M // 4 and B * rows * nband * 8 <= (1 << 30):
            ffts = 2
            note = "soft-PSL two-pass with the band cache: pass 2 reuses pass 1's in-band FFT outputs"
        full = (min(loss["k_max"], N - 1) == N - 1 and loss["d_max"] >= M // 2 and loss.get("ml_k", 0) == 0
                and loss.get("ml_d", 0) == 0 and loss.get("normalize", 1) == 1)
        if full:
            # full-plane centred soft-PSL (R13): one pass of forward + inverse FFT per row,
            # guarded fallback passes only for waveforms outside the validity rule
            ffts = 2
            single = True
            note = "full-plane soft-PSL as one optimistic pass (R13), per-waveform guarded fallback"
    flops = B * rows * ffts * 5.0 * M * math.log2(M)             # SURVEY.md §8(d) algorithmic FFT flops
    surf_bytes = 0
    if cfg["surface"]:
        per = 8 if cfg["surface"] == "c64" else 4
        surf_bytes = B * (2 * N - 1) * M * per
    io_bytes = B * N * 8 * 2
    return dict(cid=cid, cfg=cfg, loss=loss, N=N, M=M, B=B, rows=rows, ffts=ffts, flops=flops, single=single,
                surf_bytes=surf_bytes, io_bytes=io_bytes, note=note,
                launches=(2 if loss["lambda_psl"] == 0 else 4))


def describe(w: dict) -> str:
    c = w["cfg"]
    L = w["loss"]
    return (f"{c['name']}: B={w['B']} N={w['N']} M={w['M']} {c['family']}; "
            f"{'surface ' + c['surface'] + ' + ' if c['surface'] else ''}"
            f"ISL x{L['lambda_isl']} + softPSL x{L['lambda_psl']} (T={L['temperature']}) on |k|<={L['k_max']}, "
            f"|d|<={L['d_max']} minus |k|<={L['ml_k']}&|d|<={L['ml_d']}, normalize={L['normalize']}")


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "200", "-i", str(gpu_index)], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None
        self.t0 = time.time()

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        self.f.seek(0)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.f.name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def read_traffic(key: str):
    """dram read+write bytes per launch of the dominant kernel from one ncu --set full
    capture (profiles/traffic.json, key c<config>[fwd|per|match|cross]), else None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    try:
        return json.load(open(p)).get(f"c{key}")
    except Exception:
        return None


# ---------------------------------------------------------------------------
def cpu_baseline(w: dict, budget_s: float = 12.0) -> dict:
    """The float64 oracle as it stands, on the host cores, on a bounded sample."""
    from oracle import graf_oracle as O
    try:
        from threadpoolctl import threadpool_info
        threads = max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        threads = os.cpu_count()
    spec = O.LossSpec.from_dict(w["loss"])
    N, M = w["N"], w["M"]
    done, t0 = 0, time.perf_counter()
    b = 0
    while True:
        s = config_waveforms(w["cid"], batch=1, start=b % w["B"])[0]
        if w["N"] * w["M"] > 4096 * 8192:          # c5: the direct sum takes minutes per waveform
            s_small = s
            O.loss_and_grad_chunked(s_small, M, spec)
        elif w.get("match"):
            tgt = np.random.default_rng(b).random((2 * N - 1, M)) / M
            O.match_loss_and_grad(s, M, spec, tgt, -(N - 1), "centered")
        elif w.get("cross"):
            s2 = config_waveforms(w["cid"], batch=1, start=(b + 777) % w["B"])[0]
            O.cross_loss_and_grad(s, s2, M, spec)
        else:
            per = w.get("periodic", False)
            O.loss_and_grad(s, M, spec, periodic=per)
            if w["cfg"]["surface"]:
                O.surface(s, M, w["cfg"]["surface"], "centered", periodic=per,
                          **(dict(k_begin=-(N // 2), k_end=N // 2) if per else {}))
        done += 1
        b += 1
        el = time.perf_counter() - t0
        if el > budget_s or done >= w["B"]:
            break
    v = done / el
    return {"value": v, "unit": "surfaces/s", "cores": threads, "kind": "oracle",
            "sample": f"{done} of {w['B']} {w['cfg']['name']} waveforms ({el:.1f} s, float64 direct-sum oracle)"}


def run_reference(args, w) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import graf_oracle as O
    spec = O.LossSpec.from_dict(w["loss"])
    per_step = {1: 1, 2: 8, 3: 1, 4: 1, 5: 1}[w["cid"]]
    if w["cid"] == 5:
        print(json.dumps({"impl": "reference", "unavailable":
                          "float64 direct-sum oracle needs ~10 min per c5 waveform (N=M=16384)"}))
        return

    def step(i):
        for j in range(per_step):
            s = config_waveforms(w["cid"], batch=1, start=(i * per_step + j) % w["B"])[0]
            per = w.get("periodic", False)
            if w.get("match"):
                tgt = np.random.default_rng(j).random((2 * w["N"] - 1, w["M"])) / w["M"]
                O.match_loss_and_grad(s, w["M"], spec, tgt, -(w["N"] - 1), "centered")
                continue
            if w.get("cross"):
                s2 = config_waveforms(w["cid"], batch=1, start=(j + 777) % w["B"])[0]
                O.cross_loss_and_grad(s, s2, w["M"], spec)
                continue
            O.loss_and_grad(s, w["M"], spec, periodic=per)
            if w["cfg"]["surface"]:
                O.surface(s, w["M"], w["cfg"]["surface"], "centered", periodic=per,
                          **(dict(k_begin=-(w["N"] // 2), k_end=w["N"] // 2) if per else {}))

    for i in range(args.warmup):
        step(i)
    t0 = time.perf_counter()
    for i in range(args.steps):
        step(args.warmup + i)
    el = time.perf_counter() - t0
    v = per_step * args.steps / el
    try:
        from threadpoolctl import threadpool_info
        threads = max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        threads = os.cpu_count()
    line = {"metric": "AF forward+loss+grad surfaces/sec", "value": v, "unit": "surfaces/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": describe(w), "sample_per_step": f"{per_step} waveform(s)"},
            "cpu_baseline": {"value": v, "unit": "surfaces/s", "cores": threads, "kind": "oracle",
                             "sample": f"{per_step} waveform(s) per step x {args.steps} steps"},
            "e2e": {"value": v, "unit": "surfaces/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="graf", choices=["graf", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--settle-s", type=float, default=1.0)
    ap.add_argument("--mode", default="loss_grad", choices=["loss_grad", "forward", "lpi", "match", "cross", "mlw"],
                    help="forward: full-surface mode (graf_af_forward writes the config's surface, no loss)")
    ap.add_argument("--periodic", action="store_true",
                    help="the paper's circular surface (Eq. 2 / Alg. 1, SURVEY 8(f) NEXT-1); needs M == N")
    args = ap.parse_args()
    if args.mode == "lpi":
        return run_lpi(args)
    if args.mode == "mlw":
        return run_mlw(args)
    w = workload(args.config)
    w["periodic"] = bool(args.periodic)
    if args.periodic:
        if w["N"] != w["M"]:
            raise SystemExit("--periodic needs a config with M == N (c1, c2, c3, c5)")
        # folded circular rows k = 0..min(k_max, N/2), same FFT work per row
        w["rows"] = min(w["loss"]["k_max"], w["N"] // 2) + 1
        w["flops"] = w["B"] * w["rows"] * w["ffts"] * 5.0 * w["M"] * math.log2(w["M"])
        if w["cfg"]["surface"]:
            w["surf_bytes"] = w["B"] * w["N"] * w["M"] * (8 if w["cfg"]["surface"] == "c64" else 4)
        w["note"] = (w["note"] + "; " if w["note"] else "") + "periodic (circular) surface, paper Eq. 2 / Alg. 1"
    if args.mode == "forward":
        if not w["cfg"]["surface"]:
            raise SystemExit("--mode forward needs a config with a surface (c1, c3)")
        # folded rows covering the whole surface window, one forward FFT each
        w["flops"] = w["B"] * (w["N"] // 2 + 1 if args.periodic else w["N"]) * 5.0 * w["M"] * math.log2(w["M"])
        w["io_bytes"] = w["B"] * w["N"] * 8
        w["launches"] = 1
        w["note"] = "full-surface mode: graf_af_forward writes the surface; no loss or gradient"
    if args.mode == "match":
        # match loss ||x - x_target||^2 over the config's region (NEXT-3): one fused
        # pass streaming a per-waveform fp32 target of the full surface window
        w["loss"] = dict(w["loss"], lambda_isl=0.0, lambda_psl=0.0, normalize=1)
        w["match"] = True
        w["ffts"] = 2
        w["rows"] = min(w["loss"]["k_max"], w["N"] - 1) + 1
        w["flops"] = w["B"] * w["rows"] * 2 * 5.0 * w["M"] * math.log2(w["M"])
        # algorithmic bytes: s + g + the target cells of the region (both mirrored rows)
        w["surf_bytes"] = w["B"] * (2 * w["rows"] - 1) * min(w["M"], 2 * w["loss"]["d_max"] + 1) * 4
        w["launches"] = 2
        w["note"] = "match loss over the region, per-waveform fp32 target of the surface window (HBM-streamed)"
    if args.mode == "cross":
        # cross-ambiguity of waveform pairs (NEXT-4): the config's loss on
        # X = sum s1 conj(s2(n-k)) W^{mn}, rows unfolded (no mirror symmetry)
        w["cross"] = True
        w["rows"] = 2 * min(w["loss"]["k_max"], w["N"] - 1) + 1
        w["flops"] = w["B"] * w["rows"] * w["ffts"] * 5.0 * w["M"] * math.log2(w["M"])
        w["io_bytes"] = w["B"] * w["N"] * 8 * 4
        w["note"] = "cross-ambiguity of (s1, s2) pairs, unfolded rows; loss/grad w.r.t. both"
    if args.impl == "reference":
        return run_reference(args, w)

    import torch
    import torch.distributed as dist

    import paper_2506_22935_b200 as graf

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    W = max(3, args.warmup)

    B, N, M = w["B"], w["N"], w["M"]
    s_host = torch.from_numpy(config_waveforms(w["cid"], batch=B, start=rank * B)).pin_memory()
    s = s_host.to(dev)
    spec = graf.LossSpec.from_dict(w["loss"])
    out = w["cfg"]["surface"]
    if w.get("match"):
        out = None
        spec.lambda_match = 1.0
        g_ = torch.Generator(device=dev)
        g_.manual_seed(1234 + rank)
        spec.target = torch.rand((B, 2 * N - 1, M), generator=g_, device=dev) * (1.0 / M)
    ws = graf.graf.Workspace()
    grad = torch.empty((B, N), dtype=torch.complex64, device=dev)
    loss_out = torch.empty((B,), dtype=torch.float64, device=dev)
    surf = None
    # periodic: Alg. 1's N x N surface with both axes fftshifted (delays [-N/2, N/2))
    kb = dict(periodic=True, k_begin=-(N // 2), k_end=N // 2) if args.periodic else {}
    if out:
        nrows = N if args.periodic else 2 * N - 1
        surf = torch.empty((B, nrows, M), dtype=torch.complex64 if out == "c64" else torch.float32, device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    stream = torch.cuda.Stream(dev)
    ev_k0, ev_k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    delay = (w["cid"] == 5 and world > 1)   # c5: delay-axis sharding with NCCL exchange (strong scaling)
    if delay:
        from paper_2506_22935_b200 import sharding
        s_host = torch.from_numpy(config_waveforms(w["cid"], batch=B, start=0)).pin_memory()
        s = s_host.to(dev)

    if w.get("cross"):
        s2_host = torch.from_numpy(config_waveforms(w["cid"], batch=B, start=rank * B + 777)).pin_memory()
        s2 = s2_host.to(dev)

    def call(st=None):
        if w.get("cross"):
            graf.xaf_loss_grad(s, s2, M, spec, ws=ws, stream=st)
            return
        if delay:
            sharding.delay_sharded_loss_grad(s, M, spec, backend=tb)
            return
        if args.mode == "forward":
            graf.af_forward(s, M, out=out, layout="centered", ws=ws, surface=surf, stream=st, **kb)
            return
        graf.af_loss_grad(s, M, spec, out=out, layout="centered", ws=ws, grad=grad, loss_out=loss_out,
                          surface=surf, stream=st, **kb)

    with torch.cuda.stream(stream):
        call(stream)                                    # twiddle init + workspace, before capture
    torch.cuda.synchronize()
    L = graf.lib()
    launches_per_step = int(L.graf_last_launch_count())   # device ops the ABI call enqueued
    # the dominant kernel(s) are bracketed by events the ABI records around its
    # delay-row kernels (graf_set_profile_events); recorded into the captured graph,
    # so the kernel time comes from the same graph replays as the step time
    ev_k0.record(stream)        # torch creates the CUDA events lazily on first record
    ev_k1.record(stream)
    torch.cuda.synchronize()
    if delay:
        tb = TimedBackend(graf, sharding)
        class _Eager:                     # NCCL step: eager replay (no graph)
            def replay(self_inner):
                call(stream)
        g = _Eager()
    else:
        g = torch.cuda.CUDAGraph()               # the timed step (no event nodes)
        with torch.cuda.graph(g, stream=stream):
            call(stream)
        g_k = torch.cuda.CUDAGraph()             # the same call with the kernel events recorded
        L.graf_set_profile_events(ctypes_ptr(ev_k0), ctypes_ptr(ev_k1))
        with torch.cuda.graph(g_k, stream=stream):
            call(stream)
        L.graf_set_profile_events(None, None)
    torch.cuda.synchronize()

    sampler = ClockSampler(local if "CUDA_VISIBLE_DEVICES" not in os.environ else 0)
    with torch.cuda.stream(stream):
        for _ in range(W):
            flush.zero_()
            g.replay()
        t_end = time.time() + args.settle_s          # bring clocks to load before timing
        while time.time() < t_end:
            for _ in range(20):
                g.replay()
            stream.synchronize()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev_a = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev_b = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    kern_ms = []
    with torch.cuda.stream(stream):
        for i in range(args.steps):
            flush.zero_()
            ev_a[i].record(stream)
            g.replay()
            ev_b[i].record(stream)
        ev_b[-1].synchronize()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    step_ms = [a.elapsed_time(b) for a, b in zip(ev_a, ev_b)]
    # dominant kernel(s): ev_k0/ev_k1 around the delay-row kernels, same inputs, same
    # L2 flush protocol (graph replays; eager ABI calls for the NCCL-sharded step)
    if delay:
        with torch.cuda.stream(stream):
            for i in range(args.steps):
                flush.zero_()
                call(stream)
                torch.cuda.synchronize()
                kern_ms.append(tb.kernel_ms())
    else:
        with torch.cuda.stream(stream):
            for i in range(args.steps):
                flush.zero_()
                g_k.replay()
                ev_k1.synchronize()
                kern_ms.append(ev_k0.elapsed_time(ev_k1))
    total_ms = sum(step_ms)
    kern_avg = sum(kern_ms) / len(kern_ms)
    if world > 1:
        t = torch.tensor([total_ms, kern_avg], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, kern_avg = t.tolist()
    ms_per_step = total_ms / args.steps
    units = B if delay else world * B           # delay sharding: the ranks share one batch
    value = units * args.steps / (total_ms / 1e3)

    # ---- e2e: public API, pinned host buffers, H2D + call + D2H inside the timed region
    g_host = torch.empty((B, N), dtype=torch.complex64).pin_memory()
    l_host = torch.empty((B,), dtype=torch.float64).pin_memory()
    s_dev2 = torch.empty_like(s)
    zrow_host = None
    e2e_ms = []
    with torch.cuda.stream(stream):
        for i in range(W + args.steps):
            flush.zero_()
            a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            s_dev2.copy_(s_host, non_blocking=True)
            if w.get("cross"):
                lo, gr, gr2, _ = graf.xaf_loss_grad(s_dev2, s2, M, spec, ws=ws, stream=stream)
            elif delay:
                lo, gr = sharding.delay_sharded_loss_grad(s_dev2, M, spec)
            elif args.mode == "forward":
                sf, _ = graf.af_forward(s_dev2, M, out=out, layout="centered", ws=ws, surface=surf, stream=stream,
                                        **kb)
                zrow = sf[:, N // 2 if args.periodic else N - 1, :]   # zero-delay cut of every surface
                if zrow_host is None:
                    zrow_host = torch.empty(zrow.shape, dtype=zrow.dtype).pin_memory()
                zrow_host.copy_(zrow, non_blocking=True)
                b_.record(stream)
                b_.synchronize()
                if i >= W:
                    e2e_ms.append(a.elapsed_time(b_))
                continue
            else:
                lo, gr, _ = graf.af_loss_grad(s_dev2, M, spec, out=out, layout="centered", ws=ws, surface=surf,
                                              stream=stream, **kb)
            l_host.copy_(lo, non_blocking=True)
            g_host.copy_(gr, non_blocking=True)
            b_.record(stream)
            b_.synchronize()
            if i >= W:
                e2e_ms.append(a.elapsed_time(b_))
    e2e_total = sum(e2e_ms)
    if world > 1:
        t = torch.tensor([e2e_total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_total = t.item()
    e2e_value = units * len(e2e_ms) / (e2e_total / 1e3)

    # ---- roofline of the dominant kernel (af_rows_kernel), per launch window
    t_k = kern_avg / 1e3
    if delay:
        w["flops"] = w["flops"] / world       # this rank's delay rows
    fl_tf = w["flops"] / t_k / 1e12
    hbm = None
    try:
        hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        hbm = 6650.0
    bytes_k = w["surf_bytes"] + w["io_bytes"]
    t_alu = w["flops"] / (FP32_PEAK_TFLOPS * 1e12)
    t_hbm = bytes_k / (hbm * 1e9)
    if t_hbm > t_alu:
        roof = {"bound": "hbm", "achieved": bytes_k / t_k / 1e9, "peak": hbm, "unit": "GB/s",
                "frac": bytes_k / t_k / 1e9 / hbm, "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)"}
    else:
        roof = {"bound": "alu", "achieved": fl_tf, "peak": round(FP32_PEAK_TFLOPS, 2), "unit": "TFLOP/s",
                "frac": fl_tf / FP32_PEAK_TFLOPS,
                "peak_source": "derived: 148 SMs x 128 FP32 lanes x 2 flop x 1965 MHz (B200_PROFILING.md)"}
    roof["traffic"] = read_traffic(f"{w['cid']}{'fwd' if args.mode == 'forward' else ''}"
                                   f"{'per' if args.periodic else ''}{args.mode if args.mode in ('match', 'cross') else ''}")
    two_pass = " (single pass + guarded fallback)" if w.get("single") else " (pass 1 + reduce + pass 2)"
    roof["kernel"] = (f"af_rows_kernel<{M}>" + (two_pass if w["loss"]["lambda_psl"] else "")
                      + (" with the fused cluster finalize" if launches_per_step == 1 and args.mode != "forward"
                         else ""))
    roof["kernel_ms"] = kern_avg
    roof["algorithmic_flops_per_launch"] = w["flops"]
    roof["algorithmic_bytes_per_launch"] = bytes_k
    roof["share_of_step"] = kern_avg / ms_per_step
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(w)
    if rank == 0:
        line = {"metric": ("AF forward+loss+grad surfaces/sec" if args.mode != "forward"
                           else "AF forward (full-surface) surfaces/sec"), "value": value, "unit": "surfaces/s",
                "n_gpus": world, "steps": args.steps, "warmup": W, "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": "strong" if delay else "weak", "vs_baseline": None,
                "dtype": "f32",
                "data": "synthetic",
                "config": {"workload": describe(w), "B_per_gpu": B, "N": N, "M": M,
                           "cells_per_s": value * N * M,
                           "parallelism": (f"delay-sharded x{world} (NCCL all_gather + all_reduce)" if delay
                                           else f"batch-sharded x{world} (weak)"),
                           "l2": "flushed between steps (256 MiB memset, outside the events)",
                           "timing": "CUDA-graph replay of graf_af_loss_grad per step, CUDA events",
                           "note": w["note"]},
                "roofline": roof, "cpu_baseline": cpu,
                "e2e": {"value": e2e_value, "unit": "surfaces/s", "h2d_bytes_per_step": B * N * 8,
                        "d2h_bytes_per_step": (B * N * 8 + B * 8) if args.mode != "forward" else
                        B * M * (8 if out == "c64" else 4),
                        "path": ("pinned host s -> H2D -> graf.af_loss_grad (C ABI) -> D2H loss + grad"
                                 if args.mode != "forward" else
                                 "pinned host s -> H2D -> graf.af_forward (C ABI) -> D2H zero-delay cut")},
                "gpu_launches": ((w["launches"] + 1) if delay else launches_per_step) * args.steps,
                "clocks": clocks}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def run_lpi(args):
    """The paper's section-7 experiment on the GPU: Eq. 26
    L = PSL + lambda*alpha*SV on N = 256 phase codes (periodic surface, PSL over the
    plane minus the origin, alpha = 2000), Adam lr 0.01, 2000 iterations,
    for a batch of 8 lambdas x 4 seeds.  A step = one optimisation iteration of the
    whole batch (pass 1 + argmax subgradient + spectral variance + Adam); the value is
    iterations/s.  Context (not a target): the paper reports ~67 s for the 2000
    iterations of one lambda on a laptop CPU."""
    import torch
    import paper_2506_22935_b200 as graf
    from graf_inputs import SplitMix64, random_phase
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    N, lams, seeds, iters = 256, np.linspace(0.1, 2.0, 8), 4, 2000
    B = len(lams) * seeds
    th0 = np.stack([np.angle(random_phase(SplitMix64(10_000 + rank * B + b), N)) for b in range(B)])
    lam = np.repeat(lams, seeds)
    opt = graf.LpiOptimizer(torch.tensor(th0, dtype=torch.float32, device=dev), torch.tensor(lam), per_graph=50)
    W = max(3, args.warmup)
    opt.run(1 + 50 * W)                                  # capture + warm-up replays
    sampler = ClockSampler(local if "CUDA_VISIBLE_DEVICES" not in os.environ else 0)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = args.steps * 50                                  # timed iterations (whole graphs of 50)
    a.record(opt.stream)
    opt.run(K)
    b.record(opt.stream)
    b.synchronize()
    ms = a.elapsed_time(b)
    clocks = sampler.stop()
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = t.item()
    # full 2000-iteration run from a fresh start (the paper's experiment), device-timed
    opt2 = graf.LpiOptimizer(torch.tensor(th0, dtype=torch.float32, device=dev), torch.tensor(lam), per_graph=50)
    opt2.run(1)
    a.record(opt2.stream)
    loss = opt2.run(iters - 1)
    b.record(opt2.stream)
    b.synchronize()
    full_ms = a.elapsed_time(b)
    per_it = ms / K
    if rank == 0:
        line = {"metric": "section-7 LPI optimisation iterations/sec (batch of 32 waveforms)",
                "value": 1e3 / per_it, "unit": "iterations/s", "n_gpus": world, "steps": args.steps,
                "warmup": W, "ms_per_step": per_it, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": "Eq. 26 PSL + lambda*2000*SV, N=256 periodic, Adam lr 0.01; "
                                       "8 lambdas x 4 seeds per GPU", "B_per_gpu": B, "N": N,
                           "waveform_iterations_per_s": B * 1e3 / per_it,
                           "full_2000_iterations_ms": full_ms,
                           "final_loss_median": float(np.median(loss.cpu().numpy())),
                           "paper_context": "~67 s for 2000 iterations of one lambda on an i7-1165G7 CPU (P:L434)",
                           "timing": "CUDA-graph replays of 50 iterations, CUDA events on the optimiser stream"},
                "roofline": None, "cpu_baseline": None,
                "e2e": None, "gpu_launches": 5 * K, "clocks": clocks}
        print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()


def run_mlw(args):
    """Differentiable mainlobe width W = sum |tau| sigma(gamma (chi(tau,0) - chi(0,0)/2)) and
    its gradient on the c2 batch (B = 256, N = 256): a step = one
    graf_mainlobe_width call (O(N^2) direct zero-Doppler cut per waveform)."""
    import torch
    import paper_2506_22935_b200 as graf
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    B, N = 256, 256
    s = torch.from_numpy(config_waveforms(2, batch=B)).to(dev)
    loss = torch.empty(B, dtype=torch.float64, device=dev)
    grad = torch.empty((B, N), dtype=torch.complex64, device=dev)
    gam = 4.0 / float(N) ** 2
    st = torch.cuda.Stream(dev)
    with torch.cuda.stream(st):
        graf.mainlobe_width(s, gam, loss=loss, grad=grad, stream=st)
        g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        graf.mainlobe_width(s, gam, loss=loss, grad=grad, stream=st)
    W = max(3, args.warmup)
    with torch.cuda.stream(st):
        for _ in range(W):
            g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        a.record(st)
        for _ in range(args.steps):
            g.replay()
        b.record(st)
    b.synchronize()
    ms = a.elapsed_time(b) / args.steps
    print(json.dumps({"metric": "mainlobe-width loss+grad surfaces/sec", "value": B / (ms / 1e3),
                      "unit": "surfaces/s", "n_gpus": 1, "steps": args.steps, "warmup": W, "ms_per_step": ms,
                      "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                      "data": "synthetic", "config": {"workload": "c2 batch, W over the zero-Doppler cut, "
                                                                  "gamma = 4/N^2", "B": B, "N": N},
                      "roofline": None, "cpu_baseline": None, "e2e": None, "gpu_launches": args.steps}))


class TimedBackend:
    """sharding backend that brackets each ABI call's delay-row kernels with events."""

    def __init__(self, graf, sharding):
        import torch
        self.inner = sharding.GrafBackend()
        self.L = graf.lib()
        self.ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        for e in self.ev:
            e.record()
        torch.cuda.synchronize()

    def _timed(self, i, fn, *a):
        self.L.graf_set_profile_events(ctypes_ptr(self.ev[2 * i]), ctypes_ptr(self.ev[2 * i + 1]))
        try:
            return fn(*a)
        finally:
            self.L.graf_set_profile_events(None, None)

    def forward_partials(self, *a):
        return self._timed(0, self.inner.forward_partials, *a)

    def loss_grad(self, *a):
        return self._timed(1, self.inner.loss_grad, *a)

    def combine(self, *a):
        return self.inner.combine(*a)

    # delay-sharded single pass (full-plane soft-PSL, c5): phase 1 holds the row kernels
    def single_pass_eligible(self, *a):
        return self.inner.single_pass_eligible(*a)

    def sp_begin(self, *a):
        return self._timed(0, self.inner.sp_begin, *a)

    def sp_end(self, *a):
        return self.inner.sp_end(*a)

    def kernel_ms(self):
        return self.ev[0].elapsed_time(self.ev[1]) + self.ev[2].elapsed_time(self.ev[3])


def ctypes_ptr(ev):
    import ctypes
    return ctypes.c_void_p(ev.cuda_event)


def ctypes_null():
    return None


if __name__ == "__main__":
    main()
