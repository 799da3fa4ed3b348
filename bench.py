#!/usr/bin/env python
"""bench.py — GRAF ambiguity-function hot path on B200 (BASELINE.json metric:
"AF forward+loss+grad surfaces/sec (N x M cells/s) and % of HBM/FP32 roofline").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl graf|reference]

A step = one forward + loss + gradient pass of the whole hot path (SURVEY.md §8(a)
rows a0-a7, plus a8 when sharded) over one batch of seeded synthetic waveforms of the
chosen BASELINE.json config, called through the C ABI (graf_af_loss_grad).  Default:
configs[4] = c5 (B = 8, N = M = 16384, full-plane ISL + soft-PSL T = 0.01), the largest
configuration and the one the north star's fused-loss FP32 target names; c1..c4 are
behind --config.  Inputs are resident in HBM before timing; each timed step is a
CUDA-graph replay of that call (eager ABI calls for the NCCL delay-sharded step), timed
with CUDA events on the launching stream, with L2 flushed (256 MiB memset) between steps
outside the events.  The dominant kernel's duration is read from events the ABI records
around its delay-row kernels, in the SAME replays.

Multi-GPU (one process per GPU, torchrun; `--gpus N` without torchrun re-launches itself
under torch.distributed.run), SURVEY.md §8(e):
  c5      delay sharding: every rank runs its folded rows k = r (mod G) of all 8 waveforms,
          all_gather of B x 48 B partials + all_reduce of the B x N gradient (NCCL);
  c2-c4   batch sharding: B/G contiguous waveforms per rank, no collective;
  c1      replicas (one 64-sample waveform does not shard).
Time = max over ranks; value = waveforms of the whole job / time.

`--impl reference`: the paper ships no code; the reference arm is the float64 CPU oracle
(oracle/), timed on the host cores on a bounded sample of the same workload.
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

SM_COUNT, SM_MAX_MHZ = 148, 1965.0      # B200_PROFILING.md; the bench reads the live values when it can
FP32_PEAK_TFLOPS = SM_COUNT * 128 * 2 * SM_MAX_MHZ * 1e6 / 1e12   # 74.4: 128 FP32 lanes/SM x FFMA


def fft_stage_flops(M: int) -> float:
    """Nominal flops of one radix-2 stage of a length-M FFT (5 M log2 M per
    FFT = 5 M per stage)."""
    return 5.0 * M


def workload(cid: int) -> dict:
    """The config's step and its algorithmic work (SURVEY.md §8(d) counting rules)."""
    cfg = CONFIGS[cid]
    loss = dict(cfg["loss"])
    note = ""
    if cid in (1, 3):
        # DESIGN.md R12: normalised full-plane ISL is identically M-1 with a zero
        # gradient (volume identity); time the raw mode, whose gradient is real work.
        loss["normalize"] = 0
        note = "raw (unnormalised) full-plane ISL: the normalised one is constant (volume identity)"
    N, M, B = cfg["N"], cfg["M"], cfg["B"]
    L2M = int(math.log2(M))
    rows = min(loss["k_max"], N - 1) + 1                       # folded delay rows k >= 0
    stages = 2 * L2M                                           # fused ISL: forward + inverse FFT
    count = "2 FFTs per folded row (forward + inverse)"
    single = False
    if loss["lambda_psl"] != 0 and not cfg["surface"]:
        nband = 2 * min(loss["d_max"], M // 2) + 1
        full = (min(loss["k_max"], N - 1) == N - 1 and loss["d_max"] >= M // 2 and loss.get("ml_k", 0) == 0
                and loss.get("ml_d", 0) == 0 and loss.get("normalize", 1) == 1)
        if full:
            # full-plane centred soft-PSL (R13): ONE pass of forward + inverse FFT per row
            # (the guarded fallback passes exit at once for waveforms inside the rule)
            single = True
            note = "full-plane soft-PSL as one optimistic pass (R13), per-waveform guarded fallback"
        elif nband <= M // 4 and B * rows * nband * 8 <= (1 << 30):
            # band cache: pass 2 reuses pass 1's in-band FFT outputs, so a row runs pass 1's
            # forward FFT and pass 2's inverse.  Both are PRUNED to the band (§8(d): count the
            # pruned FFT): pass 1's last radix-2 stage keeps 2 of E = 16 outputs per thread
            # (1/8 of the stage) and its first stage has a zero upper half (2N <= M); pass 2's
            # first radix-16 pass has 2 nonzero inputs of 16 (its 4 stages cost ~1).
            stages = (L2M - 1 - 7.0 / 8.0) + (L2M - 3)
            count = (f"pruned: pass-1 forward {L2M - 1 - 7 / 8:.3f} + pass-2 inverse {L2M - 3} of "
                     f"{L2M} radix-2 stages (band cache, 2N <= M, band < M/E)")
            note = "soft-PSL two-pass with the band cache: pass 2 reuses pass 1's in-band FFT outputs"
        else:
            stages = 3 * L2M
            count = "3 FFTs per folded row (pass 1 forward; pass 2 forward + inverse)"
    flops = B * rows * stages * fft_stage_flops(M)
    surf_bytes = 0
    if cfg["surface"]:
        per = 8 if cfg["surface"] == "c64" else 4
        surf_bytes = B * (2 * N - 1) * M * per
    io_bytes = B * N * 8 * 2
    return dict(cid=cid, cfg=cfg, loss=loss, N=N, M=M, B=B, rows=rows, stages=stages, flops=flops,
                flop_count=count, single=single, surf_bytes=surf_bytes, io_bytes=io_bytes, note=note,
                launches=(2 if loss["lambda_psl"] == 0 else 4))


def describe(w: dict) -> str:
    c = w["cfg"]
    L = w["loss"]
    return (f"{c['name']}: B={w['B']} N={w['N']} M={w['M']} {c['family']}; "
            f"{'surface ' + c['surface'] + ' + ' if c['surface'] else ''}"
            f"ISL x{L['lambda_isl']} + softPSL x{L['lambda_psl']} (T={L['temperature']}) on |k|<={L['k_max']}, "
            f"|d|<={L['d_max']} minus |k|<={L['ml_k']}&|d|<={L['ml_d']}, normalize={L['normalize']}")


def rank_plan(w: dict, world: int, rank: int, mode: str = "loss_grad") -> dict:
    """Which waveforms / rows this rank processes and how the job's
    throughput is counted."""
    B = w["B"]
    if world == 1:
        return dict(kind="single", b0=0, B_local=B, units=B, scaling="strong", shard=(0, 1),
                    parallelism="1 GPU")
    if w["cid"] == 5 and mode == "loss_grad":
        return dict(kind="delay", b0=0, B_local=B, units=B, scaling="strong", shard=(rank, world),
                    parallelism=f"delay-sharded x{world} (rows k = r mod {world}; NCCL all_gather + all_reduce)")
    if B >= world:
        base, rem = divmod(B, world)
        b0 = rank * base + min(rank, rem)
        return dict(kind="batch", b0=b0, B_local=base + (1 if rank < rem else 0), units=B, scaling="strong",
                    shard=(0, 1), parallelism=f"batch-sharded x{world} (B/G contiguous waveforms per rank)")
    return dict(kind="replica", b0=0, B_local=B, units=B * world, scaling="weak", shard=(0, 1),
                parallelism=f"replicas x{world} (B = {B} does not shard)")


def max_over_ranks(values, dev, world):
    """Element-wise max over ranks (device-timed numbers: the slowest rank decides)."""
    if world == 1:
        return list(values)
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(values), dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


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


def host_info() -> dict:
    try:
        from threadpoolctl import threadpool_info
        threads = max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        threads = os.cpu_count()
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cores": threads, "nproc": os.cpu_count(), "cpu_model": model}


# ---------------------------------------------------------------------------
def oracle_sample(w: dict, i: int):
    """One bounded sample of the workload through the float64 oracle, as it stands.
    Returns the fraction of a waveform's work it covered.  Waveforms whose direct sum
    takes minutes (N*M > 4096*8192: c5) are sampled by CELLS: the oracle's loss_and_grad
    over the delay rows |k| <= 63 and centred Doppler bins |d| <= 1023 of waveform i
    (forward sum, loss terms and adjoint for those cells; its cost per cell is one
    length-N dot product each way, the same for every cell of the plane)."""
    from oracle import graf_oracle as O
    spec = O.LossSpec.from_dict(w["loss"])
    N, M = w["N"], w["M"]
    s = config_waveforms(w["cid"], batch=1, start=i % w["B"])[0]
    if N * M > 4096 * 8192:
        sub = O.LossSpec.from_dict(dict(w["loss"], k_max=63, d_max=1023))
        O.loss_and_grad(s, M, sub)
        return (127 * 2047) / ((2 * N - 1) * M)
    if w.get("match"):
        tgt = np.random.default_rng(i).random((2 * N - 1, M)) / M
        O.match_loss_and_grad(s, M, spec, tgt, -(N - 1), "centered")
    elif w.get("cross"):
        s2 = config_waveforms(w["cid"], batch=1, start=(i + 777) % w["B"])[0]
        O.cross_loss_and_grad(s, s2, M, spec)
    else:
        per = w.get("periodic", False)
        O.loss_and_grad(s, M, spec, periodic=per)
        if w["cfg"]["surface"]:
            O.surface(s, M, w["cfg"]["surface"], "centered", periodic=per,
                      **(dict(k_begin=-(N // 2), k_end=N // 2) if per else {}))
    return 1.0


def sample_label(w: dict) -> str:
    if w["N"] * w["M"] > 4096 * 8192:
        return ("cells |k|<=63 x |d|<=1023 (127 x 2047 of 32767 x 16384) of c5 waveforms, forward + loss + "
                "adjoint by direct float64 sums")
    return f"whole {w['cfg']['name']} waveforms, forward + loss + adjoint by direct float64 sums"


def cpu_baseline(w: dict, budget_s: float = 15.0) -> dict:
    """The float64 oracle as it stands, on the host cores, on a bounded sample."""
    done, t0, i = 0.0, time.perf_counter(), 0
    while True:
        done += oracle_sample(w, i)
        i += 1
        el = time.perf_counter() - t0
        if el > budget_s or i >= w["B"] * (1 if done >= i else 50):
            break
    hi = host_info()
    return {"value": done / el, "unit": "surfaces/s", "cores": hi["cores"], "kind": "oracle",
            "sample": f"{i} samples = {done:.4g} waveforms in {el:.1f} s: {sample_label(w)}",
            "nproc": hi["nproc"], "cpu_model": hi["cpu_model"]}


def run_reference(args, w) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    per_step = {1: 1, 2: 8, 3: 1, 4: 1, 5: 4}[w["cid"]]

    def step(i):
        d = 0.0
        for j in range(per_step):
            d += oracle_sample(w, i * per_step + j)
        return d

    for i in range(args.warmup):
        step(i)
    t0 = time.perf_counter()
    done = 0.0
    for i in range(args.steps):
        done += step(args.warmup + i)
    el = time.perf_counter() - t0
    v = done / el
    hi = host_info()
    line = {"metric": "AF forward+loss+grad surfaces/sec", "value": v, "unit": "surfaces/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": describe(w), "sample_per_step": f"{per_step} samples: {sample_label(w)}"},
            "cpu_baseline": {"value": v, "unit": "surfaces/s", "cores": hi["cores"], "kind": "oracle",
                             "sample": f"{per_step} samples per step x {args.steps} steps = {done:.4g} waveforms: "
                                       f"{sample_label(w)}", "cpu_model": hi["cpu_model"]},
            "e2e": {"value": v, "unit": "surfaces/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def relaunch_under_torchrun(n: int) -> None:
    """`--gpus N` outside torchrun: re-run this command as N ranks (127.0.0.1 rendezvous)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    raise SystemExit(subprocess.call(cmd))


def measure_fp32_peak(graf, dev, stream) -> dict:
    """FFMA-bound probe kernel (graf_probe_fp32), CUDA events, best of 5, clocks alongside."""
    import ctypes
    import torch
    L = graf.lib()
    scratch = torch.empty(4 * 256 * 1024, dtype=torch.float32, device=dev)
    fl = ctypes.c_double(0.0)
    best = 0.0
    with torch.cuda.stream(stream):
        for it in range(6):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            graf.graf.L.check(L.graf_probe_fp32(ctypes.c_void_p(scratch.data_ptr()), 4096, ctypes.byref(fl),
                                                ctypes.c_void_p(stream.cuda_stream)))
            b.record(stream)
            b.synchronize()
            if it:
                best = max(best, fl.value / (a.elapsed_time(b) / 1e3) / 1e12)
    return {"tflops": best, "how": "graf_probe_fp32: 8 FFMA chains/thread, 4 x 256-thread CTAs per SM, best of 5"}


# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=5, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="graf", choices=["graf", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--settle-s", type=float, default=1.0)
    ap.add_argument("--mode", default="loss_grad", choices=["loss_grad", "forward", "lpi", "match", "cross", "mlw"],
                    help="forward: full-surface mode (graf_af_forward writes the config's surface, no loss)")
    ap.add_argument("--periodic", action="store_true",
                    help="the paper's circular surface (Eq. 2 / Alg. 1, SURVEY 8(f) NEXT-1); needs M == N")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus != world:
        if world == 1 and args.gpus > 1 and "RANK" not in os.environ:
            relaunch_under_torchrun(args.gpus)
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE = {world}")
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
        w["flops"] = w["B"] * w["rows"] * w["stages"] * fft_stage_flops(w["M"])
        if w["cfg"]["surface"]:
            w["surf_bytes"] = w["B"] * w["N"] * w["M"] * (8 if w["cfg"]["surface"] == "c64" else 4)
        w["note"] = (w["note"] + "; " if w["note"] else "") + "periodic (circular) surface, paper Eq. 2 / Alg. 1"
    if args.mode == "forward":
        if not w["cfg"]["surface"]:
            raise SystemExit("--mode forward needs a config with a surface (c1, c3)")
        # folded rows covering the whole surface window, one forward FFT each
        w["flops"] = w["B"] * (w["N"] // 2 + 1 if args.periodic else w["N"]) * 5.0 * w["M"] * math.log2(w["M"])
        w["flop_count"] = "1 forward FFT per folded row"
        w["io_bytes"] = w["B"] * w["N"] * 8
        w["launches"] = 1
        w["note"] = "full-surface mode: graf_af_forward writes the surface; no loss or gradient"
    if args.mode == "match":
        # match loss ||x - x_target||^2 over the config's region (NEXT-3): one fused
        # pass streaming a per-waveform fp32 target of the full surface window
        w["loss"] = dict(w["loss"], lambda_isl=0.0, lambda_psl=0.0, normalize=1)
        w["match"] = True
        w["rows"] = min(w["loss"]["k_max"], w["N"] - 1) + 1
        w["flops"] = w["B"] * w["rows"] * 2 * 5.0 * w["M"] * math.log2(w["M"])
        w["flop_count"] = "2 FFTs per folded row (forward + inverse)"
        # algorithmic bytes: s + g + the target cells of the region (both mirrored rows)
        w["surf_bytes"] = w["B"] * (2 * w["rows"] - 1) * min(w["M"], 2 * w["loss"]["d_max"] + 1) * 4
        w["launches"] = 2
        w["note"] = "match loss over the region, per-waveform fp32 target of the surface window (HBM-streamed)"
    if args.mode == "cross":
        # cross-ambiguity of waveform pairs (NEXT-4): the config's loss on
        # X = sum s1 conj(s2(n-k)) W^{mn}, rows unfolded (no mirror symmetry)
        w["cross"] = True
        w["rows"] = 2 * min(w["loss"]["k_max"], w["N"] - 1) + 1
        w["flops"] = w["B"] * w["rows"] * w["stages"] * fft_stage_flops(w["M"])
        w["io_bytes"] = w["B"] * w["N"] * 8 * 4
        w["note"] = "cross-ambiguity of (s1, s2) pairs, unfolded rows; loss/grad w.r.t. both"
    if args.impl == "reference":
        return run_reference(args, w)
    run_graf(args, w, world)


def run_graf(args, w, world):
    import ctypes
    import torch
    import torch.distributed as dist

    import paper_2506_22935_b200 as graf

    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hooks (tests/test_gpu_bench_multirank.py): the multi-rank path exercised on ONE GPU
    # with gloo collectives; the driver's runs use NCCL, one GPU per rank
    backend = os.environ.get("GRAF_BENCH_DIST_BACKEND", "nccl")
    if os.environ.get("GRAF_BENCH_ONE_GPU"):
        local = 0
    if world > 1:
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    W = max(3, args.warmup)
    plan = rank_plan(w, world, rank, args.mode)
    delay = plan["kind"] == "delay"

    N, M = w["N"], w["M"]
    B = plan["B_local"]                                   # waveforms this rank processes
    s_host = torch.from_numpy(config_waveforms(w["cid"], batch=B, start=plan["b0"])).pin_memory()
    s = s_host.to(dev)
    spec = graf.LossSpec.from_dict(w["loss"])
    out = w["cfg"]["surface"]
    if w.get("match"):
        out = None
        spec.lambda_match = 1.0
        g_ = torch.Generator(device=dev)
        g_.manual_seed(1234 + plan["b0"])
        spec.target = torch.rand((B, 2 * N - 1, M), generator=g_, device=dev) * (1.0 / M)
    if w.get("cross"):
        s2_host = torch.from_numpy(config_waveforms(w["cid"], batch=B, start=plan["b0"] + 777)).pin_memory()
        s2 = s2_host.to(dev)
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
    L = graf.lib()
    graf.graf.L.check(L.graf_init(ctypes.c_void_p(stream.cuda_stream)))
    if delay:
        from paper_2506_22935_b200 import sharding
        tb = TimedBackend(graf, sharding)

    def call(st, sd=None):
        sd = s if sd is None else sd
        if w.get("cross"):
            return graf.xaf_loss_grad(sd, s2, M, spec, ws=ws, stream=st)
        if delay:
            return sharding.delay_sharded_loss_grad(sd, M, spec, backend=tb)
        if args.mode == "forward":
            return graf.af_forward(sd, M, out=out, layout="centered", ws=ws, surface=surf, stream=st, **kb)
        return graf.af_loss_grad(sd, M, spec, out=out, layout="centered", ws=ws, grad=grad, loss_out=loss_out,
                                 surface=surf, stream=st, **kb)

    with torch.cuda.stream(stream):
        call(stream)                                    # workspace + attributes, before capture
        call(stream)
    torch.cuda.synchronize()
    launches_per_step = int(L.graf_last_launch_count())   # device ops one ABI call enqueues
    ev_k0, ev_k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev_k0.record(stream)        # torch creates the CUDA events lazily on first record
    ev_k1.record(stream)
    torch.cuda.synchronize()
    if delay:
        class _Eager:                     # NCCL step: eager ABI calls (no host sync inside)
            def replay(self_inner):
                call(stream)
        g = _Eager()
    else:
        # g: the timed step.  g_k: the same call with the ABI recording ev_k0 / ev_k1 (external
        # event nodes) around its delay-row kernels.  The event nodes cost a few microseconds,
        # which matters on the latency-bound configs, so the step is timed on g and the kernel
        # window on g_k, replayed alternately under the same flush protocol; share_of_step is
        # the kernel window over g_k's own step.
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            call(stream)
        g_k = torch.cuda.CUDAGraph()
        L.graf_set_profile_events(ctypes.c_void_p(ev_k0.cuda_event), ctypes.c_void_p(ev_k1.cuda_event))
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
            for _ in range(5 if w["cid"] in (3, 5) else 20):
                g.replay()
            stream.synchronize()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms, kern_ms, inst_ms = [], [], []
    with torch.cuda.stream(stream):
        for i in range(args.steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            g.replay()
            b.record(stream)
            b.synchronize()
            step_ms.append(a.elapsed_time(b))
            if delay:
                kern_ms.append(tb.kernel_ms())
                inst_ms.append(step_ms[-1])
                continue
            flush.zero_()
            a2, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a2.record(stream)
            g_k.replay()
            b2.record(stream)
            b2.synchronize()
            kern_ms.append(ev_k0.elapsed_time(ev_k1))
            inst_ms.append(a2.elapsed_time(b2))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    total_ms, kern_avg, inst_avg = max_over_ranks([sum(step_ms), sum(kern_ms) / len(kern_ms),
                                                   sum(inst_ms) / len(inst_ms)], dev, world)
    ms_per_step = total_ms / args.steps
    value = plan["units"] * args.steps / (total_ms / 1e3)

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
            if args.mode == "forward":
                sf, _ = call(stream, s_dev2)
                zrow = sf[:, N // 2 if args.periodic else N - 1, :]   # zero-delay cut of every surface
                if zrow_host is None:
                    zrow_host = torch.empty(zrow.shape, dtype=zrow.dtype).pin_memory()
                zrow_host.copy_(zrow, non_blocking=True)
            else:
                r = call(stream, s_dev2)
                lo, gr = r[0], r[1]
                l_host.copy_(lo, non_blocking=True)
                g_host.copy_(gr, non_blocking=True)
            b_.record(stream)
            b_.synchronize()
            if i >= W:
                e2e_ms.append(a.elapsed_time(b_))
    e2e_total = max_over_ranks([sum(e2e_ms)], dev, world)[0]
    e2e_value = plan["units"] * len(e2e_ms) / (e2e_total / 1e3)

    # ---- roofline of the dominant kernel(s) (af_rows_kernel), per launch window
    t_k = kern_avg / 1e3
    flops_k = w["flops"] * B / w["B"] / (world if delay else 1)     # this rank's rows / waveforms
    fl_tf = flops_k / t_k / 1e12
    try:
        hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
        hbm_src = "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    except Exception:
        hbm, hbm_src = 6533.8, "fallback: round-1 MEASURED_PEAKS.json hbm_gbs"
    bytes_k = (w["surf_bytes"] + w["io_bytes"]) * B / w["B"]
    t_alu = flops_k / (FP32_PEAK_TFLOPS * 1e12)
    t_hbm = bytes_k / (hbm * 1e9)
    fp32_meas = measure_fp32_peak(graf, dev, stream) if rank == 0 else None
    if t_hbm > t_alu:
        roof = {"bound": "hbm", "achieved": bytes_k / t_k / 1e9, "peak": hbm, "unit": "GB/s",
                "frac": bytes_k / t_k / 1e9 / hbm, "peak_source": hbm_src}
    else:
        roof = {"bound": "alu", "achieved": fl_tf, "peak": round(FP32_PEAK_TFLOPS, 2), "unit": "TFLOP/s",
                "frac": fl_tf / FP32_PEAK_TFLOPS,
                "peak_source": "derived (DESIGN.md §5): 148 SMs x 128 FP32 lanes x 2 flop (FFMA) x 1965 MHz",
                "flop_count": w["flop_count"]}
        if w["loss"]["lambda_psl"] != 0 and args.mode == "loss_grad" and not args.periodic:
            # SURVEY.md §8(d)'s nominal count for a soft-PSL loss: 3 FFT passes per folded row
            # (pass 1 forward; pass 2 forward + inverse), whatever the build executes
            sv_flops = w["B"] * w["rows"] * 3 * 5.0 * w["M"] * math.log2(w["M"]) * (B / w["B"]) / (world if delay else 1)
            roof["survey_3pass_flops_per_launch"] = sv_flops
            roof["frac_survey_3pass"] = sv_flops / t_k / 1e12 / FP32_PEAK_TFLOPS
        if fp32_meas:
            roof["peak_measured"] = round(fp32_meas["tflops"], 2)
            roof["frac_of_measured"] = fl_tf / fp32_meas["tflops"]
            roof["peak_measured_how"] = fp32_meas["how"]
    roof["traffic"] = read_traffic(f"{w['cid']}{'fwd' if args.mode == 'forward' else ''}"
                                   f"{'per' if args.periodic else ''}{args.mode if args.mode in ('match', 'cross') else ''}")
    two_pass = " (single pass + guarded fallback)" if w.get("single") else " (pass 1 + reduce + pass 2)"
    roof["kernel"] = (f"af_rows_kernel<{M}>" + (two_pass if w["loss"]["lambda_psl"] else "")
                      + (" with the fused cluster finalize" if launches_per_step == 1 and args.mode != "forward"
                         else ""))
    roof["kernel_ms"] = kern_avg
    roof["algorithmic_flops_per_launch"] = flops_k
    roof["algorithmic_bytes_per_launch"] = bytes_k
    roof["share_of_step"] = kern_avg / inst_avg
    roof["instrumented_step_ms"] = inst_avg
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(w)
    if rank == 0:
        line = {"metric": ("AF forward+loss+grad surfaces/sec" if args.mode != "forward"
                           else "AF forward (full-surface) surfaces/sec"), "value": value, "unit": "surfaces/s",
                "n_gpus": world, "steps": args.steps, "warmup": W, "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": plan["scaling"], "vs_baseline": None,
                "dtype": "f32",
                "data": "synthetic",
                "config": {"workload": describe(w), "B": w["B"], "B_per_gpu": B, "N": N, "M": M,
                           "cells_per_s": value * N * M,
                           "parallelism": plan["parallelism"],
                           "l2": "flushed between steps (256 MiB memset, outside the events)",
                           "timing": ("eager ABI calls per step (NCCL delay sharding), CUDA events; kernel window "
                                      "from events around the ABI's row kernels in the same steps" if delay else
                                      "CUDA-graph replay of the ABI call per step, CUDA events; the kernel window "
                                      "from a second graph of the same call with event nodes around its row "
                                      "kernels, replayed alternately with the timed one"),
                           "note": w["note"]},
                "roofline": roof, "cpu_baseline": cpu,
                "e2e": {"value": e2e_value, "unit": "surfaces/s", "h2d_bytes_per_step": B * N * 8,
                        "d2h_bytes_per_step": (B * N * 8 + B * 8) if args.mode != "forward" else
                        B * M * (8 if out == "c64" else 4),
                        "path": ("pinned host s -> H2D -> graf.af_loss_grad (C ABI) -> D2H loss + grad"
                                 if args.mode != "forward" else
                                 "pinned host s -> H2D -> graf.af_forward (C ABI) -> D2H zero-delay cut")},
                "gpu_launches": (tb.launches if delay else launches_per_step) * args.steps,
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
    """sharding backend that brackets each ABI call's delay-row kernels with events and
    counts the device operations the ABI enqueues per step."""

    def __init__(self, graf, sharding):
        import torch
        self.inner = sharding.GrafBackend()
        self.L = graf.lib()
        self.ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        for e in self.ev:
            e.record()
        torch.cuda.synchronize()
        self.launches = 0
        self._n = 0
        self._used, self.used = set(), set()

    def _timed(self, i, fn, *a, **kw):
        self._used.add(i)
        self.L.graf_set_profile_events(ctypes_ptr(self.ev[2 * i]), ctypes_ptr(self.ev[2 * i + 1]))
        try:
            return fn(*a, **kw)
        finally:
            self.L.graf_set_profile_events(None, None)
            self._count()

    def _count(self):
        self._n += int(self.L.graf_last_launch_count())

    def forward_partials(self, *a, **kw):
        return self._timed(1, self.inner.forward_partials, *a, **kw)

    def loss_grad(self, *a, **kw):
        r = self._timed(2, self.inner.loss_grad, *a, **kw)
        self.launches, self._n = self._n, 0          # loss_grad closes a step
        self.used, self._used = self._used, set()
        return r

    def combine(self, *a):
        r = self.inner.combine(*a)
        self._count()
        return r

    # delay-sharded single pass (full-plane soft-PSL, c5): phase 1 holds the row kernels
    def single_pass_eligible(self, *a):
        return self.inner.single_pass_eligible(*a)

    def sp_begin(self, *a):
        return self._timed(0, self.inner.sp_begin, *a)

    def sp_end(self, *a):
        r = self.inner.sp_end(*a)
        self._count()
        return r

    def kernel_ms(self):
        return sum(self.ev[2 * i].elapsed_time(self.ev[2 * i + 1]) for i in sorted(self.used))


def ctypes_ptr(ev):
    import ctypes
    return ctypes.c_void_p(ev.cuda_event)


if __name__ == "__main__":
    main()
