#!/usr/bin/env python
"""Kernel-shape tuning harness (development tool, not part of the product path).

  python scripts/tune.py build <config> "<tag>:<defines>" ...   # here (CPU): nvcc variant libraries
  python scripts/tune.py run <config>                           # on the GPU box: time every variant

Each variant is libgraf.so compiled with -D overrides of the (E, S) table in
graf_kernels.cuh and -DGRAF_ONLY_M=<M>; `run` times graf_af_loss_grad on the
config's full batch (CUDA-graph replay, L2 flushed between steps) in a fresh
process per variant and checks it against the default library's output.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VDIR = os.path.join(ROOT, "paper_2506_22935_b200", "variants")   # in-tree: travels with gpurun


def build(cfg, specs):
    from graf_inputs import CONFIGS
    from paper_2506_22935_b200 import _build
    M = CONFIGS[cfg]["M"]
    os.makedirs(VDIR, exist_ok=True)
    srcs = [os.path.join(_build.CSRC, "graf_api.cu"), os.path.join(_build.CSRC, _build.ROW_UNIT_OF[M])]
    for spec in specs:
        tag, defs = spec.split(":", 1)
        out = os.path.join(VDIR, f"libgraf_c{cfg}_{tag}.so")
        try:
            _build.compile_link(out, srcs, defines=[f"GRAF_ONLY_M={M}"] + [d for d in defs.split(",") if d],
                                objdir=os.path.join("/tmp/graf_build", "variants", "obj_" + tag))
            print(tag, "rc 0")
        except Exception as e:   # noqa: BLE001
            print(tag, "failed", e)


def one(lib, cfg, steps=30):
    os.environ["GRAF_LIB_PATH"] = lib
    import torch
    import paper_2506_22935_b200 as graf
    from graf_inputs import CONFIGS, config_waveforms
    c = CONFIGS[cfg]
    spec = dict(c["loss"])
    if cfg in (1, 3):
        spec["normalize"] = 0
    spec = graf.LossSpec.from_dict(spec)
    s = torch.from_numpy(config_waveforms(cfg)).cuda()
    out = c["surface"]
    ws = graf.graf.Workspace()
    st = torch.cuda.Stream()
    B, N, M = c["B"], c["N"], c["M"]
    grad = torch.empty((B, N), dtype=torch.complex64, device="cuda")
    lo = torch.empty((B,), dtype=torch.float64, device="cuda")
    surf = None
    if out:
        surf = torch.empty((B, 2 * N - 1, M), dtype=torch.complex64 if out == "c64" else torch.float32,
                           device="cuda")

    fwd = os.environ.get("GRAF_TUNE_MODE") == "forward"

    def call():
        if fwd:
            graf.af_forward(s, M, out=out, layout="centered", ws=ws, surface=surf, stream=st)
        else:
            graf.af_loss_grad(s, M, spec, out=out, ws=ws, grad=grad, loss_out=lo, surface=surf, stream=st)

    with torch.cuda.stream(st):
        call()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        call()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    with torch.cuda.stream(st):
        for i in range(steps + 5):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            g.replay()
            b.record(st)
            b.synchronize()
            if i >= 5:
                ts.append(a.elapsed_time(b))
    ts.sort()
    chk = float(surf.float().abs().sum().item()) if (fwd and surf is not None) else None
    res = {"lib": os.path.basename(lib), "median_ms": ts[len(ts) // 2], "min_ms": ts[0], "surf_abs_sum": chk,
           "loss0": lo[0].item(), "gmax": grad.abs().max().item(), "g00": [grad[0, 0].real.item(), grad[0, 0].imag.item()]}
    print(json.dumps(res))


def run(cfg):
    libs = sorted(f for f in os.listdir(VDIR) if f.startswith(f"libgraf_c{cfg}_"))
    base = os.path.join(ROOT, "paper_2506_22935_b200", "libgraf.so")
    for lib in [base] + [os.path.join(VDIR, f) for f in libs]:
        r = subprocess.run([sys.executable, __file__, "one", lib, str(cfg)], capture_output=True, text=True, timeout=300)
        print(r.stdout.strip() or r.stderr.strip()[-400:], flush=True)


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "build":
        build(int(sys.argv[2]), sys.argv[3:])
    elif cmd == "run":
        run(int(sys.argv[2]))
    elif cmd == "one":
        one(sys.argv[2], int(sys.argv[3]))
