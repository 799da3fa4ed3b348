"""The multi-rank paths on ONE GPU (the pool gives one GPU per call): two processes share
cuda:0 and talk through gloo, so the code the 8-GPU runs execute — sharding.py's delay
sharding with the device-side fallback of the single pass, and bench.py's per-rank plans,
timing reduction and JSON line — runs with the real kernels.  NCCL itself is not exercised
(it refuses two ranks on one device); nothing here waits inside a kernel on another rank.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

from gradtol import grad_tol

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def _port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _torchrun(args, env_extra, timeout=900):
    env = dict(os.environ, GRAF_BENCH_DIST_BACKEND="gloo", GRAF_BENCH_ONE_GPU="1", **env_extra)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), *args]
    return subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)


@pytest.mark.parametrize("config", [5, 2])
def test_bench_two_ranks_one_gpu(config):
    r = _torchrun(["bench.py", "--gpus", "2", "--config", str(config), "--steps", "2", "--warmup", "3",
                   "--no-cpu-baseline", "--settle-s", "0"], {})
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]          # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["roofline"]["kernel_ms"] > 0
    if config == 5:
        assert d["config"]["parallelism"].startswith("delay-sharded x2")
    else:
        assert d["config"]["parallelism"].startswith("batch-sharded x2") and d["config"]["B_per_gpu"] == 128


WORKER = r"""
import os, sys, json
sys.path.insert(0, %r)
import numpy as np, torch, torch.distributed as dist
torch.cuda.set_device(0)
dist.init_process_group("gloo")
from paper_2506_22935_b200 import sharding, LossSpec
from graf_inputs import SplitMix64, random_phase, lfm, CONFIGS
N = M = 1024
s = np.stack([random_phase(SplitMix64(8_500_000), N), lfm(N, 1.0).astype(np.complex64),
              random_phase(SplitMix64(8_500_001), N)])
spec = LossSpec.from_dict(dict(CONFIGS[5]["loss"], k_max=N - 1, d_max=M // 2))
loss, g = sharding.delay_sharded_loss_grad(torch.from_numpy(s).cuda(), M, spec)
torch.cuda.synchronize()
if dist.get_rank() == 0:
    np.save(os.environ["OUT"], np.concatenate([loss.cpu().numpy().astype(np.complex128), g.cpu().numpy().ravel()]))
dist.destroy_process_group()
"""


def test_delay_sharding_two_ranks_with_fallback(tmp_path):
    """delay_sharded_loss_grad over 2 ranks (gloo) on the c5-shaped full-plane loss, N = M =
    1024, with an LFM chirp (outside the R13 rule: recomputed by the masked two-pass
    fallback) between random codes: loss and gradient against the float64 oracle."""
    from graf_inputs import CONFIGS, SplitMix64, lfm, random_phase
    from oracle import graf_oracle as O
    script = tmp_path / "worker.py"
    script.write_text(WORKER % ROOT)
    out = tmp_path / "out.npy"
    r = _torchrun([str(script)], {"OUT": str(out)}, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    res = np.load(out)
    N = M = 1024
    loss, g = res[:3].real, res[3:].reshape(3, N)
    s = np.stack([random_phase(SplitMix64(8_500_000), N), lfm(N, 1.0).astype(np.complex64),
                  random_phase(SplitMix64(8_500_001), N)])
    spec_d = dict(CONFIGS[5]["loss"], k_max=N - 1, d_max=M // 2)
    for b in range(3):
        L_ref, g_ref, t = O.loss_and_grad(s[b], M, O.LossSpec.from_dict(spec_d))
        assert abs(loss[b] - L_ref) <= 1e-4 * abs(L_ref), (b, loss[b], L_ref)
        assert np.abs(g[b] - g_ref).max() <= grad_tol(g_ref, t["sigma_g"]), b
