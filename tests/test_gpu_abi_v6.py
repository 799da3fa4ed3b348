"""ABI v6 behaviour on the GPU (include/graf.h): the per-waveform skip mask, shards that own
no loss rows, the delay-sharded single pass with its device-side fallback as sharding.py
runs it, and a first call made inside CUDA-graph capture (the twiddle table's fill is then
recorded into the graph; no host-blocking upload exists any more)."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from graf_inputs import CONFIGS, SplitMix64, complex_gaussian, lfm, random_phase
from oracle import graf_oracle as O

from gradtol import grad_tol

pytestmark = pytest.mark.gpu

graf = pytest.importorskip("paper_2506_22935_b200")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def cg(B, N, seed):
    return np.stack([complex_gaussian(SplitMix64(seed * 1000 + b), N) for b in range(B)])


SPECS = [
    dict(k_max=20, d_max=12, ml_k=0, ml_d=1, lambda_isl=1.0, lambda_psl=0.0, normalize=1),          # fused ISL
    dict(k_max=20, d_max=12, ml_k=0, ml_d=1, lambda_isl=0.5, lambda_psl=1.0, temperature=0.05, normalize=1),
    dict(k_max=200, d_max=128, lambda_isl=1.0, lambda_psl=1.0, temperature=0.01, normalize=1),   # full plane
]


@pytest.mark.parametrize("si", range(len(SPECS)))
@pytest.mark.parametrize("N,M", [(200, 256), (201, 8192), (300, 16384)])
def test_skip_mask_leaves_skipped_outputs_untouched(si, N, M):
    spec_d = dict(SPECS[si])
    if spec_d["k_max"] >= 200:
        spec_d.update(k_max=N - 1, d_max=M // 2)
    spec = graf.LossSpec.from_dict(spec_d)
    B = 4
    s = dev(cg(B, N, 40 + si))
    lo_ref, g_ref, _ = graf.af_loss_grad(s, M, spec)
    skip = torch.tensor([0, 1, 0, 1], dtype=torch.int32, device="cuda")
    lo = torch.full((B,), 123.5, dtype=torch.float64, device="cuda")
    g = torch.full((B, N), 7.0 + 3.0j, dtype=torch.complex64, device="cuda")
    graf.af_loss_grad(s, M, spec, loss_out=lo, grad=g, skip=skip)
    for b in range(B):
        if skip[b]:
            assert lo[b].item() == 123.5 and bool((g[b] == (7.0 + 3.0j)).all())
        else:
            assert torch.equal(lo[b], lo_ref[b]) and torch.equal(g[b], g_ref[b])   # bitwise (deterministic)
    # forward partials: skipped waveforms get identity partials
    _, parts = graf.af_forward(s, M, out=None, loss=spec, skip=skip)
    _, parts_ref = graf.af_forward(s, M, out=None, loss=spec)
    for b in range(B):
        if skip[b]:
            assert parts[b, 0].item() == 0.0 and parts[b, 1].item() == float("-inf")
        else:
            assert torch.equal(parts[b], parts_ref[b])


def test_rowless_shard():
    """k_max = 2 over 5 delay shards: shards 3 and 4 own no loss rows.  ISL-only: they return
    loss 0 and grad 0 and the sums over shards are the unsharded result; soft-PSL without
    `global` is rejected before any launch; with `global` every shard reports the full loss."""
    N, M, G = 64, 64, 5
    s = dev(cg(2, N, 9))
    isl = graf.LossSpec(k_max=2, d_max=8, ml_k=0, ml_d=1, lambda_isl=1.0)
    L1, g1, _ = graf.af_loss_grad(s, M, isl)
    Ls, gs = 0, 0
    for r in range(G):
        Lr, gr, _ = graf.af_loss_grad(s, M, isl, shard=(r, G))
        if r >= 3:
            assert float(Lr.abs().max()) == 0.0 and float(gr.abs().max()) == 0.0
        Ls, gs = Ls + Lr, gs + gr
    assert torch.allclose(Ls, L1, rtol=1e-6) and (gs - g1).abs().max().item() <= 1e-4 * g1.abs().max().item()
    soft = graf.LossSpec(k_max=2, d_max=8, ml_k=0, ml_d=1, lambda_isl=0.5, lambda_psl=1.0, temperature=0.05)
    with pytest.raises(graf.GrafError):
        graf.af_loss_grad(s, M, soft, shard=(4, G))
    parts = torch.stack([graf.af_forward(s, M, out=None, loss=soft, shard=(r, G))[1] for r in range(G)])
    glob = graf.combine_partials(soft, parts)
    L1s, _, _ = graf.af_loss_grad(s, M, soft)
    L4, g4, _ = graf.af_loss_grad(s, M, soft, global_partials=glob, shard=(4, G))
    assert torch.allclose(L4, L1s, rtol=1e-6) and float(g4.abs().max()) == 0.0


@pytest.mark.parametrize("N,M,G", [(256, 256, 2), (1000, 1024, 3), (300, 16384, 2)])
def test_sharded_single_pass_with_device_fallback(N, M, G):
    """sharding.py's flow on one GPU: single pass -> combine -> phase 2 (valid mask) -> the
    two-pass protocol with skip = valid -> sum over shards.  An LFM chirp (outside the R13
    rule: its ridge has x ~ 1) sits between random codes; every waveform must match the
    oracle, and the valid ones must equal the plain single pass bitwise."""
    s_np = np.stack([random_phase(SplitMix64(8_400_000), N), lfm(N, 1.0).astype(np.complex64),
                     random_phase(SplitMix64(8_400_001), N)])
    spec_d = dict(CONFIGS[5]["loss"], k_max=N - 1, d_max=M // 2)
    spec = graf.LossSpec.from_dict(spec_d)
    s = dev(s_np)
    ws = [graf.graf.Workspace() for _ in range(G)]
    parts = torch.stack([graf.af_loss_grad_sp_begin(s, M, spec, (r, G), ws=ws[r]) for r in range(G)])
    glob = graf.combine_partials(spec, parts)
    outs = [graf.af_loss_grad_sp_end(s, M, spec, (r, G), glob, ws=ws[r]) for r in range(G)]
    valid = outs[0][2]
    if N == M:
        assert valid.cpu().tolist() == [1, 0, 1]
    else:   # zero-padded Doppler: the mainlobe's neighbours (x ~ 0.4-1) put every waveform outside R13
        assert valid.cpu().tolist()[1] == 0
    skip = valid.to(torch.int32).contiguous()
    parts2 = torch.stack([graf.af_forward(s, M, out=None, loss=spec, shard=(r, G), skip=skip)[1] for r in range(G)])
    glob2 = graf.combine_partials(spec, parts2)
    g = 0
    for r in range(G):
        lo, gr, _ = graf.af_loss_grad(s, M, spec, global_partials=glob2, shard=(r, G), skip=skip,
                                      loss_out=outs[r][0], grad=outs[r][1])
        g = g + gr
    ospec = O.LossSpec.from_dict(spec_d)
    for b in range(3):
        L_ref, g_ref, t = O.loss_and_grad(s_np[b], M, ospec)
        assert abs(outs[0][0][b].item() - L_ref) <= 1e-4 * abs(L_ref), b
        tol = grad_tol(g_ref, t["sigma_g"])
        assert np.abs(g[b].cpu().numpy() - g_ref).max() <= tol, b


def test_first_call_inside_graph_capture():
    """A fresh process whose FIRST library call is inside torch.cuda.graph capture: the twiddle
    fill is captured with it; two replays give the oracle's answer."""
    code = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_2506_22935_b200 as graf
from graf_inputs import config_waveforms, CONFIGS
from oracle import graf_oracle as O
c = CONFIGS[1]
s_np = config_waveforms(1)
s = torch.from_numpy(s_np).cuda()
spec_d = dict(c["loss"], normalize=0)
spec = graf.LossSpec.from_dict(spec_d)
ws = graf.graf.Workspace()
ws.get(1 << 22, s.device)
lo = torch.empty(1, dtype=torch.float64, device="cuda")
g = torch.empty((1, 64), dtype=torch.complex64, device="cuda")
st = torch.cuda.Stream()
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr, stream=st):
    graf.af_loss_grad(s, 64, spec, ws=ws, loss_out=lo, grad=g, stream=st)
for _ in range(2):
    gr.replay()
torch.cuda.synchronize()
L_ref, g_ref, _ = O.loss_and_grad(s_np[0], 64, O.LossSpec.from_dict(spec_d))
assert abs(lo.item() - L_ref) <= 1e-4 * abs(L_ref), (lo.item(), L_ref)
assert np.abs(g.cpu().numpy()[0] - g_ref).max() <= 1e-4 * np.abs(g_ref).max()
print("ok")
""" % ROOT
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
