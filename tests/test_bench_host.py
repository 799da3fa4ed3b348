"""Host-side logic of bench.py that the multi-GPU runs depend on (no GPU here):
the per-rank work plan of SURVEY.md §8(e), the max-over-ranks reduction over a real
world-size-2 process group (gloo, CPU), the --gpus / WORLD_SIZE contract, and the
algorithmic flop counts of SURVEY.md §8(d)."""
import math
import os
import socket
import subprocess
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_rank_plan_partitions(cid, world):
    w = bench.workload(cid)
    plans = [bench.rank_plan(w, world, r) for r in range(world)]
    if world == 1:
        assert plans[0]["B_local"] == w["B"] and plans[0]["units"] == w["B"]
        return
    if cid == 5:        # delay sharding: every rank all waveforms, its own rows
        assert all(p["kind"] == "delay" and p["B_local"] == w["B"] for p in plans)
        assert sorted(p["shard"] for p in plans) == [(r, world) for r in range(world)]
        assert all(p["units"] == w["B"] for p in plans)
    elif cid == 1:      # one 64-sample waveform: replicas
        assert all(p["kind"] == "replica" and p["units"] == world for p in plans)
    else:               # batch sharding: contiguous B/G blocks covering the batch once
        spans = sorted((p["b0"], p["b0"] + p["B_local"]) for p in plans)
        assert spans[0][0] == 0 and spans[-1][1] == w["B"]
        assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
        assert max(p["B_local"] for p in plans) - min(p["B_local"] for p in plans) <= 1
        assert all(p["units"] == w["B"] and p["scaling"] == "strong" for p in plans)


def test_flop_counts():
    w5 = bench.workload(5)
    assert w5["single"] and w5["flops"] == 8 * 16384 * 2 * 14 * 5.0 * 16384
    w4 = bench.workload(4)     # pruned band-cache passes (13 radix-2 stages at M = 8192)
    assert math.isclose(w4["stages"], (13 - 1 - 7 / 8) + (13 - 3))
    assert w4["flops"] == 64 * 513 * w4["stages"] * 5.0 * 8192
    w2 = bench.workload(2)
    assert w2["flops"] == 256 * 65 * 2 * 8 * 5.0 * 256


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = bench.workload(5)
        plan = bench.rank_plan(w, world, rank)
        vals = bench.max_over_ranks([10.0 + rank, 5.0 - rank], torch.device("cpu"), world)
        q.put((rank, plan["shard"], vals))
    finally:
        dist.destroy_process_group()


def test_max_over_ranks_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [(0, 2), (1, 2)]
    for _, _, vals in res:
        assert vals == [11.0, 5.0]


def test_gpus_flag_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="4", RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"], env=env,
                       capture_output=True, text=True, timeout=120)
    assert r.returncode != 0 and "WORLD_SIZE = 4" in (r.stderr + r.stdout)
