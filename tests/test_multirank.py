"""Multi-rank host logic on CPU (gloo, world_size 2): the unit sharding used by
bench.py (independent (stream, frame) units, no data-path collective), and the
max-over-ranks timing reduction.  Each rank generates its shard's seeded
inputs with the oracle generator and the union must equal the single-rank
workload bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
import oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, q):
    import torch

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, n = bench.shard(total, rank, world)
    grid = O.gen_grid(99, lo, n, 3, 12, 8)
    t = torch.tensor([float(rank + 1) * 1.5], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    counts = [None] * world
    dist.all_gather_object(counts, (lo, n, grid.tobytes()))
    if rank == 0:
        q.put((float(t.item()), counts))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [7, 512])
def test_sharding_gloo_world2(total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    tmax, counts = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == 3.0
    assert sum(n for _, n, _ in counts) == total
    assert counts[0][0] == 0 and counts[1][0] == counts[0][1]
    whole = O.gen_grid(99, 0, total, 3, 12, 8)
    joined = np.concatenate([np.frombuffer(b, np.complex128).reshape(n, 3, 12) for _, n, b in counts])
    assert np.array_equal(joined, whole)


def test_shard_partition_properties():
    for total in (1, 4, 7, 512):
        for world in (1, 2, 3, 4, 8):
            parts = [bench.shard(total, r, world) for r in range(world)]
            assert sum(n for _, n in parts) == total
            assert all(parts[r][0] + parts[r][1] == parts[r + 1][0] for r in range(world - 1))
            assert max(n for _, n in parts) - min(n for _, n in parts) <= 1


def test_bench_self_launch_world2_gloo():
    """`bench.py --gpus 2` outside torchrun spawns 2 ranks itself (127.0.0.1
    rendezvous), asserts world == --gpus, shards the units and gathers every
    shard on rank 0 — the multi-GPU control path, on gloo without a GPU."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run", "--units", "7"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["max_t"] == 2.0
    assert line["shards"] == [[0, 4], [4, 3]]


def test_bench_rejects_world_mismatch():
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "4", "--dry-run"],
                       capture_output=True, text=True, timeout=120, env=env)
    assert r.returncode != 0 and "WORLD_SIZE" in (r.stderr + r.stdout)
