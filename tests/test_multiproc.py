"""N > 1 on CPU (gloo, world size 2, 127.0.0.1).

The B200 path runs one process per GPU as independent replicas
(DESIGN.md §8): bench.py takes the slowest rank's time (all-reduce MAX) and
reports the whole-job points/s.  The sharded build that SURVEY §8(e)
sketches rests on counters being additive; that property is checked here with
the C oracle: two shards' counters all-reduced (SUM) equal the sketch of the
union, and the merged sketch's T must be recomputed as sum c^2."""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, ws, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws),
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, str(ROOT))
    import torch
    import torch.distributed as dist

    import bench
    from oracle import Oracle

    dist.init_process_group("gloo", rank=rank, world_size=ws)
    res = {}
    # replica timing: slowest rank wins, value counts every rank's points
    ms = bench.max_over_ranks(1.5 + rank, ws)
    res["ms"] = ms
    res["value"] = bench.replica_value(1000, ws, ms)
    # additive counters: shard the rows, insert locally, all-reduce SUM
    o = Oracle()
    k, l, d, n = 8, 6, 16, 600
    w = o.directions(7, d, k, l)
    x = np.random.default_rng(3).standard_normal((n, d)).astype(np.float32)
    lo, hi = rank * n // ws, (rank + 1) * n // ws
    ids, _ = o.buckets(w, x[lo:hi], k, l)
    sk = o.sketch(k, l)
    sk.insert_ids(ids)
    c = torch.from_numpy(sk.counters().astype(np.int64))
    dist.all_reduce(c, op=dist.ReduceOp.SUM)
    res["merged"] = c.numpy()
    dist.barrier()
    dist.destroy_process_group()
    np.savez(Path(out_dir) / f"r{rank}.npz", ms=res["ms"], value=res["value"], merged=res["merged"])


@pytest.mark.timeout(300)
def test_gloo_world2_replicas_and_additive_counters(tmp_path, oracle_c):
    import torch.multiprocessing as mp

    ws = 2
    mp.spawn(_worker, args=(ws, _free_port(), str(tmp_path)), nprocs=ws, join=True)
    r = [np.load(tmp_path / f"r{i}.npz") for i in range(ws)]
    for ri in r:
        assert float(ri["ms"]) == 2.5  # max over ranks
        assert float(ri["value"]) == 1000 * ws / 2.5e-3
    assert np.array_equal(r[0]["merged"], r[1]["merged"])
    # the union's sketch, built in one piece
    k, l, d, n = 8, 6, 16, 600
    w = oracle_c.directions(7, d, k, l)
    x = np.random.default_rng(3).standard_normal((n, d)).astype(np.float32)
    ids, _ = oracle_c.buckets(w, x, k, l)
    whole = oracle_c.sketch(k, l)
    whole.insert_ids(ids)
    assert np.array_equal(r[0]["merged"], whole.counters().astype(np.int64))
    # T is not additive: recompute it from the merged counters
    merged = r[0]["merged"].astype(np.float64)
    assert abs((merged ** 2).sum() / (n * l) - whole.mean()) <= 1e-9 * whole.mean()
