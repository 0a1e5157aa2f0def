"""Multi-GPU host logic on CPU (world_size 2, gloo): the row partition of SURVEY.md §8e
and the optional gather of every rank's indices.  The per-row selection in these tests
is the oracle (the CUDA path needs a GPU); what is checked is that sharding + gathering
reproduces the unsharded result exactly."""
import os
import socket

import numpy as np
import pytest

import oracle
import synth
from paper_2604_22312_b200.shard import row_partition

K = 64


def test_partition_covers_rows_contiguously():
    rng = np.random.default_rng(5)
    for R in (0, 1, 2, 3, 7, 488, 3904):
        lens = rng.integers(0, 1000, size=R)
        for world in (1, 2, 3, 4, 8):
            b = row_partition(lens, world)
            assert b[0] == 0 and b[-1] == R and len(b) == world + 1
            assert np.all(np.diff(b) >= 0)


def test_partition_balances_work():
    lens = np.full(3904, 131_072)  # cfg5: equal rows split evenly
    for world in (1, 2, 4, 8):
        sizes = np.diff(row_partition(lens, world))
        assert sizes.max() - sizes.min() <= 1
    # ragged: the heaviest block stays within one row of the ideal share
    rng = np.random.default_rng(6)
    lens = rng.integers(8_000, 260_000, size=500)
    for world in (2, 4, 8):
        b = row_partition(lens, world)
        work = np.array([lens[b[w]:b[w + 1]].sum() + (b[w + 1] - b[w]) for w in range(world)])
        assert work.max() <= (lens.sum() + len(lens)) / world + lens.max() + 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _batch():
    rows = [synth.dist_row("normal", n, seed=700 + i) for i, n in enumerate([300, 1000, 64, 17, 5000, 800, 2048, 90, 640])]
    S = max(r.size for r in rows)
    host = np.zeros((len(rows), S), np.float32)
    lens = np.array([r.size for r in rows], np.int32)
    for i, r in enumerate(rows):
        host[i, :r.size] = r
    return host, lens


def _worker(rank, world, port, result_path):
    import torch
    import torch.distributed as dist
    from paper_2604_22312_b200.shard import row_partition, sharded_topk

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        host, lens = _batch()
        bounds = row_partition(lens, world)

        def oracle_topk(scores, k, row_lens=None, prev=None):
            return torch.from_numpy(oracle.topk_batched(scores.numpy(), k, row_lens=row_lens.numpy()))

        full = sharded_topk(torch.from_numpy(host), torch.from_numpy(lens), None, K, bounds, gather=True,
                            topk_fn=oracle_topk)
        local = sharded_topk(torch.from_numpy(host), torch.from_numpy(lens), None, K, bounds, gather=False,
                             topk_fn=oracle_topk)
        assert local.shape[0] == bounds[rank + 1] - bounds[rank]
        if rank == 0:
            np.save(result_path, full.numpy())
    finally:
        dist.destroy_process_group()


def test_world2_shard_and_gather_matches_unsharded(tmp_path):
    import torch.multiprocessing as mp

    out = str(tmp_path / "gathered.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    host, lens = _batch()
    ref = oracle.topk_batched(host, K, row_lens=lens)
    assert np.array_equal(np.load(out), ref)


@pytest.mark.parametrize("config", ["cfg2", "cfg5"])
def test_bench_launcher_starts_the_ranks(config):
    """`bench.py --gpus 2` without WORLD_SIZE starts two ranks itself (torch.distributed.run
    on 127.0.0.1); rank 0 prints one JSON line with n_gpus = 2 and the max-over-ranks
    aggregate (the --cpu-dry-run mode runs the rank plumbing on gloo without kernels)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    res = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--cpu-dry-run",
                          "--steps", "2", "--warmup", "3", "--config", config],
                         capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, res.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2
    if config == "cfg5":  # strong scaling: 64 requests x 61 layers split in halves
        assert d["scaling"] == "strong" and d["rows_all"] == 3904 and d["rows_per_rank0"] == 1952
    else:
        assert d["scaling"] == "weak" and d["rows_all"] == 2 * 488
