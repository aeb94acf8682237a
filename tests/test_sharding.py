"""Column sharding across ranks: host logic and the verification all-gather.

Runs world_size=2 over gloo on the CPU.  Each rank computes its shard with the
CPU oracle standing in for its GPU (test-only injection), then the shards are
all-gathered and must equal the single-process product bit-for-bit (tiles are
independent, reference sdmm.py:167).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from conftest import ROOT
import paper_2006_13486_b200 as ks
from paper_2006_13486_b200 import sharding
from paper_2006_13486_b200 import workloads as wl


def test_column_shards_tile_aligned():
    assert sharding.column_shards(1024, 2, 128) == [(0, 512), (512, 1024)]
    assert sharding.column_shards(1024, 3, 128) == [(0, 384), (384, 768), (768, 1024)]
    assert sharding.column_shards(256, 4, 128) == [(0, 128), (128, 256), (256, 256), (256, 256)]
    for n, world, tn in [(4096, 8, 128), (1000, 7, 8), (64, 1, 64)]:
        shards = sharding.column_shards(n, world, tn)
        assert shards[0][0] == 0 and shards[-1][1] == n
        assert all(a % tn == 0 and b % tn == 0 for a, b in shards)
        assert all(shards[i][1] == shards[i + 1][0] for i in range(world - 1))


def test_column_shards_errors():
    with pytest.raises(ks.ConfigurationError):
        sharding.column_shards(100, 2, 128)
    with pytest.raises(ks.ConfigurationError):
        sharding.column_shards(128, 0, 128)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        chain, w, inp = wl.make_operands(wl.C1A)
        params = ks.tiling_for_chain(chain)
        local = sharding.local_columns(inp, world, rank, params.tn)
        out_local = sharding.rbgp4mm_sharded(
            w, np.ascontiguousarray(local), params,
            multiply=lambda w_, x_, p_: oracle.tiled(w_, x_, p_))
        full = sharding.gather_columns(torch.from_numpy(out_local), inp.shape[1], params.tn)
        if rank == 0:
            np.save(result_path, full.numpy())
    finally:
        dist.destroy_process_group()


def test_two_rank_gather_equals_single_process(tmp_path):
    world, port = 2, _free_port()
    result = str(tmp_path / "full.npy")
    mp.spawn(_worker, args=(world, port, result), nprocs=world, join=True)
    chain, w, inp = wl.make_operands(wl.C1A)
    want = oracle.tiled(w, inp, ks.tiling_for_chain(chain))
    got = np.load(result)
    assert np.array_equal(got, want)
    # and that is the reference's own output (golden hash)
    import hashlib
    assert hashlib.sha256(got.tobytes()).hexdigest()[:16] == "9fe440861f6f8868"


def test_bench_spawns_ranks_and_verifies_the_gather():
    """`bench.py --gpus 2` outside torchrun re-launches itself as 2 ranks (torch.distributed.run
    on 127.0.0.1); the self-test mode runs the same shard -> all-gather -> reassembly plumbing as
    the GPU run's verification, over gloo on the CPU, and must report n_gpus 2 and a verified
    gather."""
    import json
    import subprocess
    import sys
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dist-selftest"],
                         capture_output=True, text=True, timeout=300, env=env)
    assert res.returncode == 0, res.stderr[-2000:]
    line = json.loads([ln for ln in res.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["gather_verified"] is True and line["backend"] == "gloo"
