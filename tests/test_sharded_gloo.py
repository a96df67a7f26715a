"""Multi-process (world_size 2, gloo, CPU) tests of the multi-GPU partitioning logic.

The per-rank compute is the CPU oracle injected as ``local_forward`` (test-only);
what is under test is the sharding arithmetic, the all-gather and the gathered
layout [G][M][rows/G] -> (M, rows) — the same host code the NCCL path runs.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import tn_oracle as O

CASES = [
    ("tt", (8, 6, 4, 5), 2, (3, 4, 2)),
    ("tr", (4, 6, 6, 4), 2, (2, 3, 2, 2)),
    ("tucker", (16, 12), 1, (4, 5)),
    ("tr", (6, 10), 1, (2, 3)),
]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_forward(L, row_range=None):
    def f(x):
        y = O.forward_torch_orient(L, x.double().numpy())
        if row_range is not None:
            y = y[:, row_range[0]:row_range[1]]
        return torch.from_numpy(np.ascontiguousarray(y))

    return f


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2602_01613_b200 import CompressedLayer
    from paper_2602_01613_b200.sharded import OutputShardedLayer, TokenShardedLayer, output_shard_ranges

    ok = []
    for i, (fam, ms, rm, ranks) in enumerate(CASES):
        L = O.synthetic_layer(fam, ms, rm, ranks, seed=100 + i)
        kw = dict(family=fam, mode_shape=ms, row_mode_count=rm)
        if fam == "tucker":
            kw.update(core=L.core, factors=L.factors)
        else:
            kw.update(cores=L.cores)
        layer = CompressedLayer(**kw)
        rows, cols = L.matrix_shape
        x = torch.from_numpy(O.synthetic_x(6, cols, seed=7))  # same on every rank
        ref = O.forward_torch_orient(L, x.numpy())
        rr = output_shard_ranges(ms, rm, world)[rank]
        osl = OutputShardedLayer(layer, local_forward=_oracle_forward(L, rr))
        assert osl.row_range == rr
        y = osl(x).numpy()
        ok.append(float(np.abs(y - ref).max()))
        tsl = TokenShardedLayer(layer, local_forward=_oracle_forward(L))
        yt = tsl(x, gather=True).numpy()
        ok.append(float(np.abs(yt - ref).max()))
    results[rank] = ok
    dist.barrier()
    dist.destroy_process_group()


def test_output_and_token_sharding_world2():
    port = _free_port()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(2, port, results), nprocs=2, join=True)
    assert set(results.keys()) == {0, 1}
    for r in (0, 1):
        assert max(results[r]) < 1e-12, results[r]


def test_shard_ranges_follow_leading_mode():
    from paper_2602_01613_b200.sharded import output_shard_ranges, token_shard_range

    # Qwen3-32B MLP gate/up: (160,160|64,80) -> i0 = 160 splits over 2/4/8
    for g in (1, 2, 4, 8):
        rr = output_shard_ranges((160, 160, 64, 80), 2, g)
        assert rr[0] == (0, 25600 // g) and rr[-1][1] == 25600
        assert all((b - a) == 25600 // g for a, b in rr)
        assert all(a % 160 == 0 for a, _ in rr)  # i0-aligned
    # Tucker-2 5120 rows
    assert output_shard_ranges((5120, 5120), 1, 8)[3] == (1920, 2560)
    with pytest.raises(Exception):
        output_shard_ranges((7, 5), 1, 2)
    assert token_shard_range(10, 0, 4) == (0, 3) and token_shard_range(10, 3, 4) == (9, 10)
