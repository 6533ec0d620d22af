"""Multi-process (world size 2, gloo, CPU) checks of the (batch, head)
sharding: per-rank results with ``unit_offset`` gathered to rank 0 equal the
single-process result bit for bit (the sampler is keyed by the global unit),
uneven splits included, and the max/sum timing reductions."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import asa_oracle as O
from paper_2508_10774_b200 import inputs, shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, units, out_dir):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        q, k, v = inputs.iid(1, units, 384, 32, seed=11)
        lo, hi = shard.unit_range(world, rank, units)
        p = O.AsaParams(tau=0.85, unit_offset=lo)
        r = O.asa_mask(q[lo:hi], k[lo:hi], p)
        o, lse = O.sparse_attention(q[lo:hi], k[lo:hi], v[lo:hi], r.kv_idx, r.kv_cnt, 128)
        g_idx = shard.gather_units(torch.from_numpy(r.kv_idx), units)
        g_smp = shard.gather_units(torch.from_numpy(r.sample_idx), units)
        g_o = shard.gather_units(torch.from_numpy(o), units)
        mx = shard.max_over_ranks([float(rank), 10.0 - rank])
        sm = shard.sum_over_ranks([float(hi - lo)])
        if rank == 0:
            np.save(os.path.join(out_dir, "kv_idx.npy"), g_idx.numpy())
            np.save(os.path.join(out_dir, "sample_idx.npy"), g_smp.numpy())
            np.save(os.path.join(out_dir, "o.npy"), g_o.numpy())
            np.save(os.path.join(out_dir, "red.npy"), np.array(mx + sm))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("units", [4, 5])
def test_two_rank_shards_equal_single_process(tmp_path, units):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, units, str(tmp_path)), nprocs=2, join=True)
    q, k, v = inputs.iid(1, units, 384, 32, seed=11)
    full = O.asa_mask(q, k, O.AsaParams(tau=0.85))
    o_full, _ = O.sparse_attention(q, k, v, full.kv_idx, full.kv_cnt, 128)
    assert (np.load(tmp_path / "kv_idx.npy") == full.kv_idx).all()
    assert (np.load(tmp_path / "sample_idx.npy") == full.sample_idx).all()
    assert (np.load(tmp_path / "o.npy") == o_full).all()
    red = np.load(tmp_path / "red.npy")
    assert list(red) == [1.0, 10.0, float(units)]


def test_unit_range_partition():
    for units in (1, 5, 12, 96):
        for world in (1, 2, 3, 8):
            ranges = [shard.unit_range(world, r, units) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == units
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            sizes = [b - a for a, b in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard.unit_range(2, 2, 4)
