"""Multi-rank host logic on CPU (gloo, world_size 2): keyframe sharding,
row bands and the max-over-ranks timing reduction bench.py uses."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2207_12244_b200 import shard


def test_keyframe_partition_covers_batch():
    for world in (1, 2, 4, 8):
        seen = []
        for r in range(world):
            seen += shard.keyframes_for_rank(64, world, r)
        assert sorted(seen) == list(range(64))
    with pytest.raises(ValueError):
        shard.keyframes_for_rank(4, 2, 2)


def test_row_bands():
    for h in (1, 7, 480, 2160):
        for world in (1, 2, 3, 8):
            bands = shard.row_bands(h, world)
            assert bands[0][0] == 0 and bands[-1][1] == h
            assert all(a[1] == b[0] for a, b in zip(bands, bands[1:]))
    assert shard.band_halo(2160, 8, 0) == (0, 1)
    assert shard.band_halo(2160, 8, 3) == (1, 1)
    assert shard.band_halo(2160, 8, 7) == (1, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2207_12244_b200 import bands_dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = shard.keyframes_for_rank(64, world, rank)
    t = shard.max_over_ranks(10.0 + rank)
    # row-band peer exchange (bands_dist): every rank gets every record, in
    # rank order, byte for byte; band counts are summed over ranks
    r0, r1 = shard.row_bands(2160, world)[rank]
    me = bands_dist.BandPeer(bytes([rank + 1]) * 64, 148 - rank, r0, r1, 3840)
    recs = bands_dist.exchange_peers(bytes(me), world)
    peers = [bands_dist.BandPeer.from_buffer_copy(r) for r in recs]
    counts = bands_dist.sum_over_ranks([100 + rank, 7 * rank], world)
    dist.barrier()
    q.put((rank, mine, t, [(p.handle[0], p.cpr, p.y0, p.y1, p.width) for p in peers], counts))
    dist.destroy_process_group()


def test_two_rank_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert res[0][2] == res[1][2] == 11.0
    assert sorted(res[0][1] + res[1][1]) == list(range(64))
    bands = shard.row_bands(2160, 2)
    expect = [(g + 1, 148 - g, bands[g][0], bands[g][1], 3840) for g in range(2)]
    assert res[0][3] == res[1][3] == expect
    assert res[0][4] == res[1][4] == [201, 7]
