"""Frame sharding: contiguous partition and the host-side
reduction, including a world_size-2 gloo run on CPU. The per-rank filter is
the CPU oracle here (checker only: the B200 bench uses the same shard logic
with the CUDA library on each rank's device)."""
import os
import socket

import numpy as np
import pytest

from paper_1505_00077_b200 import shard, synth


@pytest.mark.parametrize("n,world", [(0, 1), (1, 1), (5, 2), (192, 8), (64, 3), (7, 8)])
def test_shard_range_partitions(n, world):
    blocks = [shard.shard_range(n, r, world) for r in range(world)]
    assert blocks[0][0] == 0 and blocks[-1][1] == n
    for (a0, b0), (a1, b1) in zip(blocks, blocks[1:]):
        assert b0 == a1
    sizes = [b - a for a, b in blocks]
    assert max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes, reverse=True)
    assert sum(sizes) == n


def test_shard_range_c4_layout():
    # C4: 64 frames x 3 channels = 192 independent problems, 24 per GPU at 8 GPUs
    assert shard.shard_sizes(192, 8) == [24] * 8
    assert shard.shard_range(192, 5, 8) == (120, 144)


def test_shard_range_rejects_bad_rank():
    with pytest.raises(ValueError):
        shard.shard_range(4, 2, 2)
    with pytest.raises(ValueError):
        shard.shard_range(-1, 0, 1)


def test_reduce_job_single_rank():
    assert shard.reduce_job(1.5, [0, 2], 2, 0, 1) == (1.5, [0, 2])
    with pytest.raises(ValueError):
        shard.reduce_job(1.0, [0], 2, 0, 1)


def _frames():
    return np.stack([synth.rects_image(40, 28, 4, 10.0, 100 + i) for i in range(5)]).astype(np.float64)


def _oracle_filter(block):
    from oracle.oracle import Oracle
    o = Oracle()
    outs, fbs = [], []
    for fr in block:
        out, fb, _ = o.gpf(fr, 3.0, 20.0, 20)
        outs.append(out)
        fbs.append(fb)
    return (np.stack(outs) if outs else np.zeros((0,) + block.shape[1:])), fbs


def _worker(rank, world, port, frames, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        start, out, fb = shard.run_shard(frames, rank, world, _oracle_filter)
        secs, all_fb = shard.reduce_job(0.25 * (rank + 1), fb, len(frames), rank, world)
        gathered = [None] * world
        dist.all_gather_object(gathered, (start, out))
        if rank == 0:
            q.put((secs, all_fb, gathered))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_gloo_two_ranks_match_single_process(oracle):
    import torch.multiprocessing as mp
    frames = _frames()
    ref_out, ref_fb = _oracle_filter(frames)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, frames, q)) for r in range(2)]
    for p in procs:
        p.start()
    secs, all_fb, gathered = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert secs == pytest.approx(0.5)  # max over ranks
    assert all_fb == [int(v) for v in ref_fb]
    out = np.concatenate([o for _, o in sorted(gathered, key=lambda t: t[0])])
    np.testing.assert_array_equal(out, ref_out)  # each frame is filtered exactly once
    assert [s for s, _ in sorted(gathered, key=lambda t: t[0])] == [0, 3]
