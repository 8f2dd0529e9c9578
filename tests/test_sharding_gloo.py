"""Multi-GPU host logic on CPU: partitions, and the Gaussian-sharded deformation +
all-gather assembled by `ShardedDeform` over world_size-2 gloo process groups.

The per-rank "kernel" here is the fp64 oracle deform of the rank's slice (cast to fp32, the dtype of
the CUDA outputs), so what is tested is exactly the host logic: who deforms which rows, the padded
in-place all-gather, and the (e2) pipeline order.  The CUDA side (fgs_deform_range bit-identical to
the unsharded rows) is tested in test_gpu_parity.py::test_deform_range_and_batch_bit_identical.
"""
import os
import socket

import numpy as np
import pytest

from paper_2310_08528_b200.sharding import (ShardedDeform, frame_split, padded_rows, shard_range,
                                            views_of_times)


@pytest.mark.parametrize("n,world", [(0, 2), (1, 2), (7, 2), (8, 4), (100_003, 8), (5, 8)])
def test_shard_range_partitions(n, world):
    got = [shard_range(n, r, world) for r in range(world)]
    covered = [i for b, e in got for i in range(b, e)] if n < 1000 else None
    if covered is not None:
        assert covered == list(range(n))
    assert got[0][0] == 0 and got[-1][1] == n
    for (b0, e0), (b1, e1) in zip(got, got[1:]):
        assert e0 == b1 or (b1 == e1 == n)
    chunk = padded_rows(n, world) // world if n else 0
    assert all(e - b <= chunk for b, e in got)
    assert padded_rows(n, world) >= n and padded_rows(n, world) % world == 0


@pytest.mark.parametrize("F,world", [(20, 1), (20, 3), (64, 8), (3, 8), (0, 2)])
def test_frame_split_partitions(F, world):
    parts = [frame_split(F, r, world) for r in range(world)]
    assert sum(parts, []) == list(range(F))
    sizes = [len(p) for p in parts]
    assert max(sizes) - min(sizes) <= 1


def test_views_of_times_cover_every_frame_once():
    world, K, V = 4, 8, 8
    frames = sorted(k * V + v for r in range(world) for k, v in views_of_times(K, V, r, world))
    assert frames == list(range(K * V))


def test_bad_partition_args():
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)
    with pytest.raises(ValueError):
        frame_split(10, 0, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, times, q):
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2310_08528_b200.inputs import make_scene

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s = make_scene("tiny", n=n)
        sd = ShardedDeform(n, world, rank, "cpu", n_slots=2)
        calls = []

        def deform_fn(slot, t, b, e, bufs):
            calls.append((slot, b, e))
            ref = oracle.deform_ref(s, t, begin=b, end=e)
            for k in bufs:
                bufs[k][b:e] = torch.from_numpy(ref[k].astype(np.float32))

        out = []
        for k, t in enumerate(times):
            slot = k % 2
            sd.deform(slot, t, deform_fn)
            for w in sd.gather(slot, async_op=True):
                w.wait()
            out.append({kk: v.clone().numpy() for kk, v in sd.arrays(slot).items()})
        q.put((rank, calls, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [2000, 2001, 1])
def test_sharded_deform_allgather_gloo(n):
    import multiprocessing as mp

    import oracle
    from paper_2310_08528_b200.inputs import make_scene

    world, times = 2, [0.0, 0.37, 1.0]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, times, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict()
    for _ in range(world):
        rank, calls, out = q.get(timeout=240)
        res[rank] = (calls, out)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    s = make_scene("tiny", n=n)
    for rank in range(world):
        calls, out = res[rank]
        b, e = shard_range(n, rank, world)
        assert all((cb, ce) == (b, e) for _, cb, ce in calls)       # each rank deforms only its slice
        for k, t in enumerate(times):
            ref = oracle.deform_ref(s, t)
            for key in ref:
                assert out[k][key].shape == ref[key].shape
                assert np.array_equal(out[k][key], ref[key].astype(np.float32)), (rank, k, key)


def test_sharded_deform_fused_host_logic(monkeypatch):
    """Fused (e2) host logic without a GPU: one symmetric buffer per slot carved quats | means |
    log_scales, replica offsets = buffer_ptrs[q] - buffer_ptrs[rank] handed to the deform callback,
    and gather() = the handle's stream-ordered barrier on the slot's channel (no collective call)."""
    import torch
    import torch.distributed._symmetric_memory as symm_mem

    calls = {"barrier": []}

    class FakeHandle:
        def __init__(self, t):
            self.rank, self.world_size = 1, 3
            base = t.data_ptr()
            self.buffer_ptrs = [base - 4096, base, base + 8192]

        def barrier(self, channel=0):
            calls["barrier"].append(channel)

    monkeypatch.setattr(symm_mem, "empty", lambda n, dtype, device: torch.zeros(n, dtype=dtype))
    monkeypatch.setattr(symm_mem, "rendezvous", lambda t, grp: FakeHandle(t))
    import torch.distributed as dist
    monkeypatch.setattr(dist, "group", type("G", (), {"WORLD": "world"}))
    n, world, rank = 101, 3, 1
    sd = ShardedDeform(n, world, rank, "cpu", n_slots=2, fused=True)
    rows = padded_rows(n, world)
    assert sd.offsets == [[-4096, 0, 8192]] * 2
    b = sd.bufs[0]
    assert b["quats"].shape == (rows, 4) and b["means"].shape == (rows, 3) and b["log_scales"].shape == (rows, 3)
    # one flat buffer: quats at offset 0 (16-byte aligned), means after them, log_scales last
    assert b["means"].data_ptr() - b["quats"].data_ptr() == rows * 4 * 4
    assert b["log_scales"].data_ptr() - b["means"].data_ptr() == rows * 3 * 4
    seen = []
    sd.deform(1, 0.25, lambda slot, t, lo, hi, bufs, offsets: seen.append((slot, t, lo, hi, offsets,
                                                                           list(calls["barrier"]))))
    # the slot-free barrier (channel 2 + slot) is enqueued BEFORE the deform writes into the peers' copies
    # of the slot (a peer may still be rendering the slot's previous time)
    assert seen == [(1, 0.25) + shard_range(n, rank, world) + ([-4096, 0, 8192], [3])]
    assert sd.gather(1) == [] and calls["barrier"] == [3, 1]
    # a rank with an empty shard still joins the slot-free barrier (every rank must reach it)
    sd.begin = sd.end
    sd.deform(0, 0.5, lambda *a: seen.append(a))
    assert len(seen) == 1 and calls["barrier"] == [3, 1, 2]


def _frames_worker(rank, world, port, W, H, q):
    """(e1) frame-batch split on gloo: each rank renders (here: the oracle renders) only its frame_split
    chunk of a reduced D batch; gather_frames assembles the batch on rank 0 in frame order."""
    import torch
    import torch.distributed as dist

    import oracle
    from oracle import render as OR
    from paper_2310_08528_b200.inputs import make_scene
    from paper_2310_08528_b200.sharding import gather_frames

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s = make_scene("dnerf", n=400, width=W, height=H, n_frames=5)
        mine = frame_split(s.n_frames, rank, world)
        imgs = []
        for f in mine:
            d = oracle.deform_ref(s, float(s.times[f]))
            out = OR.render_ref(d, s.opacity_logits, s.sh, s.sh_degree, s.cameras[f])
            imgs.append(torch.from_numpy(out["image"].astype(np.float32)))
        got = gather_frames(imgs, s.n_frames, rank, world)
        q.put((rank, mine, None if got is None else [g.numpy() for g in got]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_frame_split_gather_gloo(world):
    """bench.py --gpus N frames mode: the config's batch is split (not replicated) across ranks and the
    rank-0 gather reproduces the single-process batch image for image (5 frames: ragged split)."""
    import multiprocessing as mp

    import oracle
    from oracle import render as OR
    from paper_2310_08528_b200.inputs import make_scene

    W, H = 40, 24
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_frames_worker, args=(r, world, port, W, H, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, mine, got = q.get(timeout=240)
        res[rank] = (mine, got)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sum((res[r][0] for r in range(world)), []) == list(range(5))
    assert all(res[r][1] is None for r in range(1, world))
    s = make_scene("dnerf", n=400, width=W, height=H, n_frames=5)
    got = res[0][1]
    assert len(got) == 5
    for f in range(5):
        d = oracle.deform_ref(s, float(s.times[f]))
        want = OR.render_ref(d, s.opacity_logits, s.sh, s.sh_degree, s.cameras[f])["image"].astype(np.float32)
        assert np.array_equal(got[f], want), f
