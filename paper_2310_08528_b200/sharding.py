"""Multi-GPU plumbing for the per-frame 4D-GS path — SURVEY.md §8(e), BASELINE.json north_star.

Two ways to use one 8xB200 box (one process per GPU, torch.distributed):

(e1) frame-batch split — `frame_split(n_frames, rank, world)`: a batch of (t, view) frames is cut into
     contiguous per-rank chunks; every rank holds a replica of G, the HexPlane and the MLP and renders
     its own frames.  No collective on the data path.

(e2) Gaussian-sharded deformation — `ShardedDeform`: rank r deforms only the contiguous Gaussian slice
     `shard_range(n, r, world)` (fgs_deform_range, bit-identical to the same rows of an unsharded
     fgs_deform because every Gaussian's arithmetic is independent of the shard), then the deformed
     attributes X', r', s' (40 B per Gaussian) are assembled on every rank with
     `all_gather_into_tensor` (NCCL over NVLink/NVSwitch).  The gather is issued async_op so the caller
     can render the previous time while it is in flight (the one exchange step of the path).
     `fused=True` (SURVEY §8(e2) "fused option"): the gather buffers are symmetric memory
     (torch.distributed._symmetric_memory) and fgs_deform_range_peers stores every deformed row
     straight into ALL ranks' buffers from the deform epilogue (NVLink peer stores, overlapped with
     the deformation tile by tile); the exchange step is then one stream-ordered barrier.

Host logic only: every arithmetic step of the method runs in libfgs.so (or, in the CPU tests, in a
deform callback supplied by the test); this module partitions, allocates and exchanges.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence, Tuple

# Attribute widths of the deformed arrays fgs_deform writes (include/fgs.h fgs_deformed).
DEFORMED_FIELDS: Tuple[Tuple[str, int], ...] = (("means", 3), ("log_scales", 3), ("quats", 4))


def shard_range(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous Gaussian slice [begin, end) of `rank`: equal chunks of ceil(n / world) rows, the last
    rank(s) short (possibly empty).  Equal chunk size is what all_gather_into_tensor needs."""
    if world < 1 or not (0 <= rank < world) or n < 0:
        raise ValueError(f"bad shard ({n=}, {rank=}, {world=})")
    chunk = -(-n // world) if n else 0
    begin = min(n, rank * chunk)
    return begin, min(n, begin + chunk)


def padded_rows(n: int, world: int) -> int:
    """Rows of the gather buffers: world * ceil(n / world) >= n."""
    return world * (-(-n // world)) if n else 0


def frame_split(n_frames: int, rank: int, world: int) -> List[int]:
    """(e1) frame indices of `rank`: contiguous chunks, sizes differing by at most one."""
    if world < 1 or not (0 <= rank < world) or n_frames < 0:
        raise ValueError(f"bad split ({n_frames=}, {rank=}, {world=})")
    base, extra = divmod(n_frames, world)
    begin = rank * base + min(rank, extra)
    return list(range(begin, begin + base + (1 if rank < extra else 0)))


def gather_frames(images: Sequence, n_frames: int, rank: int, world: int, group=None):
    """(e1) untimed validation step: every rank's images of its frame_split chunk -> the whole batch in
    frame order on rank 0 (other ranks get None).  One all_gather of the chunks padded to the largest
    chunk (all_gather works on NCCL and gloo alike); images are same-shape tensors on the rank's device."""
    import torch
    import torch.distributed as dist
    mine = frame_split(n_frames, rank, world)
    if len(images) != len(mine):
        raise ValueError(f"rank {rank} holds {len(images)} images for {len(mine)} frames")
    if world == 1 or not (dist.is_available() and dist.is_initialized()):
        return list(images)
    per = -(-n_frames // world)
    ref = images[0] if images else None
    shape = tuple(ref.shape) if ref is not None else None
    # every rank must agree on shape/dtype/device: take them from rank 0's first image
    meta = [shape, None if ref is None else str(ref.dtype)]
    objs = [None] * world
    dist.all_gather_object(objs, meta, group=group)
    shape, dtype = next((tuple(o[0]), o[1]) for o in objs if o[0] is not None)
    dt = getattr(torch, dtype.replace("torch.", ""))
    dev = ref.device if ref is not None else (torch.device("cuda", torch.cuda.current_device())
                                              if dist.get_backend(group) == "nccl" else torch.device("cpu"))
    buf = torch.zeros((per,) + shape, dtype=dt, device=dev)
    for i, im in enumerate(images):
        buf[i].copy_(im)
    out = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(out, buf, group=group)
    if rank != 0:
        return None
    frames = []
    for r in range(world):
        frames.extend(out[r][:len(frame_split(n_frames, r, world))].unbind(0))
    return frames


def views_of_times(n_times: int, n_views: int, rank: int, world: int) -> List[Tuple[int, int]]:
    """(e2) multi-view batch: frames (time k, view v), frame id k * n_views + v.  Views are split across
    ranks (each rank renders its views at EVERY time), so all ranks need G'(t_k) for every k — the case
    in which sharding the deformation by Gaussian pays."""
    vs = frame_split(n_views, rank, world)
    return [(k, v) for k in range(n_times) for v in vs]


class ShardedDeform:
    """Gaussian-sharded deformation with an all-gather of the deformed attributes.

    Buffers: for each slot (time) three tensors [rows][3|3|4] float32 on `device`, rows =
    padded_rows(n, world); rows >= n are padding that no fgs_render reads (the fgs_deformed struct
    keeps n).  Rank r's shard is rows [r*chunk, (r+1)*chunk), of which [begin, end) are real.

    deform_fn(slot, t, begin, end, bufs) must write rows [begin, end) of `bufs` (the CUDA path calls
    fgs_deform_range; CPU tests pass a callback).  gather(slot) all-gathers the three arrays
    (in place: each rank's input is its own chunk of the output).
    """

    def __init__(self, n: int, world: int, rank: int, device, n_slots: int = 2, group=None, fused: bool = False):
        import torch
        self.n, self.world, self.rank, self.group = n, world, rank, group
        self.rows = padded_rows(n, world)
        self.chunk = self.rows // world if world else 0
        self.begin, self.end = shard_range(n, rank, world)
        self.fused = fused
        self.bufs: List[dict] = []
        self.handles: list = []
        self.offsets: List[List[int]] = []
        rows = max(self.rows, 1)
        for _ in range(n_slots):
            if not fused:
                # padding rows are zero-filled once so a gathered buffer never holds uninitialised memory
                self.bufs.append({k: torch.zeros((rows, w), dtype=torch.float32, device=device)
                                  for k, w in DEFORMED_FIELDS})
                continue
            # one symmetric buffer per slot holding the three arrays back to back, so a replica's
            # offset from the local copy is the same for all three (fgs_deform_range_peers)
            import torch.distributed as dist
            import torch.distributed._symmetric_memory as symm_mem
            grp = group if group is not None else dist.group.WORLD
            flat = symm_mem.empty(rows * 10, dtype=torch.float32, device=device)
            flat.zero_()
            h = symm_mem.rendezvous(flat, grp)
            ptrs = [int(x) for x in h.buffer_ptrs]
            self.handles.append(h)
            self.offsets.append([ptrs[q] - ptrs[h.rank] for q in range(h.world_size)])
            # quats first: they need 16-byte alignment (float4 loads), means / log_scales only 4
            views, o = {}, 0
            for k, w in (("quats", 4), ("means", 3), ("log_scales", 3)):
                views[k] = flat[o:o + rows * w].view(rows, w)
                o += rows * w
            self.bufs.append(views)

    def deform(self, slot: int, t: float, deform_fn: Callable[..., None]) -> None:
        """deform_fn(slot, t, begin, end, bufs) — with fused=True also the peer offsets of the slot's
        replicas: deform_fn(slot, t, begin, end, bufs, offsets).

        fused: this rank's deform writes into EVERY rank's copy of the slot, so before it starts, every
        rank must have finished reading the slot's previous contents (its render of the time the slot
        held before).  A stream-ordered barrier over the group on channel 2 + slot does that: each rank
        enqueues it after its earlier render of the slot (the render was issued before this call), so
        when the barrier completes on this rank's stream, all peers' streams have passed that render.
        (The NCCL path needs none: each rank's all-gather writes only its own buffer, in its stream
        order, after its own render.)"""
        if self.fused:
            self.handles[slot].barrier(channel=2 + slot)
        if self.end > self.begin:
            if self.fused:
                deform_fn(slot, t, self.begin, self.end, self.bufs[slot], self.offsets[slot])
            else:
                deform_fn(slot, t, self.begin, self.end, self.bufs[slot])

    def gather(self, slot: int, async_op: bool = True):
        """all_gather_into_tensor of the three deformed arrays of `slot`; returns the work handles
        (wait() them, or let the NCCL stream ordering do it, before rendering the slot)."""
        import torch.distributed as dist
        works = []
        if self.fused:
            # the rows are already in every rank's buffer (peer stores of the deform epilogue): a
            # stream-ordered barrier over the group makes them visible before the render
            self.handles[slot].barrier(channel=slot)
            return works
        # world size 1 still goes through the collective when a process group exists (the same code
        # path as N > 1; NCCL copies in place), so the single-GPU bench exercises it
        if self.rows == 0 or not (dist.is_available() and dist.is_initialized()):
            return works
        c0 = self.rank * self.chunk
        for k, _ in DEFORMED_FIELDS:
            out = self.bufs[slot][k]
            w = dist.all_gather_into_tensor(out, out[c0:c0 + self.chunk], group=self.group, async_op=async_op)
            if w is not None:
                works.append(w)
        return works

    def arrays(self, slot: int) -> dict:
        """The first n rows of the gathered arrays of `slot` (views)."""
        return {k: v[:self.n] for k, v in self.bufs[slot].items()}


def fgs_range_deformer(ds, stream=None) -> Callable[..., None]:
    """deform_fn for ShardedDeform running fgs_deform_range (libfgs.so) on a fgs.DeviceScene, or
    fgs_deform_range_peers when given the replicas' offsets (fused mode)."""
    from . import fgs

    def run(slot, t, begin, end, bufs, offsets=None):
        d = ds.deformed_struct(bufs["means"], bufs["log_scales"], bufs["quats"])
        if offsets is None:
            fgs.fgs_deform_range(ds.g, ds.field, ds.mlp, float(t), begin, end, d, stream)
        else:
            fgs.fgs_deform_range_peers(ds.g, ds.field, ds.mlp, float(t), begin, end, d, offsets, stream)

    return run


def sharded_frames(ds, sd: ShardedDeform, times: Sequence[float], views: Sequence, images: Sequence,
                   ws, deform_fn=None) -> None:
    """(e2) pipeline over times: deform shard + async all-gather of t_{k+1} are issued before the render
    of t_k, so the NVLink transfer overlaps the render.  views[k] = list of (camera struct, image index)
    this rank renders at time k.  Needs sd.bufs to have >= 2 slots."""
    from . import fgs
    deform_fn = deform_fn or fgs_range_deformer(ds)
    K = len(times)
    if K == 0:
        return
    sd.deform(0, times[0], deform_fn)
    pending = sd.gather(0)
    for k in range(K):
        slot = k % len(sd.bufs)
        for w in pending:
            w.wait()                        # current stream waits for the gather of slot k
        nxt = []
        if k + 1 < K:
            sd.deform((k + 1) % len(sd.bufs), times[k + 1], deform_fn)
            nxt = sd.gather((k + 1) % len(sd.bufs))
        a = sd.bufs[slot]
        d = ds.deformed_struct(a["means"], a["log_scales"], a["quats"])
        cams = [c for c, _ in views[k]]
        if cams:
            fgs.fgs_render_batch(cams, [d] * len(cams), [images[i] for _, i in views[k]], ws)
        pending = nxt
