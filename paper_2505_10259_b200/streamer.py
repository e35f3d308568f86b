"""K1 — layer-wise target-weight streamer (pinned host DRAM → HBM window).

Reference model: a two-slot GPU window for the current and next FFN layer
(placement.py:198-199), one CPU→GPU op per non-pinned layer triggered by that
layer (prefetch_schedule, placement.py:260-283), load time
ffn_bytes / c2g_bandwidth (costmodel.py:74).  The reference starts layer ℓ's
load only when layer ℓ starts (simulator.py:168-177), idling the link during
every FFN compute.  Here the copy stream runs ``n_slots − 1``
layers ahead: copy k is enqueued as soon as compute k−n_slots has released its
slot, across pass (round) boundaries, so the PCIe link never waits for the
host loop.  No SMs are involved (copy engine DMA), the compute stream waits on
a per-slot CUDA event only right before the layer's expert GEMMs — the layer's
attention runs while its FFN bytes are still in flight.
"""
from __future__ import annotations

import concurrent.futures
import ctypes
import dataclasses
import mmap
import os
import threading
import weakref

import torch

from . import native
from .codec import Cursor, XC4Parts, XC4Unit
from .errors import InsufficientTotalMemory


class HostStore:
    """Pinned host memory for the streamed layers.

    Large regions are mmap'ed anonymously, advised to transparent huge pages,
    pre-faulted by several threads, then page-locked with cudaHostRegister —
    much faster than cudaHostAlloc for hundreds of GB (measured on the box,
    DESIGN.md §K1).  Small regions fall back to torch's pinned allocator.
    """

    def __init__(self, threads: int | None = None):
        self._maps: list[tuple[mmap.mmap, weakref.finalize, int]] = []
        self.threads = threads or min(16, os.cpu_count() or 4)
        self.bytes = 0

    def alloc(self, nbytes: int) -> torch.Tensor:
        if nbytes < (256 << 20):
            t = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
            self.bytes += nbytes
            return t
        m = mmap.mmap(-1, nbytes, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
        try:
            m.madvise(mmap.MADV_HUGEPAGE)
        except (AttributeError, OSError):
            pass
        buf = (ctypes.c_uint8 * nbytes).from_buffer(m)
        addr = ctypes.addressof(buf)
        self._prefault(addr, nbytes)
        rc = torch.cuda.cudart().cudaHostRegister(addr, nbytes, 0)
        if int(rc) != 0:
            raise InsufficientTotalMemory(f"cudaHostRegister of {nbytes} B failed ({int(rc)})")
        # the page lock lives exactly as long as the mapping's last view: the
        # finaliser runs before the buffer export is dropped, i.e. before the
        # mmap can be unmapped (a range unmapped while registered leaks its
        # pinned pages and makes the next mapping at that address fail, 712)
        fin = weakref.finalize(buf, _host_unregister, addr)
        fin.atexit = False
        self._maps.append((m, fin, nbytes))
        self.bytes += nbytes
        t = torch.frombuffer(buf, dtype=torch.uint8)
        return t

    def _prefault(self, addr: int, nbytes: int) -> None:
        page = 1 << 21
        n = self.threads
        step = (nbytes // n + page - 1) // page * page

        def touch(lo: int, hi: int) -> None:
            ctypes.memset(addr + lo, 0, max(0, hi - lo))

        ts = [threading.Thread(target=touch, args=(i * step, min(nbytes, (i + 1) * step))) for i in range(n)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()

    def close(self) -> None:
        """Unlock every region now (views stay readable as pageable memory)."""
        for _, fin, _ in self._maps:
            fin()
        self._maps.clear()


def _host_unregister(addr: int) -> None:
    torch.cuda.cudart().cudaHostUnregister(addr)


def slice_bounds(nbytes: int, rank: int, world: int) -> tuple[int, int]:
    """Byte range of ``rank``'s 1/N share of an ``nbytes`` layer (equal, page-aligned shares)."""
    if nbytes % world or (nbytes // world) % 4096:
        raise ValueError(f"layer of {nbytes} B does not split into {world} page-aligned slices")
    share = nbytes // world
    return rank * share, (rank + 1) * share


class SharedHostStore:
    """One host copy of the streamed layers for all ranks of a box.

    Rank 0 creates a file in /dev/shm; every rank maps it MAP_SHARED and
    page-locks only its own 1/N slice of each layer (the bytes it will push
    over its own PCIe link).  ``write_slice`` fills that slice from a GPU
    tensor, so the N ranks initialise the store in parallel, each over its own
    link.  Layer ℓ lives at offset ℓ·layer_bytes.
    """

    def __init__(self, name: str, layers: list[int], layer_bytes: int, rank: int, world: int, barrier=None,
                 coded: bool = False):
        self.layers = {li: i for i, li in enumerate(layers)}
        self.layer_bytes = layer_bytes
        self.rank, self.world = rank, world
        self.path = f"/dev/shm/{name}"
        self.bytes = len(layers) * layer_bytes
        if rank == 0:
            fd = os.open(self.path, os.O_RDWR | os.O_CREAT | os.O_TRUNC, 0o600)
            os.ftruncate(fd, self.bytes)
            os.close(fd)
        if barrier is not None:
            barrier()
        fd = os.open(self.path, os.O_RDWR)
        self._map = mmap.mmap(fd, self.bytes, flags=mmap.MAP_SHARED)
        os.close(fd)
        self._buf = (ctypes.c_uint8 * self.bytes).from_buffer(self._map)
        self.base = ctypes.addressof(self._buf)
        self._registered: list[int] = []
        self.coded = coded  # layer_bytes = capacity of one XC4 unit; slices are frame ranges
        self.lo, self.hi = (0, 0) if coded else slice_bounds(layer_bytes, rank, world)
        if torch.cuda.is_available() and not coded:
            for i in range(len(layers)):
                addr = self.base + i * layer_bytes + self.lo
                rc = torch.cuda.cudart().cudaHostRegister(addr, self.hi - self.lo, 0)
                if int(rc) != 0:
                    raise InsufficientTotalMemory(f"cudaHostRegister of a {self.hi - self.lo} B slice failed ({int(rc)})")
                self._registered.append(addr)

    def layer_view(self, layer: int) -> torch.Tensor:
        off = self.layers[layer] * self.layer_bytes
        return torch.frombuffer(self._buf, dtype=torch.uint8, count=self.layer_bytes, offset=off)

    def write_slice(self, layer: int, src: torch.Tensor) -> torch.Tensor:
        """Copy this rank's slice of ``src`` (the full layer, any device) into the store."""
        view = self.layer_view(layer)
        flat = src.reshape(-1).view(torch.uint8)
        view[self.lo:self.hi].copy_(flat[self.lo:self.hi])
        return view

    def write_coded(self, layer: int, enc: torch.Tensor) -> XC4Unit:
        """Store an XC4-encoded unit (``enc``: its bytes, any device): every rank
        writes the header and frame table, then only the frames it will move
        over its own link, which it page-locks."""
        nb = enc.numel()
        if nb > self.layer_bytes:
            raise InsufficientTotalMemory(f"XC4 unit of {nb} B exceeds the {self.layer_bytes} B store slot")
        view = self.layer_view(layer)
        h = native.XC4Header.from_buffer_copy(bytes(enc[:64].cpu().numpy()))
        head = 64 + 8 * (int(h.n_frames) + 1)
        view[:head].copy_(enc[:head])
        u = XC4Unit.parse(view[:nb])
        f0, f1 = u.frame_range(self.rank, self.world)
        lo, hi = int(u.frame_off[f0]), int(u.frame_off[f1])
        view[lo:hi].copy_(enc[lo:hi])
        if torch.cuda.is_available():
            base = self.base + self.layers[layer] * self.layer_bytes
            a0, a1 = (base + lo) // 4096 * 4096, (base + hi + 4095) // 4096 * 4096
            rc = torch.cuda.cudart().cudaHostRegister(a0, a1 - a0, 0)
            if int(rc) != 0:
                raise InsufficientTotalMemory(f"cudaHostRegister of {a1 - a0} B of frames failed ({int(rc)})")
            self._registered.append(a0)
        self.bytes_registered = getattr(self, "bytes_registered", 0) + (hi - lo)
        return u

    def close(self, unlink: bool = False) -> None:
        for addr in self._registered:
            torch.cuda.cudart().cudaHostUnregister(addr)
        self._registered.clear()
        if unlink and os.path.exists(self.path):
            os.unlink(self.path)


def _gloo_gather(out: torch.Tensor, mine: torch.Tensor, group) -> None:
    """All-gather through host memory: the CPU-test path, and the single-GPU
    multi-rank check (several ranks sharing one device under gloo), which
    exercises every N > 1 code path except NCCL itself."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    if out.is_cuda:
        torch.cuda.current_stream(out.device).synchronize()
        host_out = torch.empty(out.numel(), dtype=out.dtype)
        dist.all_gather(list(host_out.view(world, -1).unbind(0)), mine.cpu(), group=group)
        out.copy_(host_out)
    else:
        dist.all_gather(list(out.view(world, -1).unbind(0)), mine.clone(), group=group)


def gather_layer(slot: torch.Tensor, rank: int, world: int, group=None) -> None:
    """In-place all-gather of the 1/N slices of one layer into ``slot`` (every
    rank ends with the full layer).  NCCL reassembles over NVLink."""
    import torch.distributed as dist

    lo, hi = slice_bounds(slot.numel(), rank, world)
    if slot.is_cuda and dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(slot, slot[lo:hi], group=group)
    else:
        _gloo_gather(slot, slot[lo:hi], group)


class DiskRef:
    """A streamed layer whose unit lives in the DiskTier's file; ``meta`` is
    its XC4Unit (header and frame table, no data) or None for a raw unit."""

    __slots__ = ("layer", "nbytes", "meta")

    def __init__(self, layer: int, nbytes: int, meta):
        self.layer, self.nbytes, self.meta = layer, nbytes, meta


class DiskTier:
    """the DISK tier below pinned host DRAM.

    Reference: groups that fit neither the GPU nor the CPU go to disk
    (placement.py:241-243) and each is staged DISK → CPU one layer ahead of
    its use (prefetch_schedule, placement.py:275-282; IO_DISK events,
    simulator.py:200-207).  Here the units (raw or XC4-encoded) are appended
    to one file; a reader thread streams them, in pass order, into two
    page-locked staging buffers with ``preadv`` (the GIL is released), so the
    disk read of use j+1 overlaps the host→GPU copy of use j, and a buffer is
    refilled only after the copy engine has finished with it (a CUDA event
    recorded behind its copies)."""

    ALIGN = 1 << 21
    READERS = 8  # concurrent preadv streams per unit (NVMe queues / page-cache copies in parallel)

    def __init__(self, path: str):
        self.path = path
        self.fd = os.open(path, os.O_RDWR | os.O_CREAT | os.O_TRUNC, 0o600)
        self.entries: dict[int, tuple[int, int]] = {}   # layer → (file offset, bytes)
        self.size = 0
        self.bytes_read = 0
        self._thread = None

    def write(self, layer: int, data: torch.Tensor, meta=None) -> DiskRef:
        """Append a unit's bytes (any device) to the file."""
        buf = data.reshape(-1).view(torch.uint8)
        if buf.is_cuda:
            buf = buf.cpu()
        off = self.size
        mv = memoryview(buf.numpy())
        done = 0
        while done < len(mv):
            done += os.pwrite(self.fd, mv[done:], off + done)
        self.entries[layer] = (off, buf.numel())
        self.size = (off + buf.numel() + self.ALIGN - 1) // self.ALIGN * self.ALIGN
        return DiskRef(layer, buf.numel(), meta)

    # ---- staging pipeline (started by the streamer) ----
    def start(self, order: list[int]) -> None:
        self.order = list(order)
        cap = max(self.entries[li][1] for li in self.order)
        self.bufs = [torch.empty(cap, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
        self.copy_done = [native.Event(), native.Event()]  # recorded behind the copies that read each buffer
        self.cv = threading.Condition()
        self.filled = 0     # uses staged so far
        self.released = 0   # uses whose copies are enqueued (their buffer's event is recorded)
        self.stop = False
        self._pool = concurrent.futures.ThreadPoolExecutor(self.READERS, thread_name_prefix="disk-read")
        self._thread = threading.Thread(target=self._reader, name="disk-stage", daemon=True)
        self._thread.start()

    def _reader(self) -> None:
        dk = 0
        while True:
            with self.cv:
                # buffer dk % 2 last held use dk − 2: wait until its copies are enqueued
                while not self.stop and self.released < dk - 1:
                    self.cv.wait(0.1)
                if self.stop:
                    return
            if dk >= 2:
                self.copy_done[dk % 2].synchronize()  # the copy engine is done reading it
            off, n = self.entries[self.order[dk % len(self.order)]]
            mv = memoryview(self.bufs[dk % 2].numpy())[:n]
            list(self._pool.map(lambda r: self._read(mv, off, *r), self.pieces(n)))
            with self.cv:
                self.filled = dk + 1
                self.bytes_read += n
                self.cv.notify_all()
            dk += 1

    def pieces(self, n: int) -> list[tuple[int, int]]:
        """Byte ranges (2 MiB-aligned, ≤ READERS of them) covering an n-byte unit."""
        piece = ((n + self.READERS - 1) // self.READERS + self.ALIGN - 1) // self.ALIGN * self.ALIGN
        return [(lo, min(n, lo + piece)) for lo in range(0, n, piece)]

    def _read(self, mv, off: int, lo: int, hi: int) -> None:
        while lo < hi:
            lo += os.preadv(self.fd, [mv[lo:hi]], off + lo)

    def acquire(self, dk: int, ref: DiskRef):
        """Host view of use ``dk`` (waits for the reader): a uint8 tensor, or an
        XC4Unit over the staged bytes."""
        with self.cv:
            while self.filled <= dk:
                self.cv.wait()
        buf = self.bufs[dk % 2][: ref.nbytes]
        return buf if ref.meta is None else dataclasses.replace(ref.meta, data=buf)

    def release(self, dk: int, stream) -> None:
        """The copies reading use ``dk``'s buffer are enqueued on ``stream``."""
        self.copy_done[dk % 2].record(stream)
        with self.cv:
            self.released = dk + 1
            self.cv.notify_all()

    def close(self) -> None:
        if self._thread is not None:
            with self.cv:
                self.stop = True
                self.cv.notify_all()
            self._thread.join(timeout=5)
            self._pool.shutdown(wait=True)
        os.close(self.fd)
        if os.path.exists(self.path):
            os.unlink(self.path)


def gather_shards(slot: torch.Tensor, shard: torch.Tensor, group=None) -> None:
    """Rebuild a layer in ``slot`` from every rank's resident 1/N shard (f3).
    NCCL moves the (N−1)/N foreign bytes over NVLink; gloo (CPU tests) takes
    the list form."""
    import torch.distributed as dist

    if slot.is_cuda and dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(slot, shard, group=group)
    else:
        _gloo_gather(slot, shard, group)


class LayerStreamer:
    """Moves host-resident FFN layers through ``n_slots`` HBM slots.

    Usage on the compute stream, per layer ℓ of every pass, in layer order:
        ptr = streamer.acquire(ℓ, stream)   # waits only if ℓ is streamed
        ... expert GEMMs reading ptr ...
        streamer.release(ℓ, stream)
    Resident layers return their HBM buffer and never touch the link.

    ``segments`` (split window): the unit is moved as consecutive byte ranges
    [lo, hi) — e.g. [gate_up | down] of an FFN — each into its own slot, so the
    window holds one unit instead of two while the link still runs a whole
    unit ahead of the compute (a segment's slot frees as soon as its GEMM has
    read it).  Per layer the compute acquires segment 0, 1, … in order
    (``acquire(ℓ, stream, seg)``); the pointer returned for segment s is the
    unit's *virtual* base (slot address − lo), so unit-relative offsets keep
    working — only addresses inside [lo, hi) of that segment may be read.
    """

    RING_SLOTS = 4  # encoded frames in flight between the copy engine and the decoder (XC4 units)

    def __init__(self, layer_bytes: int, resident: dict[int, torch.Tensor], host: dict,
                 n_layer: int, device, n_slots: int = 2, chunk_bytes: int = 256 << 20, trace: bool = False,
                 rank: int = 0, world: int = 1, group=None, shards: dict[int, torch.Tensor] | None = None,
                 disk: "DiskTier | None" = None, segments: list[tuple[int, int]] | None = None):
        self.layer_bytes = layer_bytes
        self.segments = list(segments) if segments else [(0, layer_bytes)]
        S = len(self.segments)
        if (self.segments[0][0] != 0 or self.segments[-1][1] != layer_bytes
                or any(a[1] != b[0] for a, b in zip(self.segments, self.segments[1:]))
                or any(lo % 256 or hi <= lo for lo, hi in self.segments[:-1])):
            raise ValueError(f"segments must tile [0, {layer_bytes}) in 256-B aligned ranges: {self.segments}")
        if S > 1 and (world > 1 or shards or disk is not None):
            raise ValueError("a split window is single-GPU and host-DRAM only")
        if n_slots % S:
            raise ValueError(f"{n_slots} slots do not hold {S} segments per unit evenly")
        # f4: host values that are DiskRefs are staged from ``disk`` each use
        self.disk = disk
        self.disk_uses = 0
        # layers sharded across the N GPUs' HBM: rank r keeps
        # bytes slice_bounds(r) of the layer resident, and every pass rebuilds
        # the layer in a window slot with an NVLink all-gather (no host link)
        self.shards = shards or {}
        if self.shards and world < 2:
            raise ValueError("HBM-sharded layers need world > 1")
        if set(self.shards) & set(host):
            raise ValueError("a layer is either host-streamed or HBM-sharded")
        # host values are raw pinned uint8 tensors, or XC4Unit (K9: encoded
        # frames cross the link and are decoded into the slot on the GPU)
        kinds = {isinstance(v.meta if isinstance(v, DiskRef) else v, (XC4Unit, XC4Parts)) for v in host.values()}
        self.coded = kinds == {True}
        if len(kinds) > 1:
            raise ValueError("streamed layers must be all raw or all XC4-encoded")
        metas = {li: (v.meta if isinstance(v, DiskRef) else v) for li, v in host.items()}
        self.resident = resident
        self.host = host
        self.streamed = [li for li in range(n_layer) if li in host or li in self.shards]
        # one pass = every streamed layer's segments in order
        self.uses = [(li, sg) for li in self.streamed for sg in range(S)]
        self.n_slots = n_slots if self.streamed else 0
        self.chunk = chunk_bytes
        self.device = torch.device(device)
        self.copy_stream = torch.cuda.Stream(device=self.device) if host else None
        # N > 1: each rank pushes its 1/N slice over its own PCIe link, then an
        # in-place NCCL all-gather on the comm stream rebuilds the layer
        self.rank, self.world, self.group = rank, world, group
        self.lo, self.hi = slice_bounds(layer_bytes, rank, world) if world > 1 else (0, layer_bytes)
        self.comm_stream = torch.cuda.Stream(device=self.device) if (self.streamed and world > 1) else None
        self.copied = [native.Event() for _ in range(self.n_slots)] if (world > 1 and host) else []
        self.slots = [torch.empty(self.seg_bytes(j % S), dtype=torch.uint8, device=self.device)
                      for j in range(self.n_slots)]
        # events are created eagerly through the C ABI (a lazily created torch
        # event has handle 0, and record/wait on it silently no-op)
        self.loaded = [native.Event() for _ in range(self.n_slots)]
        self.free = [native.Event() for _ in range(self.n_slots)]
        self.ring = None
        if self.coded:
            for u in metas.values():
                if u.raw_bytes != layer_bytes:
                    raise ValueError(f"XC4 unit decodes to {u.raw_bytes} B, slot holds {layer_bytes} B")
                if isinstance(u, XC4Parts) != (S > 1) or (S > 1 and [p.raw_bytes for p in u.parts] != [
                        self.seg_bytes(sg) for sg in range(S)]):
                    raise ValueError("a split window streams XC4Parts encoded per segment "
                                     "(codec.encode_segments_to_host), a whole window XC4Units")
            if S == 1:
                self.frames = {li: u.frame_range(rank, world) for li, u in metas.items()}
            else:  # every segment is its own XC4 unit: all its frames, decoded from its own slot base
                self.frames = {(li, sg): (0, p.n_frames) for li, u in metas.items() for sg, p in enumerate(u.parts)}
            self.ring_slot_bytes = (max(u.max_frame_bytes() for u in metas.values()) + 255) // 256 * 256
            self.ring = torch.empty(self.RING_SLOTS * self.ring_slot_bytes, dtype=torch.uint8, device=self.device)
            self.ring_events = [native.Event() for _ in range(2 * self.RING_SLOTS)]
            self.ring_cursor = Cursor(0)
            # decode kernels jump ahead of the verify/draft kernels: they gate the next layer
            self.decode_stream = torch.cuda.Stream(device=self.device, priority=-1)
        self.k_use = 0      # global index of the next streamed use to release
        self.k_acq = 0      # global index of the next streamed use to acquire (≥ k_use)
        self.k_issued = 0   # copies enqueued so far
        self.k_base = 0     # first use of the current slot map (resize): earlier uses left no free events
        self.bytes_issued = 0      # bytes moved over this rank's host link
        self.raw_bytes_issued = 0  # layer bytes this rank's copies / shards delivered
        self.nvlink_bytes_issued = 0  # bytes this rank receives in the all-gathers
        self.trace = trace
        # (use, layer, start event, end event, resource, label)
        self.copy_marks: list[tuple] = []
        # (round, batch) of the pass that consumed each use: the engine sets
        # pass_tag before a verify pass, so a load's trace event carries the
        # round of its ffn_gpu (the reference's causality check keys on it)
        self.pass_tag: tuple | None = None
        self.use_tags: dict[int, tuple] = {}
        if disk is not None:
            disk.start([li for li in self.streamed if isinstance(host.get(li), DiskRef)])

    def seg_bytes(self, sg: int) -> int:
        lo, hi = self.segments[sg]
        return hi - lo

    @property
    def window_bytes(self) -> int:
        return sum(t.numel() for t in self.slots) + (self.ring.numel() if self.ring is not None else 0)

    def _issue(self, k: int) -> None:
        slot = k % self.n_slots
        layer, sg = self.uses[k % len(self.uses)]
        lo, hi = self.segments[sg]
        if layer in self.shards:  # f3: NVLink all-gather of the resident 1/N shards
            start = native.Event(timing=True).record(self.comm_stream) if self.trace else None
            if k - self.n_slots >= self.k_base:
                self.free[slot].wait(self.comm_stream)
            with torch.cuda.stream(self.comm_stream):
                gather_shards(self.slots[slot], self.shards[layer], self.group)
            self.loaded[slot].record(self.comm_stream)
            self.nvlink_bytes_issued += (self.world - 1) * (self.hi - self.lo)
            self.raw_bytes_issued += self.hi - self.lo
            if self.trace:
                self.copy_marks.append((k, layer, start, native.Event(timing=True).record(self.comm_stream),
                                        "IO_C2G", "ffn_load"))
            return
        if k - self.n_slots >= self.k_base and not self.coded:  # coded: the decoder waits, the link runs ahead
            self.free[slot].wait(self.copy_stream)
        src = self.host[layer]
        dk = None
        if isinstance(src, DiskRef):  # f4: the reader thread staged it in pinned memory
            dk = self.disk_uses
            self.disk_uses += 1
            src = self.disk.acquire(dk, src)
        start = None
        if self.trace:
            start = native.Event(timing=True).record(self.copy_stream)
        if self.coded:
            if len(self.segments) == 1:
                unit = src
                f0, f1 = self.frames[layer]
            else:
                unit = src.parts[sg]
                f0, f1 = self.frames[(layer, sg)]
            done = self.loaded[slot] if self.world == 1 else self.copied[slot]
            native.xc4_stream(self.slots[slot].data_ptr(), unit.data.data_ptr(), f0, f1, self.ring.data_ptr(),
                              self.ring_slot_bytes, self.ring_events, self.ring_cursor, self.copy_stream,
                              self.decode_stream, self.free[slot] if k - self.n_slots >= self.k_base else None,
                              done)
            if dk is not None:
                self.disk.release(dk, self.copy_stream)
            if self.world > 1:
                self.copied[slot].wait(self.comm_stream)
                with torch.cuda.stream(self.comm_stream):
                    gather_layer(self.slots[slot], self.rank, self.world, self.group)
                self.loaded[slot].record(self.comm_stream)
            self.bytes_issued += unit.frame_bytes(f0, f1)
            self.raw_bytes_issued += (self.hi - self.lo) if len(self.segments) == 1 else hi - lo
            if self.trace:
                # two resources (T7: one timeline per stream): the copy engine moving
                # the frames, then the decoder (and, N > 1, the all-gather) finishing the slot
                copied = native.Event(timing=True).record(self.copy_stream)
                self.copy_marks.append((k, layer, start, copied, "IO_C2G", "ffn_load_part" if sg else "ffn_load"))
                end_stream = self.decode_stream if self.world == 1 else self.comm_stream
                self.copy_marks.append((k, layer, copied, native.Event(timing=True).record(end_stream),
                                        "GPU_DECODE", "ffn_decode"))
            return
        if self.world == 1:
            native.stream_layer(self.slots[slot].data_ptr(), src.data_ptr() + lo, hi - lo, self.chunk,
                                self.copy_stream, self.loaded[slot])
            if dk is not None:
                self.disk.release(dk, self.copy_stream)
        else:
            native.stream_layer(self.slots[slot].data_ptr() + self.lo, src.data_ptr() + self.lo, self.hi - self.lo,
                                self.chunk, self.copy_stream, self.copied[slot])
            if dk is not None:
                self.disk.release(dk, self.copy_stream)
            self.copied[slot].wait(self.comm_stream)
            with torch.cuda.stream(self.comm_stream):
                gather_layer(self.slots[slot], self.rank, self.world, self.group)
            self.loaded[slot].record(self.comm_stream)
        if self.trace:
            end_stream = self.copy_stream if self.world == 1 else self.comm_stream
            self.copy_marks.append((k, layer, start, native.Event(timing=True).record(end_stream), "IO_C2G",
                                    "ffn_load_part" if sg else "ffn_load"))
        moved = (self.hi - self.lo) if len(self.segments) == 1 else hi - lo
        self.bytes_issued += moved
        self.raw_bytes_issued += moved

    def resize(self, n_slots: int) -> None:
        """Change the window's slot count between passes (nothing held).  E.g. a
        split window (one unit of HBM) for link-bound decode rounds, widened to
        two slots per segment (two units) for prefill-heavy passes, whose
        multi-chunk layers hold both segments at once and would otherwise stop
        the link for the whole layer.  Synchronises the device; copies already
        issued ahead are dropped and re-issued into the new slot map."""
        S = len(self.segments)
        if not self.streamed or n_slots == self.n_slots:
            return
        if n_slots < 2 or n_slots % S:
            raise ValueError(f"{n_slots} slots cannot hold {S} segments per unit, double-buffered")
        if self.k_acq != self.k_use:
            raise RuntimeError("resize while window slots are held")
        torch.cuda.synchronize(self.device)  # every issued copy / decode has landed; no slot is read
        self.slots = [self.slots[j] if j < len(self.slots) else
                      torch.empty(self.seg_bytes(j % S), dtype=torch.uint8, device=self.device)
                      for j in range(n_slots)]
        for evs in (self.loaded, self.free) + ((self.copied,) if self.copied else ()):
            del evs[n_slots:]
            evs.extend(native.Event() for _ in range(n_slots - len(evs)))
        self.n_slots = n_slots
        # the dropped uses are re-issued (and re-traced) under the new map
        self.copy_marks = [m for m in self.copy_marks if m[0] < self.k_use]
        self.k_issued = self.k_base = self.k_use

    def _ensure_issued(self, upto: int) -> None:
        while self.k_issued <= upto:
            self._issue(self.k_issued)
            self.k_issued += 1

    def prefetch(self) -> None:
        """Start the first window's copies (e.g. before prefill begins)."""
        if self.streamed:
            self._ensure_issued(self.k_use + self.n_slots - 1)

    def acquire(self, layer: int, stream: torch.cuda.Stream, seg: int = 0) -> int:
        """Make ``stream`` wait for segment ``seg`` of ``layer`` and return the unit's
        base address (virtual for seg > 0, see the class docstring).  Uses are
        acquired and released in pass order; up to ``n_slots`` may be held at once."""
        if layer not in self.host and layer not in self.shards:
            return self.resident[layer].data_ptr()
        k = self.k_acq
        if self.uses[k % len(self.uses)] != (layer, seg):
            raise RuntimeError(f"acquire({layer}, seg {seg}) out of pass order: next is "
                               f"{self.uses[k % len(self.uses)]}")
        if k >= self.k_use + self.n_slots:
            raise RuntimeError(f"{self.n_slots} window slots are all held: release before acquiring more")
        if self.trace and self.pass_tag is not None:
            self.use_tags[k] = self.pass_tag
        self._ensure_issued(self.k_use + self.n_slots - 1)
        self.loaded[k % self.n_slots].wait(stream)
        self.k_acq += 1
        return self.slots[k % self.n_slots].data_ptr() - self.segments[seg][0]

    def release(self, layer: int, stream: torch.cuda.Stream, seg: int = 0) -> None:
        if layer not in self.host and layer not in self.shards:
            return
        k = self.k_use
        if self.uses[k % len(self.uses)] != (layer, seg) or k >= self.k_acq:
            raise RuntimeError(f"release({layer}, seg {seg}) out of order or never acquired")
        self.free[k % self.n_slots].record(stream)
        self.k_use += 1
        # keep the link busy: the copy that waits on this release goes out now
        self._ensure_issued(self.k_use + self.n_slots - 1)
