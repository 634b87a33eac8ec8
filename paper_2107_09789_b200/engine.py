"""Device plumbing: CUDA device/stream selection, arenas, host<->device staging.

PyTorch is used only as the CUDA memory / stream / collective layer; every
computation on the hot path is a libtobf.so kernel. There is no CPU fallback:
without a CUDA device or the native library, :func:`device` raises.
"""

from __future__ import annotations

import collections
import ctypes as C
import os
import weakref

import numpy as np
import torch

from . import _native


_TORCH_DTYPE = {np.dtype(k): v for k, v in ((np.float32, torch.float32), (np.float64, torch.float64),
                                               (np.int32, torch.int32), (np.int64, torch.int64),
                                               (np.uint8, torch.uint8), (np.int8, torch.int8),
                                               (np.int16, torch.int16), (np.uint64, torch.uint64),
                                               (np.uint32, torch.uint32), (np.bool_, torch.bool))}


class DeviceUnavailable(RuntimeError):
    pass


_CTX = None


class DeviceContext:
    """Per-process (= per-GPU) engine context: library handle, device, stream."""

    def __init__(self, index: int | None = None):
        if not torch.cuda.is_available():
            raise DeviceUnavailable("no CUDA device visible: the tobf engine has no CPU fallback")
        self.lib = _native.load()
        if index is None:
            index = int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count()
        self.index = index
        self.device = torch.device("cuda", index)
        torch.cuda.set_device(self.device)
        self.stream = torch.cuda.current_stream(self.device)
        self.sms = torch.cuda.get_device_properties(self.device).multi_processor_count
        # cache of device copies of host weight arrays, keyed by id(base array);
        # the base array is held so ids are never recycled while cached
        self.weight_cache: dict[int, tuple[np.ndarray, torch.Tensor]] = {}
        self.weight_cache_bytes = 0
        self.weight_cache_limit = int(os.environ.get("TOBF_WEIGHT_CACHE_BYTES", str(24 << 30)))
        self.pinned_cache: dict[int, tuple] = {}
        self.pinned_bytes = 0
        self.launches = 0      # libtobf kernel launches issued (bench evidence)
        self.h2d_bytes = 0     # host->device bytes staged through this context
        self.wimg_bytes = 0    # bytes of packed weight images in wimg_cache

    def side_streams(self, n: int) -> list:
        """``n`` extra engine streams (created once, reused), at the highest
        stream priority: the work put on them (the latency-bound attacker
        recurrences) is dispatched ahead of the persistent conv grids whenever
        SMs free up, so it overlaps the forward instead of queueing behind it."""
        ss = self.__dict__.setdefault("_side", [])
        if not ss:
            self._side_priority = torch.cuda.Stream.priority_range()[1]  # (low, high): high is the smaller
        while len(ss) < n:
            ss.append(torch.cuda.Stream(self.device, priority=self._side_priority))
        return ss[:n]

    @property
    def sp(self) -> int:
        """Raw cudaStream_t of the engine stream."""
        return self.stream.cuda_stream

    def check(self, rc: int, what: str) -> None:
        _native.check(rc, what)

    # -- host arrays -> device ----------------------------------------------
    RING_BYTES = 64 << 20

    def _staged(self, raw: np.ndarray, dst: torch.Tensor | None = None) -> torch.Tensor:
        """Stream-ordered H2D of ``raw`` (uint8) through a pinned staging ring
        allocated once: no per-upload page pinning (a cudaHostAlloc can stall
        the host behind queued device work) and no pageable copy. A ring
        region is rewritten only after the copy that last read it completed."""
        n = raw.nbytes
        self.h2d_bytes += n
        if n > self.RING_BYTES // 4:
            src = torch.from_numpy(raw.copy()).pin_memory()
            if dst is not None:
                dst.copy_(src, non_blocking=True)
                return dst
            return src.to(self.device, non_blocking=True)
        ring = self.__dict__.get("_ring")
        if ring is None:
            ring = self._ring = torch.empty(self.RING_BYTES, dtype=torch.uint8, pin_memory=True)
            self._ring_np, self._ring_off, self._ring_busy = ring.numpy(), 0, collections.deque()
        lo = self._ring_off if self._ring_off + n <= self.RING_BYTES else 0
        hi = lo + n
        busy = self._ring_busy
        while busy and busy[0][2].query():
            busy.popleft()
        for blo, bhi, ev in busy:
            if blo < hi and lo < bhi:
                ev.synchronize()
        self._ring_np[lo:hi] = raw
        dev = torch.empty(n, dtype=torch.uint8, device=self.device) if dst is None else dst
        dev.copy_(ring[lo:hi], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.device))  # the stream the copy was issued on
        busy.append((lo, hi, ev))
        self._ring_off = (hi + 255) & ~255
        return dev

    def upload_bytes(self, buf: bytes | bytearray | memoryview) -> torch.Tensor:
        return self._staged(np.frombuffer(buf, dtype=np.uint8))

    def upload_array(self, a: np.ndarray) -> torch.Tensor:
        """Stream-ordered H2D of a small host array (never a hidden
        synchronising pageable copy)."""
        a = np.ascontiguousarray(a)
        td = _TORCH_DTYPE.get(a.dtype)
        if td is None:
            raise TypeError(f"upload_array: unsupported dtype {a.dtype}")
        return self._staged(a.reshape(-1).view(np.uint8)).view(td).reshape(a.shape)

    def upload_struct_array(self, arr) -> torch.Tensor:
        return self.upload_bytes(memoryview(arr).cast("B"))

    def cached_view(self, a: np.ndarray) -> tuple[int, tuple[int, ...]]:
        """Device address of ``a[0, ..., 0]`` and ``a``'s element strides, with
        views sharing one upload of their base buffer (cached by identity;
        the base array is held so its id cannot be recycled while cached)."""
        base = _root(a)
        if base.dtype == np.float32 and base.flags.c_contiguous and a.dtype == np.float32:
            key = id(base)
            hit = self.weight_cache.get(key)
            if hit is None or hit[0] is not base:
                dev = self._pinned_copy(base)
                self.h2d_bytes += base.nbytes
                self._remember(key, base, dev)
            dev = self.weight_cache[key][1]
            off = (a.__array_interface__["data"][0] - base.__array_interface__["data"][0]) // 4
            return dev.data_ptr() + 4 * off, tuple(st // 4 for st in a.strides)
        own = np.ascontiguousarray(a, dtype=np.float32)
        key = id(a)
        hit = self.weight_cache.get(key)
        if hit is None or hit[0] is not a:
            dev = self._pinned_copy(own, cache=False)
            self.h2d_bytes += own.nbytes
            self._remember(key, a, dev)
        return self.weight_cache[key][1].data_ptr(), tuple(st // 4 for st in own.strides)

    def _pinned_copy(self, a: np.ndarray, cache: bool = True) -> torch.Tensor:
        """Copy ``a`` (possibly read-only) to the device, stream-ordered, from
        a pinned host mirror kept per host array: clear_cache() drops device
        copies only, so a re-upload is one DMA, not a pageable memcpy."""
        hit = self.pinned_cache.get(id(a)) if cache else None
        if hit is None or hit[0] is not a:
            host = torch.empty(a.size, dtype=torch.float32, pin_memory=True)
            host.numpy()[:] = a.reshape(-1)
            if self.pinned_bytes > self.weight_cache_limit:
                self.pinned_cache.clear()
                self.pinned_bytes = 0
            hit = (a, host)
            if cache:
                self.pinned_cache[id(a)] = hit
                self.pinned_bytes += a.nbytes
        return hit[1].to(self.device, non_blocking=True)

    def _remember(self, key, base, dev) -> None:
        if self.weight_cache_bytes > self.weight_cache_limit:
            self.weight_cache.clear()
            self.weight_cache_bytes = 0
            # packed images and staged constants are keyed by the DEVICE address
            # of their source upload: once those uploads are dropped a new one
            # can land at the same address, so the derived caches go too (runs
            # already linked hold their own buffers: PlanTables.keep)
            self.reset_wimg()
            self.__dict__.pop("const_cache", None)
        self.weight_cache[key] = (base, dev)
        self.weight_cache_bytes += dev.numel() * 4

    WIMG_LIMIT = int(os.environ.get("TOBF_WIMG_CACHE_BYTES", str(32 << 30)))

    def reset_wimg(self) -> None:
        """Forget every packed weight image (their memory returns to torch's
        stream-ordered caching allocator: reuse waits for the engine-stream
        work already queued)."""
        self.__dict__.pop("wimg_cache", None)
        self.wimg_bytes = 0

    def clear_cache(self) -> None:
        """Drop every device copy of host arrays (weights, folded BatchNorm,
        staged constants, packed images): the next run re-uploads everything
        it needs."""
        self.weight_cache.clear()
        self.weight_cache_bytes = 0
        self.__dict__.pop("affine_cache", None)
        self.__dict__.pop("const_cache", None)
        self.reset_wimg()

    def sync(self) -> None:
        self.stream.synchronize()
        rc = self.lib.tobf_check_fault(C.c_void_p(self.sp))
        if rc != 0 and self.__dict__.get("splitk_cnt") is not None:
            self.splitk_cnt.zero_()  # a drained (faulted) launch may leave split-K counters mid-count
        self.check(rc, "device pipeline")


class Readback:
    """One batch's results on their way to the host: stream-ordered D2H copies
    into pinned buffers plus the device fault word, enqueued right behind the
    batch's last kernel. ``wait`` blocks on that point only, so later batches
    already queued on the engine stream keep the device busy meanwhile (a
    ``.cpu()`` or stream synchronise would wait for them too)."""

    def __init__(self, ctx: "DeviceContext", tensors: dict[str, torch.Tensor]):
        self.ctx = ctx
        with torch.cuda.stream(ctx.stream):
            self.host = {}
            for k, t in tensors.items():
                h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
                h.copy_(t, non_blocking=True)
                self.host[k] = h
            self.fault = torch.zeros(1, dtype=torch.int32, pin_memory=True)
            ctx.check(ctx.lib.tobf_fault_async(C.c_void_p(self.fault.data_ptr()), C.c_void_p(ctx.sp)),
                      "fault word read")
            self.done = torch.cuda.Event()
            self.done.record(ctx.stream)

    def wait(self) -> dict[str, np.ndarray]:
        self.done.synchronize()
        if int(self.fault[0]) != 0:
            self.ctx.sync()  # raises TOBF_E_FAULT (and clears the word)
        return {k: h.numpy() for k, h in self.host.items()}


def cat_records(arrs: list, dtype: np.dtype) -> np.ndarray:
    """np.concatenate for structured record arrays of one dtype, through
    opaque void views: numpy 2 otherwise re-promotes every (nested) field per
    call, ~1 ms for a batch of descriptor tables."""
    if not arrs:
        return np.zeros(0, dtype)
    v = np.dtype((np.void, dtype.itemsize))
    return np.concatenate([np.ascontiguousarray(a).view(v) for a in arrs]).view(dtype)


def _root(a: np.ndarray) -> np.ndarray:
    """The ndarray owning ``a``'s memory, also through as_strided views (whose
    ``.base`` is numpy's DummyArray holding the source array)."""
    base = a
    while True:
        b = base.base
        if isinstance(b, np.ndarray):
            base = b
        elif isinstance(getattr(b, "base", None), np.ndarray):
            base = b.base
        else:
            return base


def device(index: int | None = None) -> DeviceContext:
    global _CTX
    if _CTX is None:
        _CTX = DeviceContext(index)
    return _CTX


class Arena:
    """One device allocation carved into 256-B aligned float32 slices."""

    def __init__(self, ctx: DeviceContext, floats: int):
        self.ctx = ctx
        self.buf = torch.empty(max(floats, 64), dtype=torch.float32, device=ctx.device)
        self.base = self.buf.data_ptr()
        self.used = 0

    @staticmethod
    def round(n: int) -> int:
        return (n + 63) // 64 * 64

    def take(self, floats: int) -> int:
        off = self.used
        self.used += self.round(floats)
        if self.used > self.buf.numel():
            raise MemoryError("arena overflow")
        return self.base + off * 4

    def view(self, ptr: int, floats: int) -> torch.Tensor:
        off = (ptr - self.base) // 4
        return self.buf[off:off + floats]
