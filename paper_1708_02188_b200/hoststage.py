"""Host-buffer collectives: PlacedBuffer(memory="host") on the GPU path.

Reference: the DDL object carries a `memory` placement (pkg/src/ringbox/
runtime.py:51-69) and `allreduce(ctx, obj)` reduces it in
place (runtime.py:295-297).  The reference only has host memory; here a host
(numpy) buffer is reduced by the GPU kernel, so its bytes must cross PCIe both
ways.  Done naively (copy in, reduce, copy out) the three phases serialise.
This module pipelines them over element windows, each window a full-geometry
allreduce of [lo, hi) (bit-identical to those elements of a whole-buffer call,
rbx_allreduce_window), on three streams:

    copy-in (H2D)  w0  w1  w2  ...
    reduce             w0  w1  w2 ...
    copy-out (D2H)         w0  w1  w2

so PCIe runs in both directions while the NVLink kernel works on the window
before.  The numpy memory itself is page-locked once (rbx_host_register,
released when the array is garbage collected) so the copies run at the host
link's DMA rate with no staging memcpy on the CPU.
"""

from __future__ import annotations

import weakref

import numpy as np

_REGISTERED: dict = {}  # base address -> nbytes of page-locked numpy memory


def _torch():
    import torch

    return torch


def pin_array(arr: np.ndarray) -> None:
    """Page-lock the memory of `arr` (cached; unregistered when the owning
    array is collected).  Best effort: if registration fails the copies still
    work, through the driver's pageable path."""
    if arr.nbytes == 0:
        return
    base = arr
    while isinstance(base.base, np.ndarray):
        base = base.base
    addr = base.__array_interface__["data"][0]
    nbytes = base.nbytes
    hit = _REGISTERED.get(addr)
    if hit is not None and hit >= nbytes:
        return
    import ctypes

    from . import _native

    L = _native.lib()
    if hit is not None:
        L.rbx_host_unregister(ctypes.c_void_p(addr))
        del _REGISTERED[addr]
    did = ctypes.c_int(0)
    if L.rbx_host_register(ctypes.c_void_p(addr), nbytes, ctypes.byref(did)) != 0:
        return  # the copies still work, through the driver's pageable path
    if not did.value:
        return  # already page-locked memory (e.g. host_empty): not ours to release
    _REGISTERED[addr] = nbytes

    def _release(a=addr):
        if _REGISTERED.pop(a, None) is not None:
            try:
                _native.lib().rbx_host_unregister(ctypes.c_void_p(a))
            except Exception:  # noqa: BLE001 -- interpreter shutdown
                pass

    weakref.finalize(base, _release)


class HostPipeline:
    """Copy-in lanes, one reduce stream, copy-out lanes, of one device.

    `lanes` copy streams per direction: each window's copies are dealt over
    them (whole ranks when there are at least `lanes` buffers, otherwise
    sub-ranges of the window), so several copy engines share each direction
    of the host link."""

    def __init__(self, device, lanes: int = 1):
        torch = _torch()
        self.device = device
        self.lanes = max(1, int(lanes))
        with torch.cuda.device(device):
            self.s_in = [torch.cuda.Stream() for _ in range(self.lanes)]
            self.s_out = [torch.cuda.Stream() for _ in range(self.lanes)]
            self.s_red = torch.cuda.Stream()

    def _pieces(self, hosts, devs, lo, hi):
        """[(lane, host slice, device slice)] covering [lo, hi) of every buffer."""
        L = self.lanes
        parts = max(1, -(-L // len(hosts)))  # sub-ranges per buffer
        out, k = [], 0
        for h, d in zip(hosts, devs):
            for a, b in window_bounds(hi - lo, parts, taper=False):
                out.append((k % L, h[lo + a:lo + b], d[lo + a:lo + b]))
                k += 1
        return out

    def run(self, pairs, n: int, windows: int, reduce, taper: bool = False, align_bytes: int = 1 << 16) -> None:
        """pairs: [(host numpy array, device tensor)], every array n elements.
        reduce(lo, hi, stream): enqueue the collective of window [lo, hi).
        Enqueued after the caller's current stream; the current stream waits
        for the last copy-out, then the host waits for it (the result is in
        the numpy arrays when this returns).  Equal windows with 64 KB-aligned
        edges and one copy lane per direction measured best (N=1, 8 x 102.4 MB:
        18.6 ms vs 21.7 ms for tapered, unaligned windows; 2 or 4 lanes per
        direction 24-28 ms; profiles/r02_e2e_probe_*_1gpu.jsonl)."""
        torch = _torch()
        cur = torch.cuda.current_stream(self.device)
        hosts = []
        for arr, _ in pairs:
            pin_array(arr)
            hosts.append(torch.from_numpy(arr))
        devs = [d for _, d in pairs]
        align = max(1, align_bytes // max(1, hosts[0].element_size())) if hosts else 1
        start = torch.cuda.Event()
        start.record(cur)
        for s in self.s_in + self.s_out + [self.s_red]:
            s.wait_event(start)
        for lo, hi in window_bounds(n, windows, taper=taper, align=align):
            pieces = self._pieces(hosts, devs, lo, hi)
            for j, s in enumerate(self.s_in):
                with torch.cuda.stream(s):
                    for lane, h, d in pieces:
                        if lane == j:
                            d.copy_(h, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(s)
                self.s_red.wait_event(ev)
            reduce(lo, hi, self.s_red)
            ev = torch.cuda.Event()
            ev.record(self.s_red)
            for j, s in enumerate(self.s_out):
                s.wait_event(ev)
                with torch.cuda.stream(s):
                    for lane, h, d in pieces:
                        if lane == j:
                            h.copy_(d, non_blocking=True)
        for s in self.s_out:
            done = torch.cuda.Event()
            done.record(s)
            cur.wait_event(done)
        cur.synchronize()


def host_empty(n: int, dtype: str = "f32") -> np.ndarray:
    """A numpy array in page-locked memory from the CUDA host allocator (torch's pinned
    pool).  Host buffers allocated this way cross PCIe ~13 % faster than malloc'd arrays
    page-locked in place (49 vs 43 GB/s each way with both directions busy,
    profiles/r02_hostmem_probe.jsonl)."""
    torch = _torch()
    tdt = {"f32": torch.float32, "f64": torch.float64, "i64": torch.int64, "i32": torch.int32,
           "f16": torch.float16}[dtype]
    return torch.empty(n, dtype=tdt, pin_memory=True).numpy()  # the array keeps the tensor alive


def window_bounds(n: int, windows: int, taper: bool = True, align: int = 1) -> list:
    """Element windows of the pipeline.  The first window's copy-in and the last
    one's copy-out are the only transfers nothing overlaps, so from 6 windows up
    the two ends are tapered (weights 1/4, 1/2, 1, ..., 1, 1/2, 1/4) unless
    `taper` is false.  Inner edges are rounded to multiples of `align` elements:
    host<->device copies that start or end off a 64 KB boundary run measurably
    slower (profiles/r02_e2e_probe_1gpu.jsonl)."""
    windows = max(1, min(windows, n)) if n else 1
    if windows < 6 or not taper:
        w = [1.0] * windows
    else:
        w = [0.25, 0.5] + [1.0] * (windows - 4) + [0.5, 0.25]
    total = sum(w)
    edges, acc = [0], 0.0
    for x in w:
        acc += x
        e = int(round(n * acc / total))
        if align > 1:
            e = int(round(e / align)) * align
        edges.append(min(e, n))
    edges[-1] = n
    return [(a, b) for a, b in zip(edges[:-1], edges[1:]) if b > a]


def default_windows(nbytes: int, cap: int = 16) -> int:
    """Pipeline depth: ~1 window per MiB up to `cap` (one 102.4 MB buffer: 12 / 16
    equal 64 KB-aligned windows reach 0.89 / 0.89 of the host link measured in the
    same run, 4 windows 0.81, profiles/r02_e2e_probe_align_1gpu.jsonl); small
    buffers stay one window (one launch, the LL kernel when it qualifies)."""
    return max(1, min(cap, nbytes >> 20))
