"""Multi-GPU allreduce executor: the drop-in for ringbox.runtime on B200.

Reference: pkg/src/ringbox/runtime.py.  Same public names and semantics:
`PlacedBuffer` (51-69), `assign` (72-79), `Workload` (82-91),
`generate_input` (94-100), `RankResult`/`LaunchReport` (103-121),
`RankContext` (159-184), `owned_region` (187-196), `reduce_scatter`
(278-284), `allgather` (287-292), `allreduce` (295-297) and `launch`
(435-589).  What changes underneath:

* one process per GPU (spawned -- CUDA is not fork-safe), host plumbing over
  torch.distributed instead of the coordinator socket;
* the socket transport + numpy `+=` are replaced by librbx.so: a persistent
  sm_100a kernel reading/writing NVLink-mapped peer buffers, synchronised by
  epoch-tagged system-scope flags (see csrc/rbx_kernel.cuh);
* results are bit-identical to the reference's reduction order.

The buffer is mutated in place and exclusively owned by the collective while
it runs.  `reduce_scatter` returns a view of the owned chunk.
"""

from __future__ import annotations

import ctypes
import hashlib
import multiprocessing as mp
import os
import queue as queue_mod
import socket
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import CollectiveError
from .exchange import agree, allgather_objects, plan_fingerprint
from .multiring import Grid, Plan, build_grid, multiring_schedule
from .ring import chunk_bounds

DTYPES = {"f32": np.float32, "f64": np.float64, "i64": np.int64}
DEFAULT_TIMEOUT_S = 30.0  # runtime.py:39

__all__ = [
    "CollectiveError", "PlacedBuffer", "assign", "Workload", "generate_input", "RankResult", "LaunchReport",
    "host_empty",
    "RankContext", "owned_region", "reduce_scatter", "allgather", "allreduce", "allreduce_buckets", "launch",
    "plan_fingerprint", "DTYPES",
]


def _torch():
    import torch

    return torch


def host_empty(n: int, dtype: str = "f32"):
    """numpy array in page-locked host memory for PlacedBuffer(memory="host"):
    the fastest host buffers for the GPU path (hoststage.host_empty)."""
    from .hoststage import host_empty as _he

    return _he(n, dtype)


def _dtype_name(t) -> str:
    torch = _torch()
    names = {torch.float32: "f32", torch.float64: "f64", torch.int64: "i64", torch.bfloat16: "bf16",
             torch.float16: "f16", torch.int32: "i32"}
    if t.dtype not in names:
        raise ValueError(f"unsupported dtype {t.dtype}")
    return names[t.dtype]


@dataclass
class PlacedBuffer:
    """A contiguous 1-D buffer plus placement metadata (the paper's DDL object,
    PAPER.md:114-123).  `data` is a CUDA tensor (memory="device") or a numpy
    array (memory="host": collectives stage it through the GPU, H2D/D2H)."""

    data: object
    host: str = "localhost"
    device: str = "cuda:0"
    memory: str = "device"

    def __post_init__(self):
        if isinstance(self.data, np.ndarray):
            self.data = np.ascontiguousarray(self.data)
            if self.memory == "device":
                self.memory = "host"
        else:
            t = self.data
            if t.dim() != 1 or not t.is_contiguous():
                raise ValueError("PlacedBuffer data must be a contiguous 1-D tensor")

    def __len__(self) -> int:
        return len(self.data)


def assign(dst: PlacedBuffer, src: PlacedBuffer) -> PlacedBuffer:
    """Copy values only; metadata of both sides is unchanged (runtime.py:72-79)."""
    if len(dst.data) != len(src.data):
        raise ValueError(f"length mismatch: {len(dst.data)} vs {len(src.data)}")
    if str(dst.data.dtype) != str(src.data.dtype):
        raise ValueError(f"dtype mismatch: {dst.data.dtype} vs {src.data.dtype}")
    if isinstance(dst.data, np.ndarray):
        s = src.data if isinstance(src.data, np.ndarray) else src.data.cpu().numpy()
        dst.data[...] = s
    else:
        torch = _torch()
        s = src.data if not isinstance(src.data, np.ndarray) else torch.from_numpy(src.data)
        dst.data.copy_(s)
    return dst


@dataclass(frozen=True)
class Workload:
    lengths: tuple
    dtype: str = "i64"
    seed: int = 0
    crash_rank: int | None = None
    crash_phase: int | None = None
    length_overrides: dict | None = None


def generate_input(workload: Workload, iteration: int, rank: int, length: int) -> np.ndarray:
    """Deterministic per-(iteration, rank) input, bit-identical to the reference."""
    rng = np.random.default_rng(workload.seed * 100003 + iteration * 1009 + rank)
    if workload.dtype == "i64":
        return rng.integers(-1000, 1001, size=length, dtype=np.int64)
    return rng.standard_normal(length).astype(DTYPES[workload.dtype])


@dataclass
class RankResult:
    rank: int
    times: list
    digests: list
    bytes_sent: int


@dataclass
class LaunchReport:
    ranks: int
    dims: tuple
    results: dict = field(default_factory=dict)
    error: str | None = None
    failed_rank: int | None = None

    @property
    def ok(self) -> bool:
        return self.error is None


def owned_region(grid: Grid, rank: int, element_count: int) -> tuple[int, int]:
    """Range owned by `rank` after the full multi-ring reduce-scatter."""
    off, length = 0, element_count
    for c, d in zip(grid.coords(rank), grid.dims):
        if d > 1:
            o, length = chunk_bounds(length, d, (c + 1) % d)
            off += o
    return off, length


class RankContext:
    """Per-process communicator state (runtime.py:159-184): grid position,
    the native comm with NVLink-mapped peer signal areas, registered buffers,
    the per-shape agreement cache and the reference-equivalent traffic counter.

    Collective: every rank of `group` must construct it (handle exchange)."""

    def __init__(self, rank: int, grid: Grid, group=None, device=None, mode: str = "auto", nblocks: int = 0,
                 threads: int = 512, timeout_s: float = DEFAULT_TIMEOUT_S, blocking: bool = True):
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError("RankContext needs a CUDA device (there is no CPU fallback for the allreduce path)")
        self.rank = rank
        self.grid = grid
        self.group = group
        self.mode = mode
        self.blocking = blocking
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else int(device))
        torch.cuda.set_device(self.device)
        self._L = _native.lib()
        self._comm = ctypes.c_void_p()
        h = _native.IpcHandle()
        dims = list(grid.dims)
        _native.check(self._L.rbx_comm_create(ctypes.byref(self._comm), rank, grid.size, _native.ints(dims), len(dims),
                                              self.device.index, nblocks, threads, ctypes.byref(h)))
        self._L.rbx_comm_set_timeout(self._comm, float(timeout_s))
        keys = agree((tuple(dims), int(nblocks), int(threads)), group, "communicator geometry")
        del keys
        handles = allgather_objects(h.to_bytes(), group)
        if len(handles) != grid.size:
            raise ValueError(f"process group has {len(handles)} ranks, grid needs {grid.size}")
        arr = (_native.IpcHandle * grid.size)(*[_native.IpcHandle.from_raw(x) for x in handles])
        _native.check(self._L.rbx_comm_connect(self._comm, arr))
        self._registered: dict = {}  # data_ptr -> (nbytes, tensor kept alive)
        self._inbox = None
        self._old_inboxes: list = []
        self._inbox_bytes = 0
        self._agreed: set = set()
        self._staging: dict = {}
        self._pipe = None  # hoststage.HostPipeline, created on the first host-buffer allreduce
        self.host_windows = int(os.environ.get("RBX_HOST_WINDOWS", "0"))  # 0: hoststage.default_windows
        self._traffic: dict = {}
        self.bytes_sent = 0
        self.plan_hash = 0

    # -- properties ------------------------------------------------------------------
    @property
    def coords(self) -> tuple:
        return self.grid.coords(self.rank)

    @property
    def launches(self) -> int:
        n = ctypes.c_uint64()
        _native.check(self._L.rbx_comm_info(self._comm, None, None, None, None, ctypes.byref(n)))
        return n.value

    @property
    def nblocks(self) -> int:
        nb = ctypes.c_int()
        _native.check(self._L.rbx_comm_info(self._comm, None, None, ctypes.byref(nb), None, None))
        return nb.value

    def last_kernel(self) -> str:
        """Which kernel ran this rank's last collective: "fused", "rings", "ll", "step"
        (the generic interpreter) or "none" -- the evidence that a call took a
        specialised path."""
        return _native.last_kernel(self._comm)

    def trace(self) -> dict:
        """Kernel timeline of the last launch (needs RBX_TRACE=1 before creation):
        microseconds since the first CTA started, for the first and last CTA."""
        buf = (ctypes.c_uint64 * 64)()
        _native.check(self._L.rbx_comm_trace(self._comm, buf, 64))
        t0 = buf[0]
        names = {0: "start", 1: "plan_staged", 2: "entry_signalled", 30: "steps_done", 31: "exit"}
        out = {"gap_from_previous_launch_us": round((buf[0] - buf[29]) / 1e3, 3) if buf[29] else None}
        for cta, base in (("first", 0), ("last", 32)):
            row = {}
            for i in range(32):
                v = buf[base + i]
                if v and i != 29:
                    nm = names.get(i) or f"step{(i - 3) // 3}_{('waited', 'worked', 'signalled')[(i - 3) % 3]}"
                    row[nm] = round((v - t0) / 1e3, 3)
            out[cta] = row
        return out

    def schedule_for(self, element_count: int):
        return multiring_schedule(self.grid, element_count)

    # -- memory ----------------------------------------------------------------------
    def empty(self, n: int, dtype="f32"):
        """Allocate and register a symmetric device buffer (collective)."""
        torch = _torch()
        tdt = {"f32": torch.float32, "f64": torch.float64, "i64": torch.int64, "bf16": torch.bfloat16,
               "f16": torch.float16, "i32": torch.int32}[dtype]
        t = torch.empty(max(n, 1), dtype=tdt, device=self.device)[:n] if n else torch.empty(0, dtype=tdt, device=self.device)
        self.register(t)
        return t

    def register(self, tensor) -> None:
        """Collective: map every rank's copy of this buffer into this process."""
        ptr = tensor.data_ptr()
        nbytes = tensor.numel() * tensor.element_size()
        hit = self._registered.get(ptr)
        if hit is not None and hit[0] >= nbytes:
            agree(("register-hit", nbytes), self.group, "buffer registration")
            return
        if nbytes == 0:
            agree(("register-empty", 0), self.group, "buffer registration")
            return
        h = _native.IpcHandle()
        off = ctypes.c_uint64()
        _native.check(self._L.rbx_export_buffer(ctypes.c_void_p(ptr), ctypes.byref(h), ctypes.byref(off)))
        items = allgather_objects((h.to_bytes(), off.value, nbytes, _dtype_name(tensor)), self.group)
        sizes = [(x[2], x[3]) for x in items]
        bad = [r for r, s in enumerate(sizes) if s != sizes[0]]
        if bad:
            raise CollectiveError(f"length mismatch: rank {bad[0]} registers {sizes[bad[0]]}, rank 0 {sizes[0]}",
                                  rank=bad[0])
        hs = (_native.IpcHandle * len(items))(*[_native.IpcHandle.from_raw(x[0]) for x in items])
        offs = (ctypes.c_uint64 * len(items))(*[x[1] for x in items])
        bid = ctypes.c_int()
        _native.check(self._L.rbx_register_buffer(self._comm, ctypes.c_void_p(ptr), nbytes, hs, offs, ctypes.byref(bid)))
        self._registered[ptr] = (nbytes, tensor)

    def peer_pointer(self, tensor, rank: int) -> int:
        """Address (in this process) of `rank`'s copy of a registered tensor."""
        out = ctypes.c_void_p()
        _native.check(self._L.rbx_peer_pointer(self._comm, ctypes.c_void_p(tensor.data_ptr()), rank, ctypes.byref(out)))
        return out.value

    def _ensure_inbox(self, counts, dtype: str, op: str, mode: int) -> None:
        """MODE_PUSH needs a symmetric inbox (~1x the buffer bytes); grow it
        collectively when a larger buffer shows up (all ranks make the same
        calls with the same counts, so they grow together)."""
        if op not in ("allreduce", "reduce_scatter", "buckets", "window"):
            return
        fp32_partials = (mode == _native.MODES["ring_dims"] and dtype in ("bf16", "f16")
                         and sum(1 for d in self.grid.dims if d > 1) > 1)
        if mode != _native.MODES["push"] and not fp32_partials:
            return
        need = _native.inbox_bytes(list(self.grid.dims), list(counts), dtype)
        if need <= self._inbox_bytes:
            return
        torch = _torch()
        nbytes = max(need, 2 * self._inbox_bytes)
        inbox = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        h = _native.IpcHandle()
        off = ctypes.c_uint64()
        _native.check(self._L.rbx_export_buffer(ctypes.c_void_p(inbox.data_ptr()), ctypes.byref(h), ctypes.byref(off)))
        items = allgather_objects((h.to_bytes(), off.value, nbytes), self.group)
        if len({x[2] for x in items}) != 1:
            raise CollectiveError("inbox size mismatch across ranks", rank=None)
        hs = (_native.IpcHandle * len(items))(*[_native.IpcHandle.from_raw(x[0]) for x in items])
        offs = (ctypes.c_uint64 * len(items))(*[x[1] for x in items])
        _native.check(self._L.rbx_set_inbox(self._comm, ctypes.c_void_p(inbox.data_ptr()), nbytes, hs, offs))
        if self._inbox is not None:
            # a CUDA graph captured earlier may still replay plans that address it
            self._old_inboxes.append(self._inbox)
        self._inbox = inbox
        self._inbox_bytes = nbytes

    def _ensure(self, tensor) -> None:
        if tensor.numel() == 0:
            return
        ptr = tensor.data_ptr()
        for base, (nb, _) in self._registered.items():
            if base <= ptr and ptr + tensor.numel() * tensor.element_size() <= base + nb:
                return
        self.register(tensor)

    def _agree_shape(self, key) -> None:
        if key not in self._agreed:
            agree(key[1:], self.group, "length")  # runtime.py:528-543 shape agreement
            self._agreed.add(key)

    # -- accounting ----------------------------------------------------------------
    def _rank_traffic(self, count: int, itemsize: int, op: str) -> int:
        """Bytes this rank sends under the reference schedule (runtime.py:218)."""
        key = (count, op)
        if key not in self._traffic:
            sched = self.schedule_for(count)
            split = next((i for i, ph in enumerate(sched.phases)
                          if ph.transfers and ph.transfers[0].combine != "add"), len(sched.phases))
            phases = {"allreduce": sched.phases, "reduce_scatter": sched.phases[:split],
                      "allgather": sched.phases[split:]}[op]
            self._traffic[key] = sum(t.length for ph in phases for t in ph.transfers if t.src == self.rank)
        return self._traffic[key] * itemsize

    # -- collectives -----------------------------------------------------------------
    def stream(self):
        return ctypes.c_void_p(_torch().cuda.current_stream(self.device).cuda_stream)

    def collective(self, op: str, tensor, mode: str | None = None) -> tuple[int, int]:
        if tensor.device != self.device:
            raise ValueError(f"tensor on {tensor.device}, communicator on {self.device}")
        if not tensor.is_contiguous():
            raise ValueError("tensor must be contiguous")
        dt = _dtype_name(tensor)
        n = tensor.numel()
        m = _native.MODES[mode or self.mode]
        if n == 0:
            self._agree_shape((tensor.data_ptr(), op, n, dt, m))
            return (0, 0)
        self._ensure(tensor)
        self._agree_shape((tensor.data_ptr(), op, n, dt, m))
        self._ensure_inbox([n], dt, op, m)
        code = _native.DTYPE_CODES[dt]
        ptr = ctypes.c_void_p(tensor.data_ptr())
        owned = (0, n)
        if op == "allreduce":
            _native.check(self._L.rbx_allreduce(self._comm, ptr, n, code, m, self.stream()))
        elif op == "reduce_scatter":
            o, l = ctypes.c_int64(), ctypes.c_int64()
            _native.check(self._L.rbx_reduce_scatter(self._comm, ptr, n, code, m, self.stream(), ctypes.byref(o),
                                                     ctypes.byref(l)))
            owned = (o.value, l.value)
        elif op == "allgather":
            _native.check(self._L.rbx_allgather(self._comm, ptr, n, code, m, self.stream()))
        else:
            raise ValueError(op)
        self.bytes_sent += self._rank_traffic(n, tensor.element_size(), op)
        if self.blocking:
            self.synchronize()
        return owned

    def allreduce_window(self, tensor, lo: int, hi: int, mode: str | None = None) -> None:
        """Allreduce only elements [lo, hi) of `tensor`, with the full buffer's
        chunk geometry and order (bit-identical to those elements of a full call)."""
        self._window(tensor, lo, hi, mode, None)
        if self.blocking:
            self.synchronize()

    def _window(self, tensor, lo: int, hi: int, mode, stream) -> None:
        dt = _dtype_name(tensor)
        n = tensor.numel()
        m = _native.MODES[mode or self.mode]
        if not 0 <= lo <= hi <= n:
            raise ValueError(f"window [{lo}, {hi}) outside [0, {n}]")
        self._ensure(tensor)
        self._agree_shape((tensor.data_ptr(), "window", n, lo, hi, dt, m))
        self._ensure_inbox([n], dt, "window", m)
        s = self.stream() if stream is None else ctypes.c_void_p(stream.cuda_stream)
        _native.check(self._L.rbx_allreduce_window(self._comm, ctypes.c_void_p(tensor.data_ptr()), n, lo, hi,
                                                   _native.DTYPE_CODES[dt], m, s))

    def allreduce_buckets(self, tensors, mode: str | None = None) -> None:
        """All buckets of a list in ONE launch (concurrent rings); each bucket is
        chunked independently exactly like Workload.lengths entries (runtime.py:390-398)."""
        if not tensors:
            return
        dt = _dtype_name(tensors[0])
        for t in tensors:
            if _dtype_name(t) != dt or t.device != self.device or not t.is_contiguous():
                raise ValueError("bucket tensors must share dtype and device and be contiguous")
            self._ensure(t)
        m = _native.MODES[mode or self.mode]
        self._agree_shape((tuple(t.data_ptr() for t in tensors), "buckets", tuple(t.numel() for t in tensors), dt, m))
        self._ensure_inbox([t.numel() for t in tensors], dt, "buckets", m)
        ptrs = (ctypes.c_void_p * len(tensors))(*[t.data_ptr() for t in tensors])
        counts = (ctypes.c_size_t * len(tensors))(*[t.numel() for t in tensors])
        _native.check(self._L.rbx_allreduce_buckets(self._comm, ptrs, counts, len(tensors), _native.DTYPE_CODES[dt], m,
                                                    self.stream()))
        for t in tensors:
            self.bytes_sent += self._rank_traffic(t.numel(), t.element_size(), "allreduce")
        if self.blocking:
            self.synchronize()

    def barrier(self) -> None:
        """Device-side flag barrier on the current stream (no data)."""
        _native.check(self._L.rbx_barrier(self._comm, self.stream()))

    def synchronize(self) -> None:
        _torch().cuda.current_stream(self.device).synchronize()
        self.check()

    def check(self) -> None:
        _native.check(self._L.rbx_check(self._comm))

    def inject_fault(self, fraction: float) -> None:
        """Arm a crash for the NEXT collective (Workload.crash_phase, runtime.py:429-432):
        this rank moves only `fraction` of its data and returns without signalling,
        so the peers' watchdogs see a rank that died mid-collective."""
        _native.check(self._L.rbx_comm_inject_fault(self._comm, float(fraction)))

    def staging(self, n: int, dtype: str):
        key = (n, dtype)
        if key not in self._staging:
            self._staging[key] = self.empty(n, dtype)
        return self._staging[key]

    def close(self) -> None:
        if getattr(self, "_comm", None):
            self._L.rbx_comm_destroy(self._comm)
            self._comm = None


_NP_DTYPES = {np.dtype(np.float32): "f32", np.dtype(np.float64): "f64", np.dtype(np.int64): "i64",
              np.dtype(np.int32): "i32", np.dtype(np.float16): "f16"}


def _host_collective(ctx: RankContext, obj: PlacedBuffer, op: str):
    """memory="host" (a numpy array, reduced in place).  allreduce: the array is
    page-locked once and streamed through a registered device buffer in element
    windows -- H2D of window k+1, the kernel on window k and D2H of window k-1
    run concurrently (hoststage.HostPipeline); each window is a full-geometry
    allreduce of its elements, so the result is bit-identical to one call.
    reduce_scatter / allgather: one H2D, the collective, one D2H."""
    from .hoststage import HostPipeline, default_windows, pin_array

    torch = _torch()
    arr = obj.data
    if arr.dtype not in _NP_DTYPES:
        raise ValueError(f"unsupported host dtype {arr.dtype}")
    dt = _NP_DTYPES[arr.dtype]
    n = len(arr)
    dev = ctx.staging(n, dt)
    if op == "allreduce" and n:
        if ctx._pipe is None:
            ctx._pipe = HostPipeline(ctx.device)
        windows = ctx.host_windows or default_windows(arr.nbytes)
        ctx._pipe.run([(arr, dev)], n, windows, lambda lo, hi, s: ctx._window(dev, lo, hi, None, s))
        ctx.bytes_sent += ctx._rank_traffic(n, arr.itemsize, "allreduce")
        ctx.check()
        return (0, n)
    pin_array(arr)
    host = torch.from_numpy(arr)
    dev.copy_(host, non_blocking=True)
    owned = ctx.collective(op, dev)
    host.copy_(dev, non_blocking=True)
    torch.cuda.current_stream(ctx.device).synchronize()
    ctx.check()
    return owned


def reduce_scatter(ctx: RankContext, obj: PlacedBuffer):
    """Reduce-scatter half; returns a view of this rank's owned chunk."""
    if isinstance(obj.data, np.ndarray):
        off, length = _host_collective(ctx, obj, "reduce_scatter")
    else:
        off, length = ctx.collective("reduce_scatter", obj.data)
    return obj.data[off:off + length]


def allgather(ctx: RankContext, obj: PlacedBuffer) -> PlacedBuffer:
    if isinstance(obj.data, np.ndarray):
        _host_collective(ctx, obj, "allgather")
    else:
        ctx.collective("allgather", obj.data)
    return obj


def allreduce(ctx: RankContext, obj: PlacedBuffer) -> PlacedBuffer:
    """In-place sum over all ranks in the reference's reduction order (one launch)."""
    if isinstance(obj.data, np.ndarray):
        _host_collective(ctx, obj, "allreduce")
    else:
        ctx.collective("allreduce", obj.data)
    return obj


def allreduce_buckets(ctx: RankContext, objs: list) -> list:
    ctx.allreduce_buckets([o.data for o in objs])
    return objs


# ----------------------------------------------------------------------------- launch
def _free_port() -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _crash_fraction(ctx: RankContext, length: int, crash_phase) -> float:
    """The reference's dying rank runs `crash_phase` of its schedule's phases
    (runtime.py:429-432); here it moves that fraction of its data."""
    phases = len(ctx.schedule_for(length).phases) if length else 0
    return min(1.0, (crash_phase or 0) / phases) if phases else 0.0


def _worker(rank: int, ranks: int, dims: tuple, wl: dict, addr: tuple, timeout_s: float, q,
            device: int | None = None) -> None:
    try:
        import torch
        import torch.distributed as dist

        os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = addr[0], str(addr[1])
        device = rank if device is None else device
        torch.cuda.set_device(device)
        dist.init_process_group("gloo", rank=rank, world_size=ranks)
        workload = Workload(**wl)
        grid = build_grid(ranks, dims)
        lengths = tuple(workload.lengths)
        ov = (workload.length_overrides or {}).get(rank, (workload.length_overrides or {}).get(str(rank)))
        if ov is not None:
            lengths = tuple(ov for _ in lengths)
        try:
            agree(plan_fingerprint(dims, workload.dtype, lengths), None, "length")
        except CollectiveError as exc:
            q.put(("error", rank, exc.rank, None, f"length mismatch: {exc}"))
            return
        ctx = RankContext(rank, grid, device=device, timeout_s=min(timeout_s, DEFAULT_TIMEOUT_S))
        ctx.plan_hash = plan_fingerprint(dims, workload.dtype, lengths)
        times, digests = [], []
        for it, length in enumerate(lengths):
            data = generate_input(workload, it, rank, length)
            buf = PlacedBuffer(torch.from_numpy(data).to(ctx.device), device=f"cuda:{device}")
            if length:
                ctx.register(buf.data)
            if workload.crash_rank == rank and it == 0:
                # fault injection (runtime.py:393-394, 429-432): die in the middle of the first
                # allreduce, after pushing `crash_phase` phases' worth of data
                try:
                    if length:
                        ctx.inject_fault(_crash_fraction(ctx, length, workload.crash_phase))
                        allreduce(ctx, buf)
                        torch.cuda.synchronize()
                finally:
                    os._exit(3)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            allreduce(ctx, buf)
            times.append(time.perf_counter() - t0)
            digests.append(hashlib.sha256(buf.data.cpu().numpy().tobytes()).hexdigest())
        q.put(("result", rank, times, digests, ctx.bytes_sent))
        ctx.close()
        dist.destroy_process_group()
    except CollectiveError as exc:
        q.put(("error", rank, exc.rank if exc.rank is not None else rank, exc.phase, str(exc)))
    except Exception as exc:  # surfaced through the report
        q.put(("error", rank, rank, None, f"{type(exc).__name__}: {exc}"))


def launch(ranks: int, plan, workload: Workload, rendezvous=None, timeout_s: float = DEFAULT_TIMEOUT_S, *,
           share_gpus: bool = False) -> LaunchReport:
    """Spawn one process per GPU and run the workload's allreduces
    (runtime.py:435-589).  Needs `ranks` visible CUDA devices, unless
    `share_gpus` places the ranks on the GPUs round-robin (time-sliced
    contexts: correct, not fast -- for testing the N-rank path on a small box)."""
    dims = plan.grid.dims if isinstance(plan, Plan) else tuple(plan)
    build_grid(ranks, dims)
    report = LaunchReport(ranks=ranks, dims=dims)
    torch = _torch()
    ngpu = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if ngpu < 1 or (ngpu < ranks and not share_gpus):
        report.error = f"launch needs {ranks} CUDA devices, found {ngpu} (no CPU fallback)"
        return report
    addr = rendezvous if rendezvous is not None else ("127.0.0.1", _free_port())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    wl = dict(lengths=tuple(workload.lengths), dtype=workload.dtype, seed=workload.seed,
              crash_rank=workload.crash_rank, crash_phase=workload.crash_phase,
              length_overrides=dict(workload.length_overrides) if workload.length_overrides else None)
    procs = {r: ctx.Process(target=_worker, args=(r, ranks, dims, wl, addr, timeout_s, q, r % ngpu), daemon=True)
             for r in range(ranks)}
    for p in procs.values():
        p.start()
    deadline = time.monotonic() + max(timeout_s, 60.0) + 60.0  # + CUDA/process start-up
    pending = set(range(ranks))

    def finish(error=None, rank=None):
        report.error, report.failed_rank = error, rank
        for p in procs.values():
            if p.is_alive():
                p.terminate()
        for p in procs.values():
            p.join(timeout=10)
        return report

    while pending:
        if time.monotonic() > deadline:
            return finish(f"timeout waiting for ranks {sorted(pending)}")
        try:
            msg = q.get(timeout=0.2)
        except queue_mod.Empty:
            for r, p in procs.items():
                if r in pending and not p.is_alive() and p.exitcode not in (0, None):
                    return finish(f"worker rank {r} crashed before reporting a result", r)
            continue
        if msg[0] == "result":
            _, r, times, digests, sent = msg
            report.results[r] = RankResult(r, times, digests, sent)
            pending.discard(r)
        else:
            _, r, culprit, phase, text = msg
            # A peer that died makes the survivors fail too (lost connection or
            # watchdog); give the dead process a moment to be reaped so the
            # failure is attributed to it, as the reference's liveness polling does.
            dead = []
            t_wait = time.monotonic() + 5.0
            while not dead and time.monotonic() < t_wait:
                dead = [x for x, p in procs.items() if not p.is_alive() and p.exitcode not in (0, None)]
                if not dead:
                    time.sleep(0.1)
            if dead:
                culprit = dead[0]
            suffix = f" (phase {phase})" if phase is not None else ""
            return finish(f"rank {culprit} failed: {text}{suffix}", culprit)
    return finish()
