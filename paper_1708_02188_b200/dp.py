"""Data-parallel gradient reduction driven directly by autograd (no DDP).

SURVEY.md section 8(f) item 1 / BASELINE config 5: the paper's DDL sits under a
framework and reduces gradient buckets while backward still runs.  The
reference itself has no training integration (pkg/src/ringbox/bench.py:5-6);
its bucket semantics are `Workload.lengths` -- one allreduce per bucket, each
chunked on its own (pkg/src/ringbox/runtime.py:82-91, 390-398).

`MultiringDataParallel` keeps every parameter's `.grad` as a view into ONE
registered (symmetric) fp32 arena laid out bucket by bucket, so the kernel
reduces gradients in place with no bucket copies:

* buckets follow DDP's assignment (reverse parameter order, first bucket capped
  at 1 MiB, then 25 MiB; a bucket closes once it reaches its cap);
* a post-accumulate-grad hook counts each bucket's parameters; when bucket k
  is complete, buckets are launched strictly in index order (every rank must
  issue the same launch sequence: launches of a communicator pair up by epoch)
  on a communication stream that first waits for the backward stream;
* at the end of backward the backward stream waits for the communication
  stream, so `optimizer.step()` sees averaged gradients.

Everything it launches is stream-ordered and free of host synchronisation, so
a whole training step (forward, backward, bucket allreduces, optimizer) can be
captured into one CUDA graph and replayed: `capture(step_fn)`.  The bucket
kernels then sit on graph branches parallel to the remaining backward nodes,
exactly as in eager mode, and the host launch cost of the step disappears.

`comm="nccl"` runs the same arena/hook machinery with `dist.all_reduce`
instead of the multi-ring kernel (comparison only).
"""

from __future__ import annotations

import contextlib
import ctypes


def ddp_bucket_assignment(sizes_bytes, first_cap: int = 1 << 20, cap: int = 25 << 20):
    """DDP's size-based bucketing over parameters in the given order: a bucket
    closes as soon as it reaches its cap (the first bucket's cap is 1 MiB)."""
    buckets, cur, cur_bytes, limit = [], [], 0, first_cap
    for i, nb in enumerate(sizes_bytes):
        cur.append(i)
        cur_bytes += nb
        if cur_bytes >= limit:
            buckets.append(cur)
            cur, cur_bytes, limit = [], 0, cap
    if cur:
        buckets.append(cur)
    return buckets


class BucketTracker:
    """Which buckets may be launched as gradients become ready (host logic of
    one backward pass, CPU-testable).  Buckets launch strictly in index order
    -- every rank must issue the same launch sequence, because launches of a
    communicator pair up by epoch -- each exactly once, and only when all of
    its parameters are ready; `finish()` releases the rest (parameters that
    got no gradient this pass)."""

    def __init__(self, bucket_sizes):
        self.sizes = list(bucket_sizes)
        self.active = False
        self._pending = []
        self._next = 0

    def start(self) -> None:
        self.active = True
        self._pending = list(self.sizes)
        self._next = 0

    def ready(self, k: int) -> list:
        """One parameter of bucket k is ready; returns the buckets to launch now."""
        if self._pending[k] <= 0:
            raise RuntimeError(f"bucket {k}: more gradients than parameters in one backward pass")
        self._pending[k] -= 1
        out = []
        while self._next < len(self.sizes) and self._pending[self._next] == 0:
            out.append(self._next)
            self._next += 1
        return out

    def finish(self) -> list:
        out = list(range(self._next, len(self.sizes)))
        self._next = len(self.sizes)
        self.active = False
        return out


class MultiringDataParallel:
    def __init__(self, module, ctx=None, comm: str = "multiring", group=None, bucket_cap_mb: float = 25.0,
                 first_bucket_mb: float = 1.0, average: bool = True, mode: str | None = None):
        import torch
        import torch.distributed as dist

        if comm not in ("multiring", "nccl"):
            raise ValueError(f"unknown comm {comm!r}")
        if comm == "multiring" and ctx is None:
            raise ValueError("comm='multiring' needs a RankContext")
        self.module = module
        self.ctx = ctx
        self.comm = comm
        self.group = group
        self.mode = mode
        self.params = [p for p in module.parameters() if p.requires_grad]
        if not self.params:
            raise ValueError("module has no trainable parameters")
        dev = self.params[0].device
        if any(p.device != dev or p.dtype != torch.float32 for p in self.params):
            raise ValueError("all trainable parameters must be fp32 on one device")
        self.device = dev
        self.world = ctx.grid.size if ctx is not None else dist.get_world_size(group)
        self.scale = 1.0 / self.world if average else 1.0
        order = list(reversed(self.params))  # gradients become ready roughly back to front
        idx = ddp_bucket_assignment([p.numel() * 4 for p in order], int(first_bucket_mb * (1 << 20)),
                                    int(bucket_cap_mb * (1 << 20)))
        self.buckets = [[order[i] for i in b] for b in idx]
        total = sum(p.numel() for p in self.params)
        self.arena = ctx.empty(total, "f32") if comm == "multiring" else torch.empty(total, device=dev)
        self.arena.zero_()
        self.ranges = []
        self._bucket_of = {}
        self._ptr = {}
        off = 0
        for k, b in enumerate(self.buckets):
            lo = off
            for p in b:
                # same strides as the parameter (channels_last weights stay channels_last)
                p.grad = torch.as_strided(self.arena, p.size(), p.stride(), off)
                self._bucket_of[id(p)] = k
                self._ptr[id(p)] = p.grad.data_ptr()
                off += p.numel()
            self.ranges.append((lo, off))
        self.stream = torch.cuda.Stream(device=dev)
        self._launch_args = {}
        self._tracker = BucketTracker([len(b) for b in self.buckets])
        self._sync = True
        self.launched = 0
        self._hooks = [p.register_post_accumulate_grad_hook(self._on_grad) for p in self.params]

    # -- autograd side ---------------------------------------------------------------
    def __call__(self, *args, **kwargs):
        return self.module(*args, **kwargs)

    def zero_grad(self) -> None:
        """Zero the whole arena in one memset (`.grad` must stay views of it:
        do not use optimizer.zero_grad(set_to_none=True))."""
        self.arena.zero_()

    @contextlib.contextmanager
    def no_sync(self):
        """Accumulate gradients locally (no bucket allreduces) for the backward
        passes inside the block, like DDP.no_sync(); the first backward after it
        reduces the accumulated gradients."""
        prev, self._sync = self._sync, False
        try:
            yield
        finally:
            self._sync = prev

    def _on_grad(self, p) -> None:
        import torch

        if not self._sync:
            return
        if not self._tracker.active:
            self._tracker.start()
            torch.autograd.Variable._execution_engine.queue_callback(self._finish)
        if p.grad is None or p.grad.data_ptr() != self._ptr[id(p)]:
            raise RuntimeError("a parameter's .grad is no longer a view of the gradient arena "
                               "(zero_grad(set_to_none=True)?); use MultiringDataParallel.zero_grad()")
        for k in self._tracker.ready(self._bucket_of[id(p)]):
            self._launch(k)

    def _finish(self) -> None:
        import torch

        for k in self._tracker.finish():  # parameters that got no gradient this step
            self._launch(k)
        torch.cuda.current_stream(self.device).wait_stream(self.stream)

    def _launch(self, k: int) -> None:
        import torch

        lo, hi = self.ranges[k]
        t = self.arena[lo:hi]
        self.stream.wait_stream(torch.cuda.current_stream(self.device))
        if self.comm == "multiring":
            args = self._launch_args.get(k)
            if args is None:
                args = self._launch_args[k] = self._prepare(t)
            rc = self.ctx._L.rbx_allreduce(*args)
            if rc:
                from . import _native

                _native.check(rc)
        else:
            import torch.distributed as dist

            with torch.cuda.stream(self.stream):
                dist.all_reduce(t, group=self.group)
        if self.scale != 1.0:
            with torch.cuda.stream(self.stream):
                t.mul_(self.scale)
        self.launched += 1

    def _prepare(self, t):
        """First launch of a bucket (collective, same order on every rank):
        agree on its shape and cache the C-ABI arguments."""
        from . import _native

        ctx = self.ctx
        n = t.numel()
        m = _native.MODES[self.mode or ctx.mode]
        ctx._ensure(t)
        ctx._agree_shape((t.data_ptr(), "allreduce", n, "f32", m))
        ctx._ensure_inbox([n], "f32", "allreduce", m)
        return (ctx._comm, ctypes.c_void_p(t.data_ptr()), ctypes.c_size_t(n), ctypes.c_int(_native.DTYPE_CODES["f32"]),
                ctypes.c_int(m), ctypes.c_void_p(self.stream.cuda_stream))

    # -- whole-step CUDA graph -----------------------------------------------------------
    def capture(self, step_fn, warmup: int = 3):
        """Run `step_fn` eagerly `warmup` times (plans, registrations, cuDNN
        autotuning, optimizer state), then capture one call into a CUDA graph.
        Returns the graph; `graph.replay()` runs a whole step."""
        import torch

        side = torch.cuda.Stream(device=self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(side):
            for _ in range(warmup):
                step_fn()
        torch.cuda.current_stream(self.device).wait_stream(side)
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step_fn()
        return g

    def close(self) -> None:
        for h in self._hooks:
            h.remove()
        self._hooks = []
