"""All ranks of a grid on ONE GPU, in ONE launch.

Two uses:
* `mode="local"` -- the 1-GPU local-reduce roofline (north_star "1 GPU (local
  reduce/copy roofline)"): every owned region is folded from the V rank
  buffers in the reference order and written to all V buffers; HBM-bound,
  no flags.
* any other mode -- the exact multi-rank kernel (flags, epochs, pushes,
  per-dimension stages) with each rank played by a CTA group of a single
  cooperative launch, so the synchronisation logic is testable on one GPU
  without running rank kernels that wait on each other as separate launches.
"""

from __future__ import annotations

import ctypes

from . import _native
from .runtime import _dtype_name


class VirtualRanks:
    def __init__(self, dims, device: int = 0, nblocks_per_rank: int = 0, threads: int = 512, timeout_s: float = 30.0,
                 peer_devices=()):
        """peer_devices: other GPUs whose memory rank buffers may live in (the
        single launch on `device` then reads/writes them over NVLink)."""
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("VirtualRanks needs a CUDA device (no CPU fallback)")
        self.dims = tuple(dims)
        n = 1
        for d in self.dims:
            n *= d
        self.nranks = n
        self.device = torch.device("cuda", device)
        self._L = _native.lib()
        self._comm = ctypes.c_void_p()
        _native.check(self._L.rbx_vcomm_create(ctypes.byref(self._comm), n, _native.ints(self.dims), len(self.dims),
                                               device, nblocks_per_rank, threads))
        self._L.rbx_comm_set_timeout(self._comm, float(timeout_s))
        self.devices = {self.device.index}
        for p in peer_devices:
            _native.check(self._L.rbx_enable_peer_access(device, int(p)))
            self.devices.add(int(p))

    @property
    def launches(self) -> int:
        v = ctypes.c_uint64()
        _native.check(self._L.rbx_comm_info(self._comm, None, None, None, None, ctypes.byref(v)))
        return v.value

    @property
    def nblocks(self) -> int:
        v = ctypes.c_int()
        _native.check(self._L.rbx_comm_info(self._comm, None, None, ctypes.byref(v), None, None))
        return v.value

    def collective(self, tensors: list, op: str = "allreduce", mode: str = "fused", stream=None, window=None) -> None:
        """window=(lo, hi): only elements [lo, hi), with the full buffers' chunk
        geometry and reduction order (bit-identical to a full call there)."""
        import torch

        if len(tensors) != self.nranks:
            raise ValueError(f"need {self.nranks} buffers, got {len(tensors)}")
        n = tensors[0].numel()
        dt = _dtype_name(tensors[0])
        for t in tensors:
            if t.numel() != n or _dtype_name(t) != dt or not t.is_contiguous() or t.device.index not in self.devices:
                raise ValueError("virtual-rank buffers must match in length/dtype/device and be contiguous")
        ptrs = (ctypes.c_void_p * self.nranks)(*[t.data_ptr() for t in tensors])
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        lo, hi = window if window is not None else (0, n)
        _native.check(self._L.rbx_vcollective_window(self._comm, ptrs, n, lo, hi, _native.DTYPE_CODES[dt],
                                                     _native.OPS[op], _native.MODES[mode],
                                                     ctypes.c_void_p(s.cuda_stream)))

    def allreduce_host(self, arrays: list, mode: str = "local", windows: int | None = None) -> list:
        """Every rank's buffer is a host (numpy) array, reduced in place: the
        arrays are page-locked once and streamed through device buffers in
        element windows, H2D / kernel / D2H overlapped on three streams
        (hoststage.HostPipeline; each window bit-identical to a full call)."""
        import torch

        from .hoststage import HostPipeline, default_windows

        if len(arrays) != self.nranks:
            raise ValueError(f"need {self.nranks} arrays, got {len(arrays)}")
        n = len(arrays[0])
        if any(len(a) != n or a.dtype != arrays[0].dtype for a in arrays):
            raise ValueError("virtual-rank arrays must match in length and dtype")
        key = (n, str(arrays[0].dtype))
        staging = getattr(self, "_staging", {})
        self._staging = staging
        if key not in staging:
            tdt = torch.from_numpy(arrays[0][:0]).dtype
            staging.clear()
            staging[key] = [torch.empty(n, dtype=tdt, device=self.device) for _ in range(self.nranks)]
        devs = staging[key]
        if getattr(self, "_pipe", None) is None:
            self._pipe = HostPipeline(self.device)
        w = windows or default_windows(arrays[0].nbytes * self.nranks, cap=12)
        self._pipe.run(list(zip(arrays, devs)), n, w,
                       lambda lo, hi, s: self.collective(devs, mode=mode, stream=s, window=(lo, hi)))
        self.check()
        return arrays

    def last_kernel(self) -> str:
        """Which kernel ran the last collective ("local", "fused", "rings", "ll", "step")."""
        return _native.last_kernel(self._comm)

    def check(self) -> None:
        _native.check(self._L.rbx_check(self._comm))

    def close(self) -> None:
        if self._comm:
            self._L.rbx_comm_destroy(self._comm)
            self._comm = None
