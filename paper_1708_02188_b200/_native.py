"""ctypes binding of librbx.so (include/rbx.h) -- the only door to the GPU path.

There is deliberately no fallback: if the shared library is missing or was
built without sm_100a kernels, importing the runtime raises.  Status codes
map to the reference's exception types (pkg/src/ringbox/runtime.py:42-48 for
CollectiveError; ValueError for bad arguments as multiring.py:165-166).
"""

from __future__ import annotations

import ctypes
import os

from .errors import CollectiveError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RBX_LIB_PATH") or os.path.join(_HERE, "librbx.so")  # override: A/B builds only

OK, ERR_INVALID, ERR_CUDA, ERR_COLLECTIVE, ERR_UNSUPPORTED = 0, 1, 2, 3, 4
DTYPE_CODES = {"f32": 0, "f64": 1, "i64": 2, "bf16": 3, "f16": 4, "i32": 5}
ITEMSIZE = {"f32": 4, "f64": 8, "i64": 8, "bf16": 2, "f16": 2, "i32": 4}
MODES = {"auto": 0, "ring_dims": 1, "fused": 2, "fused_pull": 3, "local": 4, "push": 5, "ll": 6}
OPS = {"allreduce": 0, "reduce_scatter": 1, "allgather": 2, "barrier": 3}


class IpcHandle(ctypes.Structure):
    _fields_ = [("bytes", ctypes.c_ubyte * 64)]

    def to_bytes(self) -> bytes:
        return bytes(self.bytes)

    @classmethod
    def from_raw(cls, raw: bytes) -> "IpcHandle":
        h = cls()
        ctypes.memmove(h.bytes, raw, 64)
        return h


_lib = None
_I64P = ctypes.POINTER(ctypes.c_int64)
_INTP = ctypes.POINTER(ctypes.c_int)
_VP = ctypes.c_void_p


def _sig(fn, res, *args):
    fn.restype = res
    fn.argtypes = list(args)


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback for the allreduce path)")
    L = ctypes.CDLL(LIB_PATH)
    c_int, c_i64, c_size = ctypes.c_int, ctypes.c_int64, ctypes.c_size_t
    HP = ctypes.POINTER(IpcHandle)
    _sig(L.rbx_version, c_int)
    _sig(L.rbx_last_error, ctypes.c_char_p, _INTP, _INTP)
    _sig(L.rbx_chunk_bounds, c_int, c_i64, c_i64, c_i64, _I64P, _I64P)
    _sig(L.rbx_owned_region, c_int, _INTP, c_int, c_int, c_i64, _I64P, _I64P)
    _sig(L.rbx_fold_order, c_int, _INTP, c_int, c_int, _INTP)
    _sig(L.rbx_plan_describe, c_i64, _INTP, c_int, c_int, c_i64, c_int, c_int, c_int, _I64P, c_i64)
    _sig(L.rbx_device_count, c_int, _INTP)
    _sig(L.rbx_enable_peer_access, c_int, c_int, c_int)
    _sig(L.rbx_alloc_symmetric, c_int, c_int, c_size, ctypes.POINTER(_VP), HP)
    _sig(L.rbx_free, c_int, _VP)
    _sig(L.rbx_export_buffer, c_int, _VP, HP, ctypes.POINTER(ctypes.c_uint64))
    _sig(L.rbx_comm_create, c_int, ctypes.POINTER(_VP), c_int, c_int, _INTP, c_int, c_int, c_int, c_int, HP)
    _sig(L.rbx_comm_connect, c_int, _VP, HP)
    _sig(L.rbx_comm_destroy, c_int, _VP)
    _sig(L.rbx_comm_set_timeout, c_int, _VP, ctypes.c_double)
    _sig(L.rbx_comm_info, c_int, _VP, _INTP, _INTP, _INTP, _INTP, ctypes.POINTER(ctypes.c_uint64))
    _sig(L.rbx_comm_trace, c_int, _VP, ctypes.POINTER(ctypes.c_uint64), c_int)
    _sig(L.rbx_comm_last_kernel, c_int, _VP, ctypes.POINTER(c_int))
    _sig(L.rbx_comm_inject_fault, c_int, _VP, ctypes.c_double)
    _sig(L.rbx_stamp, c_int, _VP, _VP)
    _sig(L.rbx_host_register, c_int, _VP, c_size, _INTP)
    _sig(L.rbx_host_unregister, c_int, _VP)
    _sig(L.rbx_fused_harness, c_int, _INTP, c_int, c_int, ctypes.POINTER(_VP), c_size, c_int, c_int, c_int, _VP)
    _sig(L.rbx_register_buffer, c_int, _VP, _VP, c_size, HP, ctypes.POINTER(ctypes.c_uint64), _INTP)
    _sig(L.rbx_peer_pointer, c_int, _VP, _VP, c_int, ctypes.POINTER(_VP))
    _sig(L.rbx_inbox_bytes, c_i64, _INTP, c_int, ctypes.POINTER(c_size), c_int, c_int)
    _sig(L.rbx_set_inbox, c_int, _VP, _VP, c_size, HP, ctypes.POINTER(ctypes.c_uint64))
    _sig(L.rbx_allreduce, c_int, _VP, _VP, c_size, c_int, c_int, _VP)
    _sig(L.rbx_reduce_scatter, c_int, _VP, _VP, c_size, c_int, c_int, _VP, _I64P, _I64P)
    _sig(L.rbx_allgather, c_int, _VP, _VP, c_size, c_int, c_int, _VP)
    _sig(L.rbx_allreduce_buckets, c_int, _VP, ctypes.POINTER(_VP), ctypes.POINTER(c_size), c_int, c_int, c_int, _VP)
    _sig(L.rbx_allreduce_window, c_int, _VP, _VP, c_size, c_size, c_size, c_int, c_int, _VP)
    _sig(L.rbx_vcollective_window, c_int, _VP, ctypes.POINTER(_VP), c_size, c_size, c_size, c_int, c_int, c_int, _VP)
    _sig(L.rbx_barrier, c_int, _VP, _VP)
    _sig(L.rbx_check, c_int, _VP)
    _sig(L.rbx_vcomm_create, c_int, ctypes.POINTER(_VP), c_int, _INTP, c_int, c_int, c_int, c_int)
    _sig(L.rbx_vcollective, c_int, _VP, ctypes.POINTER(_VP), c_size, c_int, c_int, c_int, _VP)
    if L.rbx_version() != 1:
        raise ImportError("librbx.so ABI version mismatch")
    _lib = L
    return L


EXPORTED = [
    "rbx_version", "rbx_last_error", "rbx_chunk_bounds", "rbx_owned_region", "rbx_fold_order", "rbx_plan_describe",
    "rbx_device_count", "rbx_enable_peer_access", "rbx_alloc_symmetric", "rbx_free", "rbx_export_buffer", "rbx_comm_create",
    "rbx_comm_connect", "rbx_comm_destroy", "rbx_comm_set_timeout", "rbx_comm_info", "rbx_comm_trace",
    "rbx_comm_last_kernel",
    "rbx_comm_inject_fault", "rbx_stamp", "rbx_fused_harness", "rbx_host_register", "rbx_host_unregister",
    "rbx_register_buffer", "rbx_peer_pointer", "rbx_inbox_bytes", "rbx_set_inbox",
    "rbx_allreduce", "rbx_reduce_scatter", "rbx_allgather", "rbx_allreduce_buckets", "rbx_allreduce_window",
    "rbx_barrier", "rbx_check", "rbx_vcomm_create", "rbx_vcollective", "rbx_vcollective_window",
]


# rbx_comm_last_kernel codes (include/rbx.h RBX_KERNEL_*)
KERNELS = {0: "none", 1: "step", 2: "fused", 3: "rings", 4: "ll", 5: "local"}


def last_kernel(comm) -> str:
    """Which kernel ran the communicator's last collective."""
    k = ctypes.c_int(0)
    check(lib().rbx_comm_last_kernel(comm, ctypes.byref(k)))
    return KERNELS.get(k.value, str(k.value))


def check(rc: int) -> None:
    if rc == OK:
        return
    rank, stage = ctypes.c_int(-1), ctypes.c_int(-1)
    msg = lib().rbx_last_error(ctypes.byref(rank), ctypes.byref(stage)).decode(errors="replace")
    if rc == ERR_INVALID:
        raise ValueError(msg)
    if rc == ERR_COLLECTIVE:
        raise CollectiveError(msg, rank=rank.value if rank.value >= 0 else None,
                              phase=stage.value if stage.value >= 0 else None)
    if rc == ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(f"librbx: {msg}")


def ints(values) -> ctypes.Array:
    values = list(values)
    return (ctypes.c_int * max(1, len(values)))(*values)


def chunk_bounds(count: int, n: int, i: int) -> tuple[int, int]:
    off, ln = ctypes.c_int64(), ctypes.c_int64()
    check(lib().rbx_chunk_bounds(count, n, i, ctypes.byref(off), ctypes.byref(ln)))
    return off.value, ln.value


def owned_region(dims, rank: int, count: int) -> tuple[int, int]:
    off, ln = ctypes.c_int64(), ctypes.c_int64()
    check(lib().rbx_owned_region(ints(dims), len(dims), rank, count, ctypes.byref(off), ctypes.byref(ln)))
    return off.value, ln.value


def fold_order(dims, rank: int) -> list:
    n = 1
    for d in dims:
        n *= d
    out = (ctypes.c_int * n)()
    check(lib().rbx_fold_order(ints(dims), len(dims), rank, out))
    return list(out)


def plan_describe(dims, rank: int, count: int, op: str = "allreduce", mode: str = "fused", dtype: str = "f32") -> list:
    cap = 1 << 16
    buf = (ctypes.c_int64 * cap)()
    n = lib().rbx_plan_describe(ints(dims), len(dims), rank, count, OPS[op], MODES[mode], DTYPE_CODES[dtype], buf, cap)
    if n < 0:
        check(ERR_INVALID)
    assert n <= cap
    return list(buf[:n])


def inbox_bytes(dims, counts, dtype: str) -> int:
    """Symmetric inbox bytes MODE_PUSH needs for these buffers (host-only)."""
    cs = (ctypes.c_size_t * max(1, len(counts)))(*counts)
    n = lib().rbx_inbox_bytes(ints(dims), len(dims), cs, len(counts), DTYPE_CODES[dtype])
    if n < 0:
        check(ERR_INVALID)
    return n


def parse_plan(words: list) -> dict:
    """Decode rbx_plan_describe output into nested dicts (tests / debugging)."""
    it = iter(words)
    nxt = lambda: next(it)  # noqa: E731
    plan = {"steps": []}
    nsteps = nxt()
    nentry = nxt()
    plan["entry"] = [nxt() for _ in range(nentry)]
    for _ in range(nsteps):
        st = {"waits": [], "sigs": [], "segs": []}
        for _ in range(nxt()):
            st["waits"].append({"slot": nxt(), "peer": nxt(), "all": nxt()})
        st["sigs"] = [nxt() for _ in range(nxt())]
        for _ in range(nxt()):
            sg = {"off": nxt(), "len": nxt()}
            ns = nxt()
            sg["src"] = [nxt() for _ in range(ns)]
            sg["ctrl"] = [nxt() for _ in range(ns)]
            sg["nlev"] = nxt()
            sg["dst"] = [nxt() for _ in range(nxt())]
            sg["tbl"], sg["head"], sg["nvec"], sg["tail"], sg["acc"] = nxt(), nxt(), nxt(), nxt(), nxt()
            st["segs"].append(sg)
        plan["steps"].append(st)
    return plan
