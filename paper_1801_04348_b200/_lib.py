"""ctypes binding of libpk.so (include/pk.h).

The product path has no CPU fallback: if libpk.so is missing or fails to
load, every call raises ``RuntimeError`` naming the library, and compute
calls additionally require a visible CUDA device.
"""

from __future__ import annotations

import ctypes
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
# PK_LIB_PATH selects an alternative build of the same ABI (kernel-variant experiments)
LIB_PATH = os.environ.get("PK_LIB_PATH") or os.path.join(PKG, "libpk.so")

# status codes (pk.h)
PK_OK = 0
PK_E_PARAM = 1
PK_E_BOUNDS = 2
PK_E_DIV0 = 3
PK_E_UNSUPPORTED = 4
PK_E_CUDA = 5
PK_E_ALLOC = 6

# families
FAMILY_IDS = {
    "reverse": 1,
    "transpose": 2,
    "jacobi": 3,
    "jacobi2d": 4,
    "matvec": 5,
    "matmul": 6,
    "addition": 7,
}

VARIANT_STAGED = 0
VARIANT_DIRECT = 1

FLAG_GRANULARITY = 0x1
FLAG_TEMPORAL = 0x2
FLAG_MERGED = 0x4
FLAG_GENERIC = 0x8
FLAG_TF32X3 = 0x10
FLAG_NARROW = 0x20

DTYPE_I32 = 0
DTYPE_F32 = 1
DTYPE_I64 = 2
DTYPE_F64 = 3
DTYPE_NAMES = {DTYPE_I32: "i32", DTYPE_F32: "f32", DTYPE_I64: "i64", DTYPE_F64: "f64"}

# every symbol include/pk.h declares
EXPORTS = (
    "pk_query_machine",
    "pk_launch",
    "pk_launch_checked",
    "pk_required_elems",
    "pk_run_host",
    "pk_run_host_checked",
    "pk_run_host_io",
    "pk_launch_multi",
    "pk_jacobi_sweep",
    "pk_launch_block",
    "pk_jacobi_sweep_peer",
    "pk_ipc_export",
    "pk_ipc_open",
    "pk_ipc_close",
    "pk_jacobi_narrow",
    "pk_footprint_words",
    "pk_launch_count",
    "pk_last_error",
    "pk_version",
    "pk_jit_compile",
    "pk_jit_launch",
    "pk_jit_release",
)


class PkLaunch(ctypes.Structure):
    _fields_ = [
        ("family", ctypes.c_int32),
        ("variant", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("flags", ctypes.c_int32),
        ("N", ctypes.c_int64),
        ("T", ctypes.c_int64),
        ("s", ctypes.c_int64),
        ("B", ctypes.c_int64),
        ("B0", ctypes.c_int64),
        ("B1", ctypes.c_int64),
        ("ub1", ctypes.c_int64),
        ("lo", ctypes.c_int64),
        ("hi", ctypes.c_int64),
        ("tblock", ctypes.c_int64),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class PkPeer(ctypes.Structure):
    """pk_peer_t: the neighbours of a rank for pk_jacobi_sweep_peer."""

    _fields_ = [
        ("left_base", ctypes.c_void_p),
        ("right_base", ctypes.c_void_p),
        ("wait_left", ctypes.c_void_p),
        ("wait_right", ctypes.c_void_p),
        ("signal_left", ctypes.c_void_p),
        ("signal_right", ctypes.c_void_p),
        ("error", ctypes.c_void_p),
    ]


class PkMachine(ctypes.Structure):
    _fields_ = [
        ("device", ctypes.c_int32),
        ("cc_major", ctypes.c_int32),
        ("cc_minor", ctypes.c_int32),
        ("sm_count", ctypes.c_int32),
        ("warp_size", ctypes.c_int32),
        ("max_threads_per_block", ctypes.c_int32),
        ("max_threads_per_sm", ctypes.c_int32),
        ("regs_per_thread", ctypes.c_int32),
        ("regs_per_block", ctypes.c_int32),
        ("regs_per_sm", ctypes.c_int32),
        ("smem_per_block", ctypes.c_int64),
        ("smem_per_block_optin", ctypes.c_int64),
        ("smem_per_sm", ctypes.c_int64),
        ("l2_bytes", ctypes.c_int64),
        ("global_mem_bytes", ctypes.c_int64),
        ("clock_khz", ctypes.c_int32),
        ("mem_clock_khz", ctypes.c_int32),
        ("mem_bus_width_bits", ctypes.c_int32),
        ("name", ctypes.c_char * 256),
    ]


class PkError(RuntimeError):
    """A libpk failure without a closer Python equivalent."""


_lock = threading.Lock()
_lib = None


def load() -> ctypes.CDLL:
    """Load libpk.so once; raise loudly if it is missing (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                "libpk.so not found at %s: build it with `python -m "
                "paper_1801_04348_b200.build` (there is no CPU fallback)" % LIB_PATH
            )
        lib = ctypes.CDLL(LIB_PATH)
        vp = ctypes.c_void_p
        lib.pk_query_machine.argtypes = [ctypes.c_int, ctypes.POINTER(PkMachine)]
        lib.pk_query_machine.restype = ctypes.c_int
        lib.pk_launch.argtypes = [ctypes.POINTER(PkLaunch), ctypes.POINTER(vp), ctypes.c_int, vp]
        lib.pk_launch.restype = ctypes.c_int
        lib.pk_run_host.argtypes = [ctypes.POINTER(PkLaunch), ctypes.POINTER(vp), ctypes.c_int, ctypes.c_int]
        lib.pk_run_host.restype = ctypes.c_int
        i64p = ctypes.POINTER(ctypes.c_int64)
        lib.pk_launch_checked.argtypes = [ctypes.POINTER(PkLaunch), ctypes.POINTER(vp), i64p, ctypes.c_int, vp]
        lib.pk_launch_checked.restype = ctypes.c_int
        lib.pk_required_elems.argtypes = [ctypes.POINTER(PkLaunch), i64p, ctypes.c_int]
        lib.pk_required_elems.restype = ctypes.c_int
        lib.pk_run_host_checked.argtypes = [ctypes.POINTER(PkLaunch), ctypes.POINTER(vp), i64p, ctypes.c_int,
                                            ctypes.c_int]
        lib.pk_run_host_checked.restype = ctypes.c_int
        lib.pk_run_host_io.argtypes = [ctypes.POINTER(PkLaunch), ctypes.POINTER(vp), ctypes.POINTER(vp), i64p,
                                       ctypes.c_int, ctypes.c_int]
        lib.pk_run_host_io.restype = ctypes.c_int
        lib.pk_launch_multi.argtypes = [ctypes.POINTER(PkLaunch), ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                        ctypes.POINTER(vp), ctypes.c_int, ctypes.c_int64, ctypes.c_int]
        lib.pk_launch_multi.restype = ctypes.c_int
        lib.pk_launch_block.argtypes = [ctypes.POINTER(PkLaunch), ctypes.POINTER(ctypes.c_int64), ctypes.c_int,
                                         ctypes.POINTER(ctypes.c_int64), ctypes.c_int, ctypes.POINTER(vp),
                                         ctypes.c_int, vp]
        lib.pk_launch_block.restype = ctypes.c_int
        lib.pk_jacobi_sweep.argtypes = [ctypes.POINTER(PkLaunch), vp, vp, ctypes.c_int64, ctypes.c_int64, vp]
        lib.pk_jacobi_sweep.restype = ctypes.c_int
        lib.pk_jacobi_sweep_peer.argtypes = [ctypes.POINTER(PkLaunch), vp, ctypes.c_int64, ctypes.c_int64,
                                             ctypes.c_int64, ctypes.POINTER(PkPeer), vp]
        lib.pk_jacobi_sweep_peer.restype = ctypes.c_int
        lib.pk_ipc_export.argtypes = [vp, vp, ctypes.POINTER(ctypes.c_int64)]
        lib.pk_ipc_export.restype = ctypes.c_int
        lib.pk_ipc_open.argtypes = [vp, ctypes.c_int64, ctypes.POINTER(vp)]
        lib.pk_ipc_open.restype = ctypes.c_int
        lib.pk_ipc_close.argtypes = [vp, ctypes.c_int64]
        lib.pk_ipc_close.restype = ctypes.c_int
        lib.pk_jacobi_narrow.argtypes = [ctypes.POINTER(PkLaunch), vp, ctypes.POINTER(ctypes.c_int32), vp]
        lib.pk_jacobi_narrow.restype = ctypes.c_int
        lib.pk_footprint_words.argtypes = [ctypes.POINTER(PkLaunch)]
        lib.pk_footprint_words.restype = ctypes.c_int64
        lib.pk_launch_count.argtypes = []
        lib.pk_launch_count.restype = ctypes.c_int64
        lib.pk_last_error.argtypes = []
        lib.pk_last_error.restype = ctypes.c_char_p
        lib.pk_jit_compile.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_char_p),
                                       ctypes.c_int, ctypes.POINTER(vp)]
        lib.pk_jit_compile.restype = ctypes.c_int
        lib.pk_jit_launch.argtypes = [vp, ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint32),
                                      ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint64),
                                      ctypes.POINTER(ctypes.c_int32), ctypes.c_int, vp]
        lib.pk_jit_launch.restype = ctypes.c_int
        lib.pk_jit_release.argtypes = [vp]
        lib.pk_jit_release.restype = ctypes.c_int
        lib.pk_version.argtypes = []
        lib.pk_version.restype = ctypes.c_int
        _lib = lib
        return lib


def last_error() -> str:
    msg = load().pk_last_error()
    return msg.decode("utf-8", "replace") if msg else ""


def check(rc: int) -> None:
    """Map a pk.h status code onto the reference interpreter's exceptions."""
    if rc == PK_OK:
        return
    msg = last_error()
    if rc == PK_E_PARAM:
        raise ValueError(msg)
    if rc == PK_E_BOUNDS:
        raise IndexError(msg)
    if rc == PK_E_DIV0:
        raise ZeroDivisionError(msg)
    if rc == PK_E_UNSUPPORTED:
        raise NotImplementedError(msg)
    if rc == PK_E_ALLOC:
        raise MemoryError(msg)
    raise PkError("libpk error %d: %s" % (rc, msg))


def ptr_array(ptrs) -> "ctypes.Array":
    arr = (ctypes.c_void_p * len(ptrs))()
    for i, p in enumerate(ptrs):
        arr[i] = ctypes.c_void_p(int(p))
    return arr


def launch(L: PkLaunch, ptrs, stream: int = 0) -> None:
    lib = load()
    arr = ptr_array(ptrs)
    check(lib.pk_launch(ctypes.byref(L), arr, len(ptrs), ctypes.c_void_p(stream or None)))


def run_host(L: PkLaunch, host_ptrs, device: int = 0, elems=None) -> None:
    """pk_run_host (pk_run_host_checked when element counts are given)."""
    lib = load()
    arr = ptr_array(host_ptrs)
    if elems is None:
        check(lib.pk_run_host(ctypes.byref(L), arr, len(host_ptrs), device))
    else:
        n = (ctypes.c_int64 * len(elems))(*[int(e) for e in elems])
        check(lib.pk_run_host_checked(ctypes.byref(L), arr, n, len(host_ptrs), device))


def run_host_io(L: PkLaunch, in_ptrs, out_ptrs, elems, device: int = 0) -> None:
    """pk_run_host_io: inputs and outputs in separate host buffers (None / 0 = absent)."""
    n = (ctypes.c_int64 * len(elems))(*[int(e) for e in elems])
    check(load().pk_run_host_io(ctypes.byref(L), ptr_array([p or 0 for p in in_ptrs]),
                                ptr_array([p or 0 for p in out_ptrs]), n, len(in_ptrs), device))


def launch_checked(L: PkLaunch, ptrs, elems, stream: int = 0) -> None:
    lib = load()
    n = (ctypes.c_int64 * len(elems))(*[int(e) for e in elems])
    check(lib.pk_launch_checked(ctypes.byref(L), ptr_array(ptrs), n, len(ptrs), ctypes.c_void_p(stream or None)))


def required_elems(L: PkLaunch, nptrs: int) -> list[int]:
    """1 + the largest flat index the launch touches in each array (pk_required_elems)."""
    need = (ctypes.c_int64 * 3)()
    check(load().pk_required_elems(ctypes.byref(L), need, 3))
    return [int(need[i]) for i in range(nptrs)]


def launch_multi(L: PkLaunch, devices, ptr_lists, halo: int = 0, gather: bool = True) -> None:
    """pk_launch_multi: ptr_lists[k] are the arrays (declaration order) on devices[k]."""
    lib = load()
    n = len(devices)
    devs = (ctypes.c_int * n)(*devices)
    flat = ptr_array([p for ptrs in ptr_lists for p in ptrs])
    nptrs = len(ptr_lists[0]) if ptr_lists else 0
    check(lib.pk_launch_multi(ctypes.byref(L), n, devs, flat, nptrs, int(halo), 1 if gather else 0))


def launch_block(L: PkLaunch, grid, ctx, ptrs, stream: int = 0) -> None:
    """pk_launch_block: one thread block at grid indices ``grid`` and context values ``ctx``."""
    g = (ctypes.c_int64 * max(1, len(grid)))(*[int(v) for v in grid])
    c = (ctypes.c_int64 * max(1, len(ctx)))(*[int(v) for v in ctx])
    check(load().pk_launch_block(ctypes.byref(L), g, len(grid), c, len(ctx), ptr_array(ptrs), len(ptrs),
                                 ctypes.c_void_p(stream or None)))


def jacobi_sweep(L: PkLaunch, src: int, dst: int, lo: int, hi: int, stream: int = 0) -> None:
    lib = load()
    check(lib.pk_jacobi_sweep(ctypes.byref(L), ctypes.c_void_p(src), ctypes.c_void_p(dst), lo, hi,
                              ctypes.c_void_p(stream or None)))


def jacobi_sweep_peer(L: PkLaunch, a: int, step: int, lo: int, hi: int, peer: PkPeer, stream: int = 0) -> None:
    lib = load()
    check(lib.pk_jacobi_sweep_peer(ctypes.byref(L), ctypes.c_void_p(a), step, lo, hi, ctypes.byref(peer),
                                   ctypes.c_void_p(stream or None)))


def ipc_export(ptr: int) -> tuple[bytes, int]:
    """(64-byte handle, offset from the allocation base) of a device pointer."""
    lib = load()
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_int64(0)
    check(lib.pk_ipc_export(ctypes.c_void_p(ptr), h, ctypes.byref(off)))
    return h.raw, off.value


def ipc_open(handle: bytes, offset: int) -> int:
    lib = load()
    out = ctypes.c_void_p(0)
    check(lib.pk_ipc_open(ctypes.create_string_buffer(handle, 64), offset, ctypes.byref(out)))
    return int(out.value)


def ipc_close(ptr: int, offset: int) -> None:
    check(load().pk_ipc_close(ctypes.c_void_p(ptr), offset))


def jacobi_narrow(L: PkLaunch, a: int, stream: int = 0) -> bool:
    out = ctypes.c_int32(0)
    check(load().pk_jacobi_narrow(ctypes.byref(L), ctypes.c_void_p(a), ctypes.byref(out),
                                  ctypes.c_void_p(stream or None)))
    return bool(out.value)


def footprint_words(L: PkLaunch) -> int:
    return int(load().pk_footprint_words(ctypes.byref(L)))


def launch_count() -> int:
    return int(load().pk_launch_count())


def query_machine(device: int = 0) -> dict:
    m = PkMachine()
    check(load().pk_query_machine(device, ctypes.byref(m)))
    out = {name: getattr(m, name) for name, _ in PkMachine._fields_}
    out["name"] = m.name.decode("utf-8", "replace")
    return out


def jit_compile(source: str, name: str, options=()) -> int:
    """Compile CUDA text for sm_100a (NVRTC); returns an opaque kernel handle."""
    h = ctypes.c_void_p()
    opts = (ctypes.c_char_p * max(1, len(options)))(*[o.encode() for o in options])
    check(load().pk_jit_compile(source.encode(), name.encode(), opts, len(options), ctypes.byref(h)))
    return int(h.value)


def jit_launch(handle: int, grid, block, args, kinds, smem: int = 0, stream: int = 0) -> None:
    g = (ctypes.c_uint32 * 3)(*(list(grid) + [1] * (3 - len(grid))))
    b = (ctypes.c_uint32 * 3)(*(list(block) + [1] * (3 - len(block))))
    n = len(args)
    av = (ctypes.c_uint64 * max(1, n))(*[int(x) & 0xFFFFFFFFFFFFFFFF for x in args])
    kv = (ctypes.c_int32 * max(1, n))(*kinds)
    check(load().pk_jit_launch(ctypes.c_void_p(handle), g, b, smem, av, kv, n, ctypes.c_void_p(stream or None)))


def jit_release(handle: int) -> None:
    load().pk_jit_release(ctypes.c_void_p(handle))


def version() -> tuple[int, int]:
    v = int(load().pk_version())
    return v >> 16, v & 0xFFFF
