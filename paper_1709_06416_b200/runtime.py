"""ctypes binding to libweldgpu.so (include/weldgpu.h).

The library is built in-tree by ``__graft_entry__.build()``.  There is no
fallback: if the library or a GPU is missing, device operations raise.
"""
from __future__ import annotations

import ctypes
import hashlib
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libweldgpu.so")
HEADER_PATH = os.path.join(_HERE, "csrc", "weld_device.cuh")

NVRTC_OPTS = ("-arch=sm_100a", "-std=c++17", "-fmad=false", "-default-device", "-lineinfo")

u64 = ctypes.c_uint64
i64 = ctypes.c_int64
c_int = ctypes.c_int
c_char_p = ctypes.c_char_p
c_void_p = ctypes.c_void_p

_SIGS = {
    "wg_last_error": (c_char_p, []),
    "wg_version": (c_int, []),
    "wg_device_count": (c_int, [ctypes.POINTER(c_int)]),
    "wg_init": (c_int, [c_int]),
    "wg_sm_count": (c_int, [ctypes.POINTER(c_int)]),
    "wg_stream": (c_int, [ctypes.POINTER(u64)]),
    "wg_sync": (c_int, []),
    "wg_alloc": (c_int, [u64, ctypes.POINTER(u64)]),
    "wg_free": (c_int, [u64]),
    "wg_mem_trim": (c_int, []),
    "wg_mem_stats": (c_int, [ctypes.POINTER(u64), ctypes.POINTER(u64)]),
    "wg_mem_reset_peak": (c_int, []),
    "wg_memset": (c_int, [u64, c_int, u64]),
    "wg_h2d": (c_int, [u64, c_void_p, u64]),
    "wg_d2h": (c_int, [c_void_p, u64, u64]),
    "wg_d2h_async": (c_int, [c_void_p, u64, u64]),
    "wg_d2d": (c_int, [u64, u64, u64]),
    "wg_host_alloc": (c_int, [u64, ctypes.POINTER(c_void_p)]),
    "wg_host_free": (c_int, [c_void_p]),
    "wg_host_register": (c_int, [c_void_p, u64]),
    "wg_host_unregister": (c_int, [c_void_p]),
    "wg_error_ptr": (c_int, [ctypes.POINTER(u64)]),
    "wg_read_error": (c_int, [ctypes.POINTER(i64), ctypes.POINTER(i64)]),
    "wg_last_sync_error": (c_int, [ctypes.POINTER(i64), ctypes.POINTER(i64)]),
    "wg_d2h_checked": (c_int, [c_void_p, u64, u64, ctypes.POINTER(i64), ctypes.POINTER(i64)]),
    "wg_compile": (c_int, [c_char_p, c_char_p, c_int, ctypes.POINTER(c_char_p), ctypes.POINTER(c_char_p), c_int,
                           ctypes.POINTER(c_char_p), ctypes.POINTER(u64), c_char_p, u64]),
    "wg_compile_check": (c_int, [c_char_p, c_char_p, c_int, ctypes.POINTER(c_char_p), ctypes.POINTER(c_char_p),
                                 c_int, ctypes.POINTER(c_char_p), ctypes.POINTER(u64), c_char_p, u64]),
    "wg_compile_ptx": (c_int, [c_char_p, c_char_p, c_int, ctypes.POINTER(c_char_p), ctypes.POINTER(c_char_p), c_int,
                               ctypes.POINTER(c_char_p), c_char_p, u64, ctypes.POINTER(u64), c_char_p, u64]),
    "wg_module_load": (c_int, [c_char_p, ctypes.POINTER(u64)]),
    "wg_module_function": (c_int, [u64, c_char_p, ctypes.POINTER(u64)]),
    "wg_occupancy": (c_int, [u64, c_int, c_int, ctypes.POINTER(c_int)]),
    "wg_launch": (c_int, [u64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, c_void_p, u64]),
    "wg_table_init": (c_int, [u64, u64, c_int, ctypes.POINTER(u64)]),
    "wg_table_compact": (c_int, [u64, u64, c_int, c_int, ctypes.POINTER(u64), c_int, ctypes.POINTER(u64)]),
    "wg_dict_finish_small": (c_int, [u64, u64, c_int, c_int, c_int, c_int, ctypes.POINTER(c_int), c_int,
                                     ctypes.POINTER(c_int), ctypes.POINTER(u64), u64, ctypes.POINTER(u64)]),
    "wg_order_key": (c_int, [u64, c_int, u64, u64, u64]),
    "wg_iota_u32": (c_int, [u64, u64]),
    "wg_iota_i64": (c_int, [u64, u64, i64]),
    "wg_seg_stats": (c_int, [u64, u64, u64, u64]),
    "wg_neg_zero": (c_int, [u64, u64, c_int]),
    "wg_exclusive_scan_i64": (c_int, [u64, u64, u64, u64]),
    "wg_sort_pairs": (c_int, [u64, u64, u64, u64, u64, c_int, c_int]),
    "wg_gather": (c_int, [u64, u64, u64, u64, c_int]),
    "wg_narrow": (c_int, [u64, u64, c_int, u64]),
    "wg_widen": (c_int, [u64, u64, c_int, u64]),
    "wg_run_starts": (c_int, [ctypes.POINTER(u64), c_int, u64, u64, ctypes.POINTER(u64)]),
    "wg_group_finish1": (c_int, [u64, c_int, u64, c_int, u64, u64, u64, u64, ctypes.POINTER(u64)]),
    "wg_gen_column": (c_int, [u64, u64, u64, c_int, c_int, u64, u64, i64, u64, ctypes.c_double, ctypes.c_double,
                              ctypes.c_double, c_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i64)]),
    "wg_mul_inplace_f64": (c_int, [u64, u64, u64]),
    "wg_flush_l2": (c_int, [u64, u64, ctypes.c_uint32]),
    "wg_event_create": (c_int, [ctypes.POINTER(u64)]),
    "wg_event_record": (c_int, [u64]),
    "wg_event_elapsed_ms": (c_int, [u64, u64, ctypes.POINTER(ctypes.c_float)]),
    "wg_event_destroy": (c_int, [u64]),
    "wg_prof_enable": (c_int, [c_int]),
    "wg_prof_count": (c_int, [ctypes.POINTER(c_int)]),
    "wg_prof_record": (c_int, [c_int, c_char_p, c_int, ctypes.POINTER(ctypes.c_float)]),
    "wg_stream_select": (c_int, [c_int]),
    "wg_stream_wait_event": (c_int, [u64]),
    "wg_sync_all": (c_int, []),
    "wg_partition": (c_int, [u64, c_int, ctypes.POINTER(u64), c_int, c_int, ctypes.POINTER(u64), ctypes.POINTER(u64),
                             ctypes.POINTER(c_int), u64, ctypes.POINTER(u64)]),
    "wg_nccl_unique_id": (c_int, [c_char_p, c_int]),
    "wg_nccl_init": (c_int, [c_int, c_int, c_char_p]),
    "wg_nccl_finalize": (c_int, []),
    "wg_nccl_allgather": (c_int, [u64, u64, u64]),
    "wg_nccl_allreduce": (c_int, [u64, u64, u64, c_int, c_int]),
    "wg_nccl_sendrecv": (c_int, [c_int, ctypes.POINTER(u64), ctypes.POINTER(u64), ctypes.POINTER(c_int), c_int,
                                 ctypes.POINTER(u64), ctypes.POINTER(u64), ctypes.POINTER(c_int)]),
}

EXPORTED = tuple(_SIGS)


class WeldGpuError(RuntimeError):
    pass


_lib = None
_lock = threading.RLock()
_inited = False


def load_library():
    """Load libweldgpu.so (no device initialisation)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise WeldGpuError(
                    f"{LIB_PATH} is missing: run __graft_entry__.build() (there is no CPU fallback)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
        return _lib


def _check(rc):
    if rc != 0:
        raise WeldGpuError(load_library().wg_last_error().decode(errors="replace"))


TRACE = os.environ.get("WELDGPU_TRACE", "") == "1"
TRACE_TIMES = {}


def _traced(name, fn):
    import time
    _check(lib().wg_sync())
    t0 = time.perf_counter()
    r = fn()
    _check(lib().wg_sync())
    TRACE_TIMES[name] = TRACE_TIMES.get(name, 0.0) + time.perf_counter() - t0
    return r


def call(name, *args):
    if TRACE:
        _traced(name, lambda: _check(getattr(lib(), name)(*args)))
    else:
        _check(getattr(lib(), name)(*args))
    LAUNCHES[0] += _KERNEL_CALLS.get(name, 0)


def lib():
    """Library handle with the device initialised."""
    global _inited
    if _inited:
        return _lib
    L = load_library()
    if not _inited:
        with _lock:
            if not _inited:
                dev = int(os.environ.get("LOCAL_RANK", os.environ.get("WELDGPU_DEVICE", "0")))
                n = c_int(0)
                rc = L.wg_device_count(ctypes.byref(n))
                if rc != 0 or n.value == 0:
                    raise WeldGpuError("no CUDA device visible: the weldgpu executor has no CPU fallback")
                _check(L.wg_init(dev % n.value))
                _inited = True
    return L


_SM_COUNT = [0]


def sm_count():
    if not _SM_COUNT[0]:
        n = c_int(0)
        _check(lib().wg_sm_count(ctypes.byref(n)))
        _SM_COUNT[0] = n.value
    return _SM_COUNT[0]


def stream_handle():
    s = u64(0)
    _check(lib().wg_stream(ctypes.byref(s)))
    return s.value


def sync():
    _check(lib().wg_sync())


# ---------------------------------------------------------------------------
# Device buffers


class DeviceBuffer:
    """One stream-ordered device allocation; freed when garbage collected."""

    __slots__ = ("ptr", "nbytes", "__weakref__")

    def __init__(self, nbytes: int):
        p = u64(0)
        if TRACE:
            _traced("alloc", lambda: _check(lib().wg_alloc(max(int(nbytes), 1), ctypes.byref(p))))
        else:
            _check(lib().wg_alloc(max(int(nbytes), 1), ctypes.byref(p)))
        self.ptr = p.value
        self.nbytes = int(nbytes)

    def free(self):
        if self.ptr:
            L = _lib
            if L is not None:
                L.wg_free(self.ptr)
            self.ptr = 0

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def __repr__(self):
        return f"<DeviceBuffer 0x{self.ptr:x} {self.nbytes}B>"


def alloc(nbytes):
    return DeviceBuffer(nbytes)


def host_register(arr):
    """Pin a numpy array's pages (cudaHostRegister) for async copies."""
    _check(lib().wg_host_register(arr.ctypes.data, arr.nbytes))


def host_unregister(arr):
    _check(lib().wg_host_unregister(arr.ctypes.data))


def memset(buf_ptr, value, nbytes):
    _check(lib().wg_memset(buf_ptr, value, nbytes))


def h2d(dst_ptr, host_ptr, nbytes):
    if TRACE:
        _traced("h2d", lambda: _check(lib().wg_h2d(dst_ptr, host_ptr, nbytes)))
    else:
        _check(lib().wg_h2d(dst_ptr, host_ptr, nbytes))


def d2h(host_ptr, src_ptr, nbytes):
    if TRACE:
        _traced("d2h", lambda: _check(lib().wg_d2h(host_ptr, src_ptr, nbytes)))
    else:
        _check(lib().wg_d2h(host_ptr, src_ptr, nbytes))


def d2h_async(host_ptr, src_ptr, nbytes):
    _check(lib().wg_d2h_async(host_ptr, src_ptr, nbytes))


def d2d(dst_ptr, src_ptr, nbytes):
    _check(lib().wg_d2d(dst_ptr, src_ptr, nbytes))


def d2h_checked(host_ptr, src_ptr, nbytes):
    """Copy device -> host and read the error word; one synchronisation.
    Returns (code, info)."""
    c, i = i64(0), i64(0)
    _check(lib().wg_d2h_checked(host_ptr, src_ptr, nbytes, ctypes.byref(c), ctypes.byref(i)))
    return c.value, i.value


def host_alloc(nbytes):
    """Pinned host memory (cudaMallocHost; device-accessible at the same
    address under unified addressing)."""
    p = c_void_p(0)
    _check(lib().wg_host_alloc(nbytes, ctypes.byref(p)))
    return p.value


def clear_error():
    """Reset the device error word (after a raise read from a host mirror)."""
    read_error()


def read_error():
    c, i = i64(0), i64(0)
    _check(lib().wg_read_error(ctypes.byref(c), ctypes.byref(i)))
    return c.value, i.value


def last_sync_error():
    """Error word captured by the last wg_dict_finish_small (no device sync)."""
    c, i = i64(0), i64(0)
    _check(lib().wg_last_sync_error(ctypes.byref(c), ctypes.byref(i)))
    return c.value, i.value


_ERR_PTR = [0]


def error_ptr():
    """Device address of the error word (allocated once at library init)."""
    if not _ERR_PTR[0]:
        p = u64(0)
        _check(lib().wg_error_ptr(ctypes.byref(p)))
        _ERR_PTR[0] = p.value
    return _ERR_PTR[0]


def mem_stats():
    a, b = u64(0), u64(0)
    _check(lib().wg_mem_stats(ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


# ---------------------------------------------------------------------------
# NVRTC kernels


_header_text = None
_modules = {}


def header_text():
    global _header_text
    if _header_text is None:
        with open(HEADER_PATH) as f:
            _header_text = f.read()
    return _header_text


_TABLES = ("wg_erf_table.h", "wg_log_table.h", "wg_exp_table.h")     # generated by tools/gen_*_table.py
_table_texts = None


def _nvrtc_args(src):
    global _table_texts
    if _table_texts is None:
        _table_texts = []
        for t in _TABLES:
            with open(os.path.join(_HERE, "csrc", t)) as f:
                _table_texts.append(f.read().encode())
    hs = (c_char_p * (1 + len(_TABLES)))(header_text().encode(), *_table_texts)
    hn = (c_char_p * (1 + len(_TABLES)))(b"weld_device.cuh", *(t.encode() for t in _TABLES))
    opts = [o.encode() for o in NVRTC_OPTS]
    oa = (c_char_p * len(opts))(*opts)
    return hs, hn, oa, len(opts)


def compile_check(src: str, name="weld_loop.cu"):
    """Compile for sm_100a without loading (works with no GPU).  Returns the
    cubin size; raises WeldGpuError with the NVRTC log on failure."""
    L = load_library()
    hs, hn, oa, no = _nvrtc_args(src)
    sz = u64(0)
    log = ctypes.create_string_buffer(1 << 16)
    rc = L.wg_compile_check(src.encode(), name.encode(), 1 + len(_TABLES), hs, hn, no, oa, ctypes.byref(sz), log, 1 << 16)
    if rc != 0:
        raise WeldGpuError(L.wg_last_error().decode(errors="replace"))
    return sz.value


# Instrumentation: number of this library's kernels launched, and an
# optional hook called around each generated-kernel launch (bench timing).
LAUNCHES = [0]
LAUNCH_HOOK = [None]
_KERNEL_CALLS = {"wg_dict_finish_small": 1, "wg_table_init": 1, "wg_table_compact": 1, "wg_order_key": 1, "wg_iota_u32": 1, "wg_iota_i64": 1, "wg_seg_stats": 1, "wg_neg_zero": 1, "wg_exclusive_scan_i64": 1,
                 "wg_sort_pairs": 1, "wg_gather": 1, "wg_narrow": 1, "wg_widen": 1, "wg_run_starts": 2, "wg_group_finish1": 12,
                 "wg_gen_column": 1, "wg_mul_inplace_f64": 1, "wg_flush_l2": 1}


class Kernel:
    __slots__ = ("fn", "name", "occ")

    def __init__(self, fn, name):
        self.fn = fn
        self.name = name
        self.occ = {}

    def blocks_per_sm(self, block, smem=0):
        key = (block, smem)
        v = self.occ.get(key)
        if v is None:
            n = c_int(0)
            _check(lib().wg_occupancy(self.fn, block, smem, ctypes.byref(n)))
            v = self.occ[key] = max(1, n.value)
        return v

    def launch(self, grid, block, params: bytes, smem=0):
        buf = params          # bytes: passed as a pointer, copied by cuLaunchKernel
        hook = LAUNCH_HOOK[0]
        if hook is not None:
            hook("before", self)
        if TRACE:
            _traced("kernel:" + self.name, lambda: _check(lib().wg_launch(self.fn, grid, block, smem, buf, len(params))))
        else:
            _check(lib().wg_launch(self.fn, grid, block, smem, buf, len(params)))
        LAUNCHES[0] += 1
        if hook is not None:
            hook("after", self)


def compile_ptx(src: str, name="weld_loop.cu") -> str:
    L = load_library()
    hs, hn, oa, no = _nvrtc_args(src)
    size = u64(0)
    log = ctypes.create_string_buffer(1 << 16)
    if L.wg_compile_ptx(src.encode(), name.encode(), 1 + len(_TABLES), hs, hn, no, oa, None, 0, ctypes.byref(size), log, 1 << 16):
        raise WeldGpuError(L.wg_last_error().decode(errors="replace"))
    buf = ctypes.create_string_buffer(size.value)
    _check(L.wg_compile_ptx(src.encode(), name.encode(), 1 + len(_TABLES), hs, hn, no, oa, buf, size.value, ctypes.byref(size),
                            log, 1 << 16))
    return buf.value.decode()


def get_kernel(src: str, name: str) -> Kernel:
    """Compile (cached by source hash) and return the named kernel."""
    key = hashlib.sha1(src.encode()).hexdigest()
    with _lock:
        mod = _modules.get(key)
        if mod is None:
            L = lib()
            hs, hn, oa, no = _nvrtc_args(src)
            m = u64(0)
            log = ctypes.create_string_buffer(1 << 16)
            rc = L.wg_compile(src.encode(), f"wg_{key[:12]}.cu".encode(), 1 + len(_TABLES), hs, hn, no, oa, ctypes.byref(m),
                              log, 1 << 16)
            if rc != 0:
                raise WeldGpuError(L.wg_last_error().decode(errors="replace"))
            mod = _modules[key] = (m.value, {})
        handle, fns = mod
        k = fns.get(name)
        if k is None:
            f = u64(0)
            _check(lib().wg_module_function(handle, name.encode(), ctypes.byref(f)))
            k = fns[name] = Kernel(f.value, name)
        return k


# ---------------------------------------------------------------------------
# Events (bench timing on the library's own stream)


def stream_select(which):
    _check(lib().wg_stream_select(which))


def stream_wait(ev):
    _check(lib().wg_stream_wait_event(ev.h))


def sync_all():
    _check(lib().wg_sync_all())


class Event:
    def __init__(self):
        e = u64(0)
        _check(lib().wg_event_create(ctypes.byref(e)))
        self.h = e.value

    def record(self):
        _check(lib().wg_event_record(self.h))

    def elapsed_ms(self, later: "Event") -> float:
        ms = ctypes.c_float(0)
        _check(lib().wg_event_elapsed_ms(self.h, later.h, ctypes.byref(ms)))
        return ms.value

    def __del__(self):
        try:
            if _lib is not None:
                _lib.wg_event_destroy(self.h)
        except Exception:
            pass


# ---------------------------------------------------------------------------
# Per-launch device timing (wg_prof_*): every kernel the library launches,
# bracketed by events on its own stream.


def prof_enable(on=True):
    _check(lib().wg_prof_enable(1 if on else 0))


def prof_records():
    """[(kernel name, ms)] for every launch since prof_enable(True)."""
    n = c_int(0)
    _check(lib().wg_prof_count(ctypes.byref(n)))
    out = []
    buf = ctypes.create_string_buffer(256)
    ms = ctypes.c_float(0)
    for i in range(n.value):
        _check(lib().wg_prof_record(i, buf, 256, ctypes.byref(ms)))
        out.append((buf.value.decode(), ms.value))
    return out
