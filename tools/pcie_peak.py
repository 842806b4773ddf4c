"""Host<->device copy bandwidth on this box through libweldgpu (pinned host
buffers, the executor's copy streams): H2D alone, D2H alone, and both at
once on the two copy streams -- the ceiling of every e2e number."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1709_06416_b200  # noqa: F401
from paper_1709_06416_b200 import runtime as rt
from paper_1709_06416_b200.columns import pinned_empty

NB = 1 << 30
h_in = pinned_empty(NB // 8, "<f8")
h_out = pinned_empty(NB // 8, "<f8")
h_in[:] = 1.0
d_in = rt.alloc(NB)
d_out = rt.alloc(NB)


def timed(fn, reps=5):
    best = 1e30
    for _ in range(reps):
        rt.sync_all()
        t = time.perf_counter()
        fn()
        rt.sync_all()
        best = min(best, time.perf_counter() - t)
    return best


def h2d():
    rt.stream_select(1)
    rt.h2d(d_in.ptr, h_in.ctypes.data, NB)
    rt.stream_select(0)


def d2h():
    rt.stream_select(2)
    rt.d2h_async(h_out.ctypes.data, d_out.ptr, NB)
    rt.stream_select(0)


def both():
    rt.stream_select(1)
    rt.h2d(d_in.ptr, h_in.ctypes.data, NB)
    rt.stream_select(2)
    rt.d2h_async(h_out.ctypes.data, d_out.ptr, NB)
    rt.stream_select(0)


for name, fn, nbytes in (("H2D", h2d, NB), ("D2H", d2h, NB), ("H2D+D2H concurrent", both, 2 * NB)):
    t = timed(fn)
    print(f"{name}: {nbytes / t / 1e9:.1f} GB/s ({nbytes / 1e9:.2f} GB in {t * 1e3:.1f} ms)")
