"""End to end through the reference's public API (weldmill.api.evaluate_object)
for C1 (TPC-H Q6, 1M rows): the reference CPU engine, the device executor
behind the plain seam (install(zero_copy=False): every leaf still goes
list -> boundary bytes -> list, api.py:224-226), and the zero-copy bridge
(install(): numpy leaves bound straight to HBM).  Prints ms per call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1709_06416_b200 as wg
from paper_1709_06416_b200 import workloads as W
from weldmill.api import evaluate_object, free_result, new_computed_object, new_data_object
from weldmill.parser import parse_type_text

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
wl = W.WORKLOADS["q6"]
cols = W.host_columns(wl, n)
names = [c.name for c in wl.columns]
tys = {c.name: parse_type_text(f"vec[{c.ty}]") for c in wl.columns}
prog = wl.program


def timed(objs_fn, reps):
    best = 1e30
    out = None
    for _ in range(reps):
        objs = objs_fn()
        t = time.perf_counter()
        r = evaluate_object(new_computed_object(objs, prog))
        out = r.result_bytes()
        free_result(r)
        best = min(best, time.perf_counter() - t)
    return best * 1e3, out


lists = {k: cols[k].tolist() for k in names}
list_objs = lambda: {k: new_data_object(lists[k], tys[k]) for k in names}
np_objs = lambda: {k: new_data_object(cols[k], tys[k], wg.column_encoder) for k in names}
res = {}
if "--cpu" in sys.argv:
    res["reference CPU engine (list leaves)"] = timed(list_objs, 1)
wg.install(zero_copy=False)
res["device, plain seam (list leaves, encode/decode per leaf)"] = timed(list_objs, 3)
wg.uninstall()
wg.install()
res["device, zero-copy bridge (list leaves)"] = timed(list_objs, 3)
res["device, zero-copy bridge (numpy leaves)"] = timed(np_objs, 5)
wg.uninstall()
import struct
ref = None
for k, (ms, b) in res.items():
    v = struct.unpack("<d", b)[0]
    ref = v if ref is None else ref
    print(f"{k}: {ms:.2f} ms per evaluate_object (result {v!r}, rel. diff {abs(v - ref) / max(1.0, abs(ref)):.1e})")
