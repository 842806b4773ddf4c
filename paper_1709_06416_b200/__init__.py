"""paper_1709_06416_b200 -- a B200-native executor for the Weld IR's
data-parallel core (``for(vector, builders, func)`` + merger / vecbuilder /
dictmerger / groupbuilder / vecmerger).

Drop-in for the reference executor seam ``weldmill.engine.evaluate``
(/root/reference/pkg/src/weldmill/engine/run.py:1008-1074)::

    from paper_1709_06416_b200 import evaluate          # same signature
    value, stats = evaluate(typed_expr, env, EngineConfig(), externs)

    import paper_1709_06416_b200 as wg
    wg.install()   # weldmill.api.evaluate_object / CLI / foreign now run here

Programs still go through the reference front end (parse -> sugar -> type
check -> linearity -> optimize); every loop then runs as an NVRTC-compiled
sm_100a kernel over HBM-resident columns via libweldgpu.so (C ABI in
include/weldgpu.h).  There is no CPU fallback.
"""
from __future__ import annotations

from . import _ref  # noqa: F401  (makes the weldmill front end importable)
from weldmill.engine import EngineConfig, EvalStats, Value  # noqa: F401

from .executor import DeviceUnsupported, evaluate  # noqa: F401
from .columns import DVec, to_device, to_numpy, to_payload, to_boundary_bytes  # noqa: F401

__version__ = "0.1.0"

_installed = {}


def install(zero_copy=True):
    """Rebind the reference API's executor (api.py:23 imports `evaluate` by
    name; api.py:374 calls it) so evaluate_object, the CLI and the foreign
    surface run on the GPU.  zero_copy=True (default) also binds data
    leaves straight to HBM and encodes flat-vector results from the device
    columns (api_bridge: no per-leaf encode/decode round trip, api.py:224-226)."""
    import weldmill.api as api
    uninstall()
    if zero_copy:
        from . import api_bridge
        api_bridge.install()
        _installed["bridge"] = True
    else:
        _installed["api"] = api.evaluate
        api.evaluate = evaluate


def uninstall():
    import weldmill.api as api
    if _installed.pop("bridge", None):
        from . import api_bridge
        api_bridge.uninstall()
    if "api" in _installed:
        api.evaluate = _installed.pop("api")


from .api_bridge import column_encoder  # noqa: E402,F401

__all__ = ["evaluate", "install", "uninstall", "column_encoder", "EngineConfig", "EvalStats", "Value", "DeviceUnsupported", "DVec",
           "to_device", "to_numpy", "to_payload", "to_boundary_bytes"]
