"""Locate the reference front end (weldmill: parser, sugar, type checker,
optimizer, error taxonomy) that this executor sits behind.

The executor replaces only ``weldmill.engine.evaluate``
(/root/reference/pkg/src/weldmill/engine/run.py:1008-1074); programs still
arrive as typed, optimized ``weldmill.expr`` trees.  The front end is the
unmodified reference package installed (git-ignored) under
``baseline/_ref`` by ``pip install --target baseline/_ref``; it travels to the
GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import sys

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_CANDIDATES = (
    os.path.join(_ROOT, "baseline", "_ref"),
)


def ensure_weldmill():
    try:
        import weldmill  # noqa: F401
        return
    except ImportError:
        pass
    for path in _CANDIDATES:
        if os.path.isdir(os.path.join(path, "weldmill")):
            if path not in sys.path:
                sys.path.insert(0, path)
            import weldmill  # noqa: F401
            return
    raise ImportError(
        "the weldmill front end is not importable; install it with "
        "`python -m pip install --no-index --no-build-isolation --target "
        "baseline/_ref <reference>/pkg`"
    )


ensure_weldmill()
