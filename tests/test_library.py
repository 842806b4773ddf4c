"""The C-ABI library builds for sm_100a, loads without a GPU, and exports
every entry point include/weldgpu.h declares (no device calls here)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "weldgpu.h")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(wg_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_1709_06416_b200 import runtime
    if not os.path.exists(runtime.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    return runtime.load_library()


def test_header_declares_entry_points():
    names = declared()
    assert "wg_compile" in names and "wg_launch" in names and len(names) > 30


def test_every_declared_symbol_is_exported(lib):
    for name in declared():
        assert hasattr(lib, name), name


def test_ctypes_signatures_cover_header():
    from paper_1709_06416_b200 import runtime
    assert set(declared()) == set(runtime.EXPORTED)


def test_library_targets_sm100a(lib):
    from paper_1709_06416_b200 import runtime
    out = subprocess.run(["cuobjdump", "--list-elf", runtime.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_no_device_is_a_loud_error(lib):
    """No CPU fallback: without a GPU the runtime refuses, it does not emulate."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1709_06416_b200 import runtime
    with pytest.raises(runtime.WeldGpuError):
        runtime.lib()


def test_library_exports_no_torch_types():
    text = open(HEADER).read()
    assert "torch" not in text.lower().replace("no torch types", "")
