"""CPU checks of the drop-in boundary: the C-ABI library loads and exports
every entry point include/qgtc_b200.h declares (no compute without a GPU)."""

import os
import re
import subprocess

from paper_2111_09547_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "qgtc_b200.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*int\s+(qg_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_the_python_export_list():
    assert _declared() == sorted(N.EXPORTS)


def test_library_loads_and_exports_every_declared_symbol():
    lib = N.lib()
    for name in _declared():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", N.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (qg_\w+)", out))
    assert set(_declared()) <= exported
    assert lib.qg_version() == len(_declared())


def test_library_is_built_for_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_side_argument_errors_need_no_gpu():
    # argument validation happens before any launch and maps to the reference's exceptions
    import pytest
    with pytest.raises(ValueError):
        N.check(N.QG_ERR_ARG, "x")
    with pytest.raises(N.ShapeError):
        N.check(N.QG_ERR_SHAPE, "x")
    assert N.lib().qg_quantize_pack(None, 0, 4, 4, 4, 0.0, 1.0, 9, 0, 8, None, None, None, None, None, None) \
        in (N.QG_ERR_ARG, N.QG_ERR_BITS)
