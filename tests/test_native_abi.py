"""CPU checks of the drop-in boundary: the C-ABI library loads and exports
every entry point include/qgtc_b200.h declares (no compute without a GPU)."""

import os
import re
import subprocess

import pytest

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


def test_counter_closed_forms_match_the_oracle():
    """qg_bmm_counters / qg_gemm_counters (host-only C-ABI) == the oracle's closed forms of
    the reference counters (bitgemm.py:335-370, 409-461) on random flag maps."""
    import ctypes

    import numpy as np

    from oracle import qgtc_oracle as O
    from paper_2111_09547_b200 import _native as N
    lib = N.lib()
    rng = np.random.default_rng(0)
    for _ in range(200):
        rt, ct, s, t, n_chunks = (int(v) for v in rng.integers(1, 9, 5))
        jump, cross = bool(rng.integers(0, 2)), bool(rng.integers(0, 2))
        flags = rng.uniform(0, 1, (rt, ct)) < rng.uniform(0, 1)
        out = (ctypes.c_int64 * 5)()
        assert lib.qg_bmm_counters(rt, ct, int(flags.sum()), s, n_chunks, int(jump), int(cross), ctypes.byref(out)) == 0
        want = O.counters_bmm(flags, s, n_chunks, jump=jump, cross_tile=cross)
        assert list(out) == [want[k] for k in ("tile_mma_count", "tile_fetch_count", "tiles_skipped",
                                               "word_and_popcount_count", "tiles_total")]
        planes = [rng.uniform(0, 1, (rt, ct)) < rng.uniform(0, 1) for _ in range(s)]
        zeros = (ctypes.c_int64 * s)(*[int(f.sum()) for f in planes])
        assert lib.qg_gemm_counters(rt, ct, zeros, s, t, n_chunks, int(jump), int(cross), ctypes.byref(out)) == 0
        want = O.counters_gemm(planes, t, n_chunks, jump=jump, cross_tile=cross)
        assert list(out) == [want[k] for k in ("tile_mma_count", "tile_fetch_count", "tiles_skipped",
                                               "word_and_popcount_count", "tiles_total")]
    # argument errors are host-side status codes, no GPU involved
    assert lib.qg_bmm_counters(2, 2, 5, 1, 1, 1, 1, ctypes.byref(out)) == N.QG_ERR_ARG
    assert lib.qg_batch_h2d(None, 16, None, None) == N.QG_ERR_ARG


def _build_capi_demo(tmp_path):
    import shutil
    import subprocess

    from paper_2111_09547_b200 import _native as N
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib_dir = os.path.dirname(N.LIB_PATH)
    exe = str(tmp_path / "capi_demo")
    cmd = ["gcc", "-O2", "-I", os.path.join(root, "include"), os.path.join(root, "examples", "capi_demo.c"),
           "-L", lib_dir, "-lqgtc_b200", "-L/usr/local/cuda/lib64", "-lcudart", "-lm",
           f"-Wl,-rpath,{lib_dir}", "-Wl,-rpath,/usr/local/cuda/lib64", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_plain_c_consumer_builds_and_runs_host_only(tmp_path):
    """A plain-C host (examples/capi_demo.c) compiles against include/qgtc_b200.h, links the
    library and gets the reference counter closed forms through the C-ABI."""
    import subprocess
    exe = _build_capi_demo(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=60)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "host-only checks OK" in out.stdout


@pytest.mark.gpu
def test_plain_c_consumer_device_bit_qnt(tmp_path):
    import subprocess
    exe = _build_capi_demo(tmp_path)
    out = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "device bit_qnt: OK" in out.stdout


def test_ctypes_struct_layouts_match_the_header(tmp_path):
    """Every ctypes mirror of a header struct has the C compiler's size and field
    offsets (a drifted mirror would pass garbage through the C ABI)."""
    import shutil

    from paper_2111_09547_b200 import tiled
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    mirrors = {"qg_epilogue": N.Epilogue, "qg_gemm_args": N.GemmArgs, "qg_tseg": tiled.TSeg,
               "qg_tiled_args": tiled.TiledArgs, "qg_chain": tiled.Chain, "qg_entry_seg": tiled.EntrySeg,
               "qg_block_seg": tiled.BlockSeg}
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "qgtc_b200.h"', "int main(void) {"]
    for cname, cls in mirrors.items():
        lines.append(f'  printf("{cname} sizeof %zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            lines.append(f'  printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True,
                   capture_output=True, text=True)
    got = {}
    for line in subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.splitlines():
        cname, field, val = line.split()
        got[cname, field] = int(val)
    for cname, cls in mirrors.items():
        assert got[cname, "sizeof"] == ctypes_sizeof(cls), cname
        for fname, _ in cls._fields_:
            assert got[cname, fname] == getattr(cls, fname).offset, (cname, fname)


def ctypes_sizeof(cls):
    import ctypes
    return ctypes.sizeof(cls)


def test_tiled_chain_argument_validation_needs_no_gpu():
    """qg_tiled_gemm rejects malformed qg_chain requests before any CUDA call."""
    import ctypes

    from paper_2111_09547_b200 import tiled
    lib = N.lib()
    lib.qg_tiled_gemm.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    lib.qg_tiled_gemm.restype = ctypes.c_int
    epi, epi2 = N.Epilogue(), N.Epilogue()
    epi.out_kind, epi2.out_kind = N.OUT_PLANES, N.OUT_PLANES
    fake = ctypes.c_uint64(0)                  # never dereferenced by the validation

    def call(**kw):
        a = tiled.TiledArgs()
        a.segs, a.nsegs, a.total_ctas = ctypes.addressof(fake), 1, 2
        a.b_npad, a.n, a.bn, a.n_tiles = 64, 64, 64, 1
        a.mode, a.out_layout = N.GEMM_EPILOGUE, 1
        a.epi = ctypes.pointer(epi)
        c = tiled.Chain()
        c.w, c.w_npad, c.n, c.out_layout, c.out_npad = ctypes.addressof(fake), 64, 40, 2, 64
        c.epi = ctypes.pointer(epi2)
        for k, v in kw.items():                  # c_<field>: the chain, else the launch args
            if k.startswith("c_"):
                setattr(c, k[2:], v)
            else:
                setattr(a, k, v)
        a.chain = ctypes.addressof(c)
        return lib.qg_tiled_gemm(ctypes.byref(a), None)

    assert call(c_w_npad=48) == N.QG_ERR_ARG                  # not a power of two
    assert call(c_n=65) == N.QG_ERR_ARG                       # more columns than w_npad
    assert call(c_out_layout=1) == N.QG_ERR_ARG               # stage 2 writes right tiles or fp64
    assert call(c_out_layout=0) == N.QG_ERR_ARG               # fp64 output needs an OUT_REAL epilogue
    assert call(n_tiles=2, b_npad=128) == N.QG_ERR_UNSUPPORTED  # stage 1 is one N tile
    assert call(c_reserved=1) == N.QG_ERR_UNSUPPORTED         # reserved field (removed split chain)
    assert call(reserved3=1) == N.QG_ERR_UNSUPPORTED          # reserved field (removed dataflow epoch)
    assert call(mode=N.GEMM_I32) == N.QG_ERR_UNSUPPORTED      # stage 1 must requantize
    mean = (ctypes.c_double * 1)(0.0)
    epi2.bn_mean = ctypes.cast(mean, ctypes.c_void_p)         # BN without its other vectors
    assert call() == N.QG_ERR_ARG
