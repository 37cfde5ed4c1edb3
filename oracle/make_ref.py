"""Recipe: stage the REAL reference next to the oracle -- TEST INFRASTRUCTURE ONLY.

The reference (``bitgnn``, /root/reference/pkg) is pure Python + numpy, so there
is nothing to compile: "building" it means copying its package and its own test
suite, unmodified, into ``oracle/_ref/`` (git-ignored, NOT gpurun-ignored, so it
travels to the GPU box like the built ``.so``).  Nothing is copied into tracked
files.  Run from the repo root where /root/reference exists (``__graft_entry__.
build()`` calls it):

    python oracle/make_ref.py

Layout written:
    oracle/_ref/bitgnn/            reference package   (pkg/src/bitgnn)
    oracle/_ref/bitgnn_bindings/   reference bindings  (pkg/bindings/src/bitgnn_bindings)
    oracle/_ref/ref_tests/         reference test suite (pkg/tests/*.py, pkg/bindings/tests/*.py)
    oracle/_ref/MANIFEST.json      source path + sha256 of every staged file

Users (only as checker or as the timed CPU baseline, never as the product):
* ``bench.py --impl reference`` and the ``cpu_baseline`` leg time
  ``oracle/_ref/bitgnn.model_forward`` on host-built batches;
* ``tests/test_gpu_ref_suite.py`` runs ``oracle/_ref/ref_tests`` with ``bitgnn``
  aliased to ``paper_2111_09547_b200`` (tests/ref_alias.py).
"""

from __future__ import annotations

import hashlib
import json
import os
import shutil
import sys

REF = os.environ.get("QGTC_REFERENCE", "/root/reference/pkg")
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "_ref")

COPIES = [
    ("src/bitgnn", "bitgnn"),
    ("bindings/src/bitgnn_bindings", "bitgnn_bindings"),
    ("tests", "ref_tests"),
    ("bindings/tests", "ref_tests"),
]


def _sha(path: str) -> str:
    with open(path, "rb") as fh:
        return hashlib.sha256(fh.read()).hexdigest()


def stage(ref: str = REF, out: str = OUT) -> bool:
    """Copy the reference package + tests; False (and nothing written) when absent."""
    if not os.path.isdir(os.path.join(ref, "src", "bitgnn")):
        return False
    tmp = out + ".tmp"
    shutil.rmtree(tmp, ignore_errors=True)
    manifest = {"source": os.path.abspath(ref), "files": {}}
    for src_rel, dst_rel in COPIES:
        src = os.path.join(ref, src_rel)
        dst = os.path.join(tmp, dst_rel)
        os.makedirs(dst, exist_ok=True)
        for name in sorted(os.listdir(src)):
            if not name.endswith(".py"):
                continue
            shutil.copyfile(os.path.join(src, name), os.path.join(dst, name))
            manifest["files"][f"{dst_rel}/{name}"] = {"from": f"{src_rel}/{name}",
                                                       "sha256": _sha(os.path.join(src, name))}
    with open(os.path.join(tmp, "MANIFEST.json"), "w") as fh:
        json.dump(manifest, fh, indent=1, sort_keys=True)
    shutil.rmtree(out, ignore_errors=True)
    os.replace(tmp, out)
    return True


def available(out: str = OUT) -> bool:
    return os.path.exists(os.path.join(out, "bitgnn", "engine.py"))


def import_reference(out: str = OUT):
    """Import the staged reference package (as ``bitgnn``) without shadowing ours."""
    if not available(out):
        raise FileNotFoundError(f"{out}/bitgnn missing: run `python oracle/make_ref.py` where /root/reference exists")
    if out not in sys.path:
        sys.path.insert(0, out)
    import bitgnn  # noqa: E402  (the staged reference)
    if not os.path.abspath(bitgnn.__file__).startswith(os.path.abspath(out)):
        raise ImportError(f"`bitgnn` resolved to {bitgnn.__file__}, not the staged reference")
    return bitgnn


if __name__ == "__main__":
    ok = stage()
    print("staged reference into oracle/_ref" if ok else f"reference not found at {REF}: nothing staged")
