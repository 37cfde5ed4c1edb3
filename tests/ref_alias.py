"""pytest plugin: run the reference's OWN test suite against this package.

Loaded with ``-p ref_alias`` by tests/test_gpu_ref_suite.py on the staged copy
of the reference tests (``oracle/_ref/ref_tests``, see oracle/make_ref.py).  It
registers ``bitgnn`` -> ``paper_2111_09547_b200`` and ``bitgnn_bindings`` ->
``paper_2111_09547_b200.bindings`` in ``sys.modules`` before the test modules
import them, so every ``from bitgnn import ...`` in the reference tests binds our
CUDA-backed implementation.  Every name the tests use -- graph IO and the
partitioner included (graph.py:85-262; the partitioner runs natively,
csrc/qgtc_partition.cu) -- comes from this package; nothing is served by the
reference.
"""

from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _install():
    import paper_2111_09547_b200 as ours
    from paper_2111_09547_b200 import bindings as our_bindings

    sys.modules["bitgnn"] = ours
    import paper_2111_09547_b200.cli  # noqa: F401  (bitgnn.cli: the bench CLI on the B200 path)
    for sub in ("bitgemm", "bitpack", "engine", "errors", "graph", "quantize", "cli"):
        sys.modules[f"bitgnn.{sub}"] = getattr(ours, sub)
    sys.modules["bitgnn_bindings"] = our_bindings


_install()


def pytest_report_header(config):
    import paper_2111_09547_b200 as ours
    return [f"ref_alias: bitgnn -> {ours.__file__} (no names served by the reference)"]
