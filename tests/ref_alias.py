"""pytest plugin: run the reference's OWN test suite against this package.

Loaded with ``-p ref_alias`` by tests/test_gpu_ref_suite.py on the staged copy
of the reference tests (``oracle/_ref/ref_tests``, see oracle/make_ref.py).  It
registers ``bitgnn`` -> ``paper_2111_09547_b200`` and ``bitgnn_bindings`` ->
``paper_2111_09547_b200.bindings`` in ``sys.modules`` before the test modules
import them, so every ``from bitgnn import ...`` in the reference tests binds our
CUDA-backed implementation.

Out-of-scope names (graph IO and the BFS partitioner,
graph.py:85-262 -- host preprocessing outside the reference's timed region) are
not part of this package.  The reference tests still call them to BUILD their
inputs, so the alias serves exactly those six names from the staged reference
(loaded as ``_ref_bitgnn``), converting Graph / PartitionAssignment objects at
the boundary.  Everything the hot path computes comes from our package.
"""

from __future__ import annotations

import importlib.util
import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DIR = os.path.join(ROOT, "oracle", "_ref")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

OUT_OF_SCOPE = ("partition", "edge_cut", "import_partition", "export_partition", "load_graph", "save_graph")


def _load_staged_reference():
    init = os.path.join(REF_DIR, "bitgnn", "__init__.py")
    spec = importlib.util.spec_from_file_location("_ref_bitgnn", init,
                                                  submodule_search_locations=[os.path.dirname(init)])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["_ref_bitgnn"] = mod
    # one exception hierarchy: the reference's host helpers raise OUR classes, which
    # the tests import from `bitgnn` (pytest.raises(FormatError, ...))
    from paper_2111_09547_b200 import errors as our_errors
    sys.modules["_ref_bitgnn.errors"] = our_errors
    spec.loader.exec_module(mod)
    return mod


def _install():
    import paper_2111_09547_b200 as ours
    from paper_2111_09547_b200 import bindings as our_bindings

    ref = _load_staged_reference()

    def to_ref_graph(g):
        return ref.Graph(g.num_nodes, g.edges, g.features)

    def to_ours_assign(a):
        return ours.PartitionAssignment(a.num_parts, a.part_of, a.edge_cut)

    def partition(g, num_parts, seed=0):
        return to_ours_assign(ref.partition(to_ref_graph(g), num_parts, seed=seed))

    def edge_cut(g, assign):
        return ref.edge_cut(to_ref_graph(g), ref.PartitionAssignment(assign.num_parts, assign.part_of))

    def import_partition(path, num_nodes=None, *args, **kw):
        return to_ours_assign(ref.import_partition(path, num_nodes, *args, **kw))

    def export_partition(assign, path):
        return ref.export_partition(ref.PartitionAssignment(assign.num_parts, assign.part_of), path)

    def load_graph(path, fmt="edge-list-text"):
        g = ref.load_graph(path, fmt)
        return ours.Graph(g.num_nodes, g.edges, g.features)

    def save_graph(g, path, fmt="edge-list-text"):
        return ref.save_graph(to_ref_graph(g), path, fmt)

    alias = types.ModuleType("bitgnn")
    alias.__dict__.update({k: v for k, v in vars(ours).items() if not k.startswith("__")})
    alias.__doc__ = "alias of paper_2111_09547_b200 for the reference test suite"
    alias.__path__ = list(ours.__path__)
    for name, fn in zip(OUT_OF_SCOPE, (partition, edge_cut, import_partition, export_partition, load_graph,
                                       save_graph)):
        setattr(alias, name, fn)
    alias._served_by_reference = OUT_OF_SCOPE
    sys.modules["bitgnn"] = alias
    for sub in ("bitgemm", "bitpack", "engine", "errors", "graph", "quantize"):
        sys.modules[f"bitgnn.{sub}"] = getattr(ours, sub)
    sys.modules["bitgnn_bindings"] = our_bindings


_install()


def pytest_report_header(config):
    import paper_2111_09547_b200 as ours
    return [f"ref_alias: bitgnn -> {ours.__file__}; served by the staged reference: {', '.join(OUT_OF_SCOPE)}"]
