"""RunReport / CSV schema (cli.py:41-94, tests/test_cli.py TestCsv) on CPU, and one
harness run over device batches (-m gpu)."""

import csv
import dataclasses

import numpy as np
import pytest

from paper_2111_09547_b200 import report as R


def _fake(**kw):
    base = {f.name: (0 if f.type in ("int", int) else 0.0 if f.type in ("float", float) else
                     False if f.type in ("bool", bool) else "x") for f in dataclasses.fields(R.RunReport)}
    base.update(dict(dataset="cliques.txt", model="gcn", reuse="cross-tile", jump=True, self_loops=True,
                     skip_ratio=0.25, layers=3, hidden=16, tiles_total=64, tiles_skipped=16))
    base.update(kw)
    return R.RunReport(**base)


def test_columns_match_the_reference_schema():
    # cli.py:41-79 field order is the CSV contract
    assert R.CSV_COLUMNS[:3] == ["dataset", "num_parts", "batch_size"]
    assert R.CSV_COLUMNS[-2:] == ["mean_logit_dev", "max_logit_dev"]
    assert len(R.CSV_COLUMNS) == 30


def test_skip_ratio_is_validated():
    with pytest.raises(ValueError):
        _fake(skip_ratio=1.5)


def test_single_report_two_lines_and_round_trip(tmp_path):
    rep = _fake(mean_logit_dev=0.125, compound_bytes=1234)
    out = tmp_path / "r.csv"
    R.emit_csv([rep], out)
    lines = out.read_text().strip().splitlines()
    assert len(lines) == 2 and lines[0].split(",") == R.CSV_COLUMNS
    with open(out, newline="") as fh:
        row = list(csv.DictReader(fh))[0]
    for f in dataclasses.fields(rep):
        assert row[f.name] == str(getattr(rep, f.name))


def test_empty_reports_rejected(tmp_path):
    with pytest.raises(ValueError):
        R.emit_csv([], tmp_path / "r.csv")
    assert not (tmp_path / "r.csv").exists()


@pytest.mark.gpu
def test_run_batches_on_two_cliques():
    """The reference's clustered-graph harness checks (test_cli.py TestRun) over device batches."""
    import paper_2111_09547_b200 as bg
    from paper_2111_09547_b200 import engine
    size, cliques = 80, 2
    edges = np.array([(b * size + i, b * size + j) for b in range(cliques) for i in range(size)
                      for j in range(size) if i != j])
    rng = np.random.default_rng(3)
    feats = rng.uniform(0.0, 1.0, (size * cliques, 12))
    g = bg.Graph(size * cliques, edges, feats)
    assign = bg.PartitionAssignment(2, np.repeat(np.arange(cliques), size))
    xp = bg.QuantParams(float(feats.min()), float(feats.max()), 4)
    batch = bg.build_batch(g, assign, [0, 1], xp)
    model = engine.gcn_model(12, 4, hidden_dim=16, num_layers=3, feature_bits=4, weight_bits=4, seed=3)
    engine.calibrate_model(model, batch, feats[batch.node_ids])
    rep = R.run_batches([batch], [feats[batch.node_ids]], model, rounds=1, num_parts=2, batch_size=2,
                        dataset="cliques.txt", seed=3)
    assert rep.model == "gcn" and rep.hidden == 16 and rep.layers == 3
    assert 0.0 <= rep.skip_ratio <= 1.0 and rep.tiles_skipped > 0
    assert rep.compound_bytes < rep.float32_dense_bytes
    nojump = R.run_batches([batch], [feats[batch.node_ids]], model, rounds=1, jump=False)
    assert nojump.mean_logit_dev == rep.mean_logit_dev and nojump.max_logit_dev == rep.max_logit_dev
    # the device fp32 reference agrees with the host numpy one (fidelity only)
    host = engine.reference_forward_f32(batch, feats[batch.node_ids], model)
    dev = engine.reference_forward_f32_device(batch, feats[batch.node_ids], model)
    np.testing.assert_allclose(dev, host, rtol=1e-4, atol=1e-4)
