"""Host-side policy for chained stage pairs (engine._chain_ok): which aggregation ->
update pairs of the benchmark configs run as one launch, and in which form.  Pure host
logic (no GPU)."""

import types

import pytest

from paper_2111_09547_b200 import engine, synth


def _run(**kw):
    return types.SimpleNamespace(clock=kw.get("clock"), tally=kw.get("tally"))


def _row_blocks(cfg):
    return sum(-(-int(s.sum()) // 128) for s in synth.batch_part_sizes(cfg))


@pytest.fixture(autouse=True)
def _defaults():
    saved = engine.CHAIN
    engine.CHAIN = True
    yield
    engine.CHAIN = saved


def test_benchmark_configs_chain_as_measured():
    c1, c2, c3, c4 = (synth.CONFIGS[k] for k in ("C1", "C2", "C3", "C4"))
    # C1: 24 row blocks, split N, launch-latency bound -> one CTA per row block
    assert engine._chain_ok(_run(), c1.in_dim, c1.hidden, _row_blocks(c1)) == 1
    # C2: 79 row blocks, the two-launch path splits N in two -> stays two launches
    assert _row_blocks(c2) == 79
    assert engine._chain_ok(_run(), c2.hidden, c2.hidden, 79) == 0
    # C3 / C4: enough row blocks for full-width N tiles -> chained
    assert engine._chain_ok(_run(), c3.in_dim, c3.hidden, _row_blocks(c3)) == 1
    assert engine._chain_ok(_run(), c4.hidden, c4.hidden, _row_blocks(c4)) == 1


def test_split_stages_chain_only_with_few_row_blocks():
    assert engine._chain_ok(_run(), 64, 64, 79) == 0          # npad 64 split into 2 x 32
    assert engine._chain_ok(_run(), 32, 64, 79) == 1          # 32 columns: already one full-width tile
    assert engine._chain_ok(_run(), 256, 64, 50) == 0         # 4-way split, too many row blocks
    assert engine._chain_ok(_run(), 256, 64, 30) == 1         # 4-way split, few row blocks


def test_chain_is_off_whenever_its_preconditions_fail():
    assert engine._chain_ok(_run(clock={}), 128, 64, 500) == 0       # per-phase clock needs stages
    assert engine._chain_ok(_run(tally=object()), 128, 64, 500) == 0  # tallies need the codes
    assert engine._chain_ok(_run(), 300, 64, 500) == 0               # stage-1 wider than one tile
    assert engine._chain_ok(_run(), 128, 300, 500) == 0              # stage-2 wider than one tile
    engine.CHAIN = False
    assert engine._chain_ok(_run(), 128, 64, 500) == 0
