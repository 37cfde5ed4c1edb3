"""Benchmark report over device-resident batches: RunReport, CSV emission, one run.

Mirror of the reporting half of the reference harness (cli.py:41-93 RunReport /
CSV_COLUMNS / emit_csv, and the timed region + counters + fidelity of
cli.py:195-273).  Graph loading and partitioning (cli.py:150-193) are out of
scope here: ``run_batches`` starts from already-built
``SubgraphBatch``es, e.g. ``build_batch`` over a supplied partition or
``synth.planted_batches``, and the caller passes the partition / pack times it
measured.

Differences from the reference, by design:
* phase times come from the engine's per-stage clock with a device sync per
  stage (the reference times numpy phases);
* the float32 fidelity reference runs on the GPU (cuBLAS fp32) for batches
  above ``HOST_F32_MAX_NODES`` nodes, where the reference's dense numpy pass
  would take minutes; below it the host numpy pipeline of the reference is
  used as is.
"""

from __future__ import annotations

import csv
from dataclasses import asdict, dataclass, fields

import numpy as np

from .bitgemm import CROSS_BIT, CROSS_TILE
from .engine import KernelTally, model_forward, reference_forward_f32, reference_forward_f32_device
from .graph import float32_dense_bytes, pack_batch

HOST_F32_MAX_NODES = 4096


@dataclass
class RunReport:
    """One benchmark run: configuration, timings, counters, fidelity (cli.py:41-79)."""

    dataset: str
    num_parts: int
    batch_size: int
    bits_x: int
    bits_w: int
    model: str
    layers: int
    hidden: int
    rounds: int
    seed: int
    jump: bool
    reuse: str
    self_loops: bool
    partition_s: float
    pack_s: float
    aggregate_s: float
    update_s: float
    epilogue_s: float
    tile_mma_count: int
    tile_fetch_count: int
    tiles_skipped: int
    tiles_total: int
    skip_ratio: float
    word_and_popcount_count: int
    agg_word_and_popcount_count: int
    compound_bytes: int
    float32_dense_bytes: int
    bytes_ratio: float
    mean_logit_dev: float
    max_logit_dev: float

    def __post_init__(self):
        if not 0.0 <= self.skip_ratio <= 1.0:
            raise ValueError("skip_ratio must lie in [0, 1]")


CSV_COLUMNS = [f.name for f in fields(RunReport)]


def emit_csv(reports, path) -> None:
    """Write reports as CSV: stable column order, header row, one row per run (cli.py:85-94)."""
    reports = list(reports)
    if not reports:
        raise ValueError("no reports to write")
    with open(path, "w", newline="", encoding="utf-8") as fh:
        writer = csv.DictWriter(fh, fieldnames=CSV_COLUMNS)
        writer.writeheader()
        for r in reports:
            writer.writerow(asdict(r))


def run_batches(batches, batch_features, model, *, rounds: int = 1, jump: bool = True, reuse: str = CROSS_TILE,
                dataset: str = "synthetic", num_parts: int | None = None, batch_size: int = 8, seed: int = 0,
                self_loops: bool = True, partition_s: float = 0.0, pack_s: float = 0.0) -> RunReport:
    """The timed region + counters + fidelity of one reference harness run (cli.py:212-273)
    over built batches.  ``batch_features``: the real-valued features of each batch
    (rows in batch order), used only by the float32 fidelity reference."""
    if not batches:
        raise RuntimeError("no non-empty batches were produced")
    if rounds < 1:
        raise ValueError("rounds must be >= 1")
    clock: dict[str, float] = {}
    tally = KernelTally()
    logits = []
    for rnd in range(rounds):
        round_logits = [model_forward(b, model, jump=jump, reuse=reuse, clock=clock,
                                      tally=tally if rnd == 0 else None) for b in batches]
        if rnd == 0:
            logits = round_logits

    # ablation guard: scheduling flags must never change the logits (cli.py:224-228)
    other = CROSS_BIT if reuse == CROSS_TILE else CROSS_TILE
    check = model_forward(batches[0], model, jump=not jump, reuse=other)
    if not np.array_equal(check, logits[0]):
        raise RuntimeError("scheduling options changed the logits")

    abs_sum, abs_max, count = 0.0, 0.0, 0
    for b, feats, out in zip(batches, batch_features, logits):
        if b.total_nodes <= HOST_F32_MAX_NODES:
            ref = reference_forward_f32(b, feats, model)
        else:
            ref = reference_forward_f32_device(b, feats, model)
        d = np.abs(out - ref.astype(np.float64))
        abs_sum += float(d.sum())
        abs_max = max(abs_max, float(d.max()) if d.size else 0.0)
        count += d.size

    compound = sum(pack_batch(b).nbytes for b in batches)
    dense = sum(float32_dense_bytes(b) for b in batches)
    agg = tally.aggregation
    first = model.layers[0]
    hidden = model.layers[0].out_dim if len(model.layers) > 1 else first.out_dim
    return RunReport(
        dataset=dataset,
        num_parts=int(num_parts if num_parts is not None else sum(b.num_subgraphs for b in batches)),
        batch_size=batch_size,
        bits_x=model.feature_bits,
        bits_w=model.weight_bits,
        model="gcn" if model.kind == "cluster-gcn" else "gin",
        layers=len(model.layers),
        hidden=hidden,
        rounds=rounds,
        seed=seed,
        jump=jump,
        reuse=reuse,
        self_loops=self_loops,
        partition_s=partition_s,
        pack_s=pack_s,
        aggregate_s=clock.get("aggregate", 0.0) / rounds,
        update_s=clock.get("update", 0.0) / rounds,
        epilogue_s=clock.get("epilogue", 0.0) / rounds,
        tile_mma_count=tally.total.tile_mma_count,
        tile_fetch_count=tally.total.tile_fetch_count,
        tiles_skipped=agg.tiles_skipped,
        tiles_total=agg.tiles_total,
        skip_ratio=agg.tiles_skipped / agg.tiles_total if agg.tiles_total else 0.0,
        word_and_popcount_count=tally.total.word_and_popcount_count,
        agg_word_and_popcount_count=agg.word_and_popcount_count,
        compound_bytes=compound,
        float32_dense_bytes=dense,
        bytes_ratio=compound / dense if dense else 0.0,
        mean_logit_dev=abs_sum / count if count else 0.0,
        max_logit_dev=abs_max,
    )
