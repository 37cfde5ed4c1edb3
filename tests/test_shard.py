"""Multi-GPU host logic on CPU: LPT batch sharding and the one-
collective logit gather, exercised with world_size 2 over gloo (the GPU run uses
NCCL with the same code)."""

import os
import socket

import numpy as np
import pytest
import torch

from paper_2111_09547_b200 import shard, synth


def test_lpt_plan_is_a_deterministic_partition():
    rng = np.random.default_rng(0)
    costs = rng.uniform(1, 10, 188)
    for world in (1, 2, 4, 8):
        plan = shard.assign_lpt(costs, world)
        assert plan == shard.assign_lpt(costs, world)
        flat = sorted(i for ids in plan for i in ids)
        assert flat == list(range(188))
        # LPT bound: makespan <= (4/3 - 1/(3m)) OPT <= that x mean-based bound
        assert shard.imbalance(costs, plan) <= 4 / 3
    # equal costs (C4: equal parts) -> round-robin-like: sizes differ by at most one
    plan = shard.assign_lpt([1.0] * 188, 8)
    sizes = [len(p) for p in plan]
    assert max(sizes) - min(sizes) <= 1


def test_batch_costs_follow_part_sizes():
    cfg = synth.CONFIGS["C4"]
    sizes = synth.batch_part_sizes(cfg)
    assert len(sizes) == -(-cfg.num_parts // cfg.parts_per_batch)
    assert sum(int(s.sum()) for s in sizes) == cfg.num_nodes
    costs = [shard.batch_cost(s, cfg.in_dim, cfg.bits) for s in sizes]
    assert all(c > 0 for c in costs)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gather_worker(rank, world, port, rows, classes, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        costs = [float(r) ** 2 for r in rows]
        plan = shard.assign_lpt(costs, world)
        g = shard.LogitGather(plan, rows, classes, device="cpu")
        starts = np.cumsum([0] + list(rows))
        # batch b's logits: global row index * 1000 + class (recognisable after the gather)
        outs = []
        for b in plan[rank]:
            r = torch.arange(starts[b], starts[b + 1], dtype=torch.float64)[:, None]
            outs.append(r * 1000 + torch.arange(classes, dtype=torch.float64)[None, :])
        for _ in range(2):                       # buffers are reused across epochs
            full = g.gather(outs)
        if rank == 0:
            q.put(full.numpy())
        else:
            assert full is None
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_logit_gather_world2_gloo(world):
    rows = [7, 130, 1, 64, 300, 5, 33]
    classes = 3
    ctx = torch.multiprocessing.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, rows, classes, q)) for r in range(world)]
    for p in procs:
        p.start()
    full = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = np.arange(sum(rows), dtype=np.float64)[:, None] * 1000 + np.arange(classes)[None, :]
    np.testing.assert_array_equal(full, want)


@pytest.mark.gpu
def test_sharded_epoch_assembles_like_the_whole_epoch():
    """Single-process check of the sharded bench path: every rank's LPT share runs as its
    own epoch graph; reassembling the shares in global batch order (LogitGather.assemble,
    what rank 0 does after the all_gather) equals the whole epoch on one GPU, bit for bit."""
    from paper_2111_09547_b200.runtime import EpochRunner
    cfg = synth.with_bits(synth.CONFIGS["C3"], 4)
    ids = list(range(6))
    sizes = synth.batch_part_sizes(cfg)[:6]
    batches, feats, _ = synth.planted_batches(cfg, seed=0, batch_ids=ids)
    model = synth.calibrated_model(cfg, batches[0], feats[0])
    whole = torch.cat([o.cpu() for o in EpochRunner(model, batches, rescan=False).capture().run()])
    world = 2
    plan = shard.assign_lpt([shard.batch_cost(s, cfg.in_dim, cfg.bits) for s in sizes], world)
    rows = [b.total_nodes for b in batches]
    g = shard.LogitGather(plan, rows, model.layers[-1].out_dim, device="cpu")
    recv = torch.zeros_like(g.recv)
    for rank in range(world):
        r = EpochRunner(model, [batches[i] for i in plan[rank]], rescan=False).capture()
        outs = r.run()
        torch.cuda.synchronize()
        flat = torch.cat([o.cpu() for o in outs]) if outs else torch.zeros((0, g.classes), dtype=torch.float64)
        recv[rank * g.pad: rank * g.pad + flat.shape[0]] = flat
    assert torch.equal(g.assemble(recv), whole)
