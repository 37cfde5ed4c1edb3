"""QGTC B200 benchmark (driver contract).

Metric (BASELINE.json): QGNN inference ms/epoch per bitwidth, plus bit-GEMM
effective TOPS vs the tensor-pipe peak.  Default workload: configs[3] = C4, the
north star's target config -- a 3-layer GIN (hidden 256, 8-bit features /
activations / weights) over a synthetic ogbn-products-shaped planted graph
(2,449,029 nodes, 61.9M undirected edges, 1,500 parts, 8 parts per batch =
188 subgraph batches).  It fits one B200.

A step = one epoch = the reference's timed region (cli.py:215-222): every batch
through ``model_forward``.

* ``value``: device-resident ms/epoch, the epoch replayed as ONE CUDA graph, L2
  flushed between steps (the C4 inputs are also > L2).
* ``e2e``: the public runtime (``runtime.HostEpochRunner``): pinned host QGT3
  images -> H2D -> epoch -> fp64 logits D2H into pinned host memory, every
  step.  ``e2e_dropin``: the reference-API call sequence per batch,
  ``model_forward(unpack_batch(QGTB bytes), model)`` -> numpy (eager).
* N > 1: ``--gpus N`` spawns N ranks itself (torch.distributed.run) unless
  launched under torchrun.  Multi-batch configs (C3/C4) SHARD the batches (LPT,
  strong scaling, no data-path collective: every rank D2Hs its own logits over
  its own PCIe link); the NCCL gather of all logits to rank 0 is timed
  separately (``collective``).  Single-batch configs (C1/C2) run replicas.

``--impl reference`` times the REAL reference (``oracle/_ref/bitgnn``, staged
by oracle/make_ref.py) -- ``model_forward`` on batches built on the host by the
reference's own ``build_batch``, nothing from this package's kernels -- over a
process pool on all host cores, on a bounded sample of subgraph parts,
extrapolated to the epoch and labelled so.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")
METRIC = "QGNN inference ms/epoch per bitwidth; bit-GEMM effective TOPS vs TC peak"
PROFILE_SUMMARY = os.path.join(ROOT, "profiles", "ncu_summary.json")
INT8_PEAK_FILE = os.path.join(ROOT, "profiles", "int8_peak.json")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=30)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--config", default="C4", choices=["C1", "C2", "C3", "C4"])
    p.add_argument("--bits", type=int, default=None, help="feature/weight bits (default: the config's)")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-extras", action="store_true", help="skip the C2 bit sweep, the C5 point and bit_qnt")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-dropin", action="store_true")
    p.add_argument("--ref-budget-s", type=float, default=120.0)
    p.add_argument("--c5-n", type=int, default=16384)
    return p.parse_args()


# ----------------------------------------------------------------- helpers
def spawn_ranks(args) -> None:
    """--gpus N without torchrun: re-launch this script under torch.distributed.run."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def dist_setup(impl):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and impl == "ours":
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(world, v: float) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def host_info(cores_used: int) -> dict:
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"os_cpu_count": os.cpu_count(), "cores_used": cores_used, "lscpu_model": model}


class ClockSampler:
    """NVML sampler of SM clock + throttle reasons during the timed region."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index=0, period=0.0005):
        self.samples, self.reasons, self.period = [], set(), period
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max = None
        self._stop = threading.Event()

    def _loop(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def int8_peak_tops():
    if os.path.exists(INT8_PEAK_FILE):
        with open(INT8_PEAK_FILE) as fh:
            d = json.load(fh)
        return float(d["int8_tops"]), d.get("source", INT8_PEAK_FILE)
    bf16 = json.load(open(MEASURED))["bf16_tflops"] if os.path.exists(MEASURED) else 1590.0
    return 2.0 * bf16, "2 x measured bf16 (MEASURED_PEAKS.json)"


def hbm_peak_gbs():
    if os.path.exists(MEASURED):
        return float(json.load(open(MEASURED))["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    return 6531.9, "B200_PROFILING.md fallback"


def so_loaded() -> list:
    """In-tree native libraries mapped into this process (evidence for the arms)."""
    try:
        with open("/proc/self/maps") as fh:
            return sorted({ln.split()[-1] for ln in fh if ln.rstrip().endswith(".so") and ROOT in ln})
    except OSError:
        return []


# --------------------------------------------------------------- workload
def config_of(name, bits):
    from paper_2111_09547_b200 import synth_host
    base = synth_host.CONFIGS[name]
    return synth_host.with_bits(base, bits) if bits is not None else base


def build_workload(cfg, seed, batch_ids=None):
    """Batches (all, or ``batch_ids``) + a model calibrated on global batch 0 (cli.py:209)."""
    from paper_2111_09547_b200 import synth
    if batch_ids is None:
        batches, feats, _ = synth.planted_batches(cfg, seed=seed)
        model = synth.calibrated_model(cfg, batches[0], feats[0], seed=seed)
        return batches, feats, model
    b0, f0, _ = synth.planted_batches(cfg, seed=seed, batch_ids=[0])
    model = synth.calibrated_model(cfg, b0[0], f0[0], seed=seed)
    batches, feats, _ = synth.planted_batches(cfg, seed=seed, batch_ids=batch_ids)
    return batches, feats, model


def time_device_epochs(runner, steps, warmup, world):
    import torch
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")   # > 126 MB L2
    st = runner.stream
    with torch.cuda.stream(st):
        for _ in range(warmup):
            flush.zero_()
            runner.run()
    torch.cuda.synchronize()
    barrier(world)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    sampler = ClockSampler(torch.cuda.current_device())
    with sampler:
        torch.cuda.synchronize()
        with torch.cuda.stream(st):
            for s, e in ev:
                flush.zero_()
                s.record(st)
                runner.run()
                e.record(st)
        torch.cuda.synchronize()
    barrier(world)
    total_ms = sum(s.elapsed_time(e) for s, e in ev)
    return total_ms, sampler.summary()


def time_e2e(host_runner, steps, warmup, world):
    import torch
    st = host_runner.stream
    for _ in range(warmup):
        host_runner.run_host()
        st.synchronize()
    barrier(world)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    t0 = time.perf_counter()
    for s, e in ev:
        s.record(st)
        out = host_runner.run_host()
        e.record(st)
        st.synchronize()            # the caller reads the logits every step
        _ = float(out[0, 0])
    wall = (time.perf_counter() - t0) * 1e3
    barrier(world)
    return sum(s.elapsed_time(e) for s, e in ev), wall


def time_dropin(batches, model, steps, world):
    """Reference-API sequence per batch: QGTB bytes on the host -> unpack_batch (one H2D)
    -> model_forward -> numpy fp64 logits.  Wall clock per epoch (host-synchronous API)."""
    import torch
    import paper_2111_09547_b200 as bg
    bufs = [bg.pack_batch(b).data for b in batches]
    h2d = sum(len(x) for x in bufs)
    d2h = sum(b.total_nodes for b in batches) * model.layers[-1].out_dim * 8

    def epoch():
        return [bg.model_forward(bg.unpack_batch(x), model) for x in bufs]
    epoch()
    torch.cuda.synchronize()
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(steps):
        outs = epoch()
    ms = (time.perf_counter() - t0) * 1e3 / steps
    barrier(world)
    return ms, h2d, d2h, outs


def kernel_roofline(model, batches, reps=20):
    """Bit-GEMM launch durations inside the epoch graph.  CUDA events cannot sit between
    the kernels of one graph, so an identical epoch graph is captured with per-CTA
    %globaltimer stamps (first CTA entry -> last CTA exit = the launch's span); it is
    replayed like a timed step (L2 flushed before each replay) and CUDA events around
    each replay give the step time the spans are a share of."""
    import torch
    from paper_2111_09547_b200.runtime import EpochRunner
    r = EpochRunner(model, batches, rescan=False).capture(stamps=True)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    spans, ops, launches, step_ms = 0.0, 0.0, 0, 0.0
    per = None
    with torch.cuda.stream(r.stream):
        for i in range(reps + 3):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(r.stream)
            r.run()
            e.record(r.stream)
            torch.cuda.synchronize()
            if i < 3:
                continue
            ks = r.kernel_spans()
            per = [[0.0, w] for _, w in ks] if per is None else per
            for j, (t, _) in enumerate(ks):
                per[j][0] += t
            spans += sum(t for t, _ in ks)
            ops += sum(w for _, w in ks)
            launches += len(ks)
            step_ms += s.elapsed_time(e)
    del r
    kernel_roofline.per_launch = [(t / reps, w) for t, w in (per or [])]
    return spans / reps, ops / reps, launches / reps, step_ms / reps


# --------------------------------------------------- real reference (CPU)
def _ref_module():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import ref_inputs
    return ref_inputs.ref_module()


def _ref_model(R, cfg, seed):
    import ref_inputs
    return ref_inputs.ref_model(R, cfg, seed)


def ref_part_batch(R, cfg, seed, b, p):
    import ref_inputs
    return ref_inputs.ref_part_batch(R, cfg, seed, b, p)


def sample_parts(cfg, n, seed=0):
    """A fixed spread of (batch, part) ids: first and last part, the rest seeded random."""
    from paper_2111_09547_b200 import synth_host as H
    nb = H.num_batches(cfg)
    allp = [(b, p) for b in range(nb) for p in range(len(H.batch_part_sizes(cfg)[b]))]
    if n >= len(allp):
        return allp
    rng = np.random.default_rng(seed)
    mid = rng.choice(np.arange(1, len(allp) - 1), size=max(0, n - 2), replace=False)
    return [allp[0]] + [allp[i] for i in sorted(mid)] + [allp[-1]]


_POOL_STATE = {}


def _pool_forward(i):
    from threadpoolctl import threadpool_limits
    R, model, batches = _POOL_STATE["R"], _POOL_STATE["model"], _POOL_STATE["batches"]
    with threadpool_limits(1):
        t0 = time.perf_counter()
        R.model_forward(batches[i], model)
        return time.perf_counter() - t0


def reference_arm(args, world, rank):
    """--impl reference: the real bitgnn.model_forward on host-built batches, all cores."""
    if rank != 0:
        return
    import multiprocessing as mp
    cfg = config_of(args.config, args.bits)
    R = _ref_module()
    if R is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not staged (python oracle/make_ref.py)"}))
        return
    from paper_2111_09547_b200 import synth_host as H
    cores = os.cpu_count() or 1
    total_parts = cfg.num_parts
    t0 = time.perf_counter()
    model = _ref_model(R, cfg, seed=0)
    sample = sample_parts(cfg, cores)
    batches = [ref_part_batch(R, cfg, 0, b, p)[0] for b, p in sample]
    setup_s = time.perf_counter() - t0
    _POOL_STATE.update(R=R, model=model, batches=batches)
    pool_n = min(cores, len(batches))
    ctx = mp.get_context("fork")
    with ctx.Pool(pool_n) as pool:
        t0 = time.perf_counter()
        pool.map(_pool_forward, range(len(batches)), chunksize=1)
        one = time.perf_counter() - t0
        steps = max(1, min(args.steps, int(args.ref_budget_s / max(one, 1e-3))))
        warm = min(args.warmup, 1)          # the probe step above is the first warm-up
        for _ in range(max(0, warm - 1)):
            pool.map(_pool_forward, range(len(batches)), chunksize=1)
        times = []
        for _ in range(steps):
            t0 = time.perf_counter()
            pool.map(_pool_forward, range(len(batches)), chunksize=1)
            times.append(time.perf_counter() - t0)
    step_s = float(np.mean(times))
    sample_nodes = sum(b.total_nodes for b in batches)
    ms = step_s * 1e3 * cfg.num_nodes / sample_nodes
    hi = host_info(pool_n)
    line = {
        "metric": METRIC, "impl": "reference",
        "value": round(ms, 3), "unit": "ms/epoch", "n_gpus": world, "steps": steps, "warmup": warm,
        "ms_per_step": round(ms, 3), "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": f"u{cfg.bits} codes (numpy bit-serial AND+popcount, fp64 epilogue)",
        "data": "synthetic planted-partition graph, U[0,1) features, random-init weights",
        "config": {"workload": cfg.name, "model": f"{cfg.model} {cfg.layers} layers hidden {cfg.hidden}",
                   "bits": cfg.bits, "nodes": cfg.num_nodes, "edges_undirected": cfg.num_edges,
                   "parts": cfg.num_parts, "batches": H.num_batches(cfg)},
        "cpu_baseline": {"value": round(ms, 3), "unit": "ms/epoch", "cores": pool_n, "kind": "reference",
                         "sample": (f"real reference bitgnn.model_forward (oracle/_ref, staged unmodified from "
                                    f"/root/reference) on {len(batches)} of {total_parts} subgraph parts "
                                    f"({sample_nodes} of {cfg.num_nodes} nodes; first, last and seeded-random "
                                    f"parts), each a one-part SubgraphBatch from the reference's build_batch, "
                                    f"{pool_n}-process pool (1 BLAS thread each); step time x "
                                    f"{cfg.num_nodes / sample_nodes:.1f} (node-proportional) = EXTRAPOLATED "
                                    f"ms/epoch"),
                         "host": hi, "setup_s": round(setup_s, 1), "step_s": [round(t, 3) for t in times]},
        "e2e": {"value": round(ms, 3), "unit": "ms/epoch", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "our_native_so_loaded": so_loaded(),
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_one_core(cfg, model_ours, logits_batch0, budget_s=60.0):
    """1-core real-reference time on the first part(s) of batch 0, extrapolated; the
    reference's logits are compared with ours for those rows (config-scale parity)."""
    from threadpoolctl import threadpool_limits
    R = _ref_module()
    if R is None:
        return None
    t0 = time.perf_counter()
    model = _ref_model(R, cfg, seed=0)
    setup_s = time.perf_counter() - t0
    # calibrated grids must be the ones our engine derived (engine.calibrate_model mirror)
    def grid(q):
        return None if q is None else (q.alpha_min, q.alpha_max, q.bits)
    grids_equal = all(
        grid(a.mid_params) == grid(b.mid_params) and grid(a.out_params) == grid(b.out_params)
        for a, b in zip(model.layers, model_ours.layers))
    rb, lo, hi = ref_part_batch(R, cfg, 0, 0, 0)
    with threadpool_limits(1):
        t0 = time.perf_counter()
        out = R.model_forward(rb, model)
        t = time.perf_counter() - t0
    exact = bool(np.array_equal(out, logits_batch0[lo:hi]))
    ms = t * 1e3 * cfg.num_nodes / (hi - lo)
    return {"value": round(ms, 1), "unit": "ms/epoch", "cores": 1, "kind": "reference",
            "sample": (f"real reference bitgnn.model_forward (oracle/_ref), 1 core, on part 0 of batch 0 "
                       f"({hi - lo} nodes, {t:.2f} s), x{cfg.num_nodes / (hi - lo):.0f} node-proportional = "
                       f"EXTRAPOLATED ms/epoch"),
            "parity_vs_reference_on_sample": "bit-exact" if exact else "MISMATCH",
            "calibrated_grids_equal": bool(grids_equal), "setup_s": round(setup_s, 1),
            "host": host_info(1)}


# ------------------------------------------------------------------ extras
def c2_sweep(steps):
    """configs[1]: the C2 bit sweep 1..8 (device ms/epoch, one graph per epoch)."""
    from paper_2111_09547_b200.runtime import EpochRunner
    out = {}
    for bits in range(1, 9):
        cfg = config_of("C2", bits)
        bb, _, mm = build_workload(cfg, seed=0)
        rr = EpochRunner(mm, bb, rescan=False).capture()
        t, _ = time_device_epochs(rr, steps, 5, 1)
        out[str(bits)] = round(t / steps, 5)
        del rr, bb, mm
    return out


def c5_point(n, bits, peak):
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from c5_sweep import run_point
    c5 = run_point(n, 0.1, bits, reps=10, int8_peak=peak, packed=True)
    c5.update({"bound": "tensor", "peak": peak, "unit": "TOPS",
               "kernel": "tc_pair_kernel (2-SM cluster, tcgen05.mma.cta_group::2.kind::i8 M=256, TMA)",
               "config": "C5: A Bernoulli(0.1) 1-bit x X uniform codes, reduce_bitplanes(bmm_1bit_by_nbit) "
                         "in one launch, CUDA-graph replays timed with CUDA events; *_from_packed adds the "
                         "operand preparation from packed inputs (zero-tile scan + block expansion of A, "
                         "X planes -> tiled codes), timed separately with CUDA events"})
    # block-diagonal A (16 diagonal blocks): zero-tile jumping skips 15/16 of the tiles
    bd = run_point(n, 0.1, bits, reps=10, int8_peak=peak, diag_blocks=16, packed=True)
    c5["block_diagonal_16"] = {k: bd[k] for k in ("ms", "alg_tops", "eff_tops", "frac", "nonzero_blocks",
                                                  "total_blocks", "parity_sampled_rows", "ms_from_packed",
                                                  "frac_from_packed")}
    return c5


# ------------------------------------------------------------------- ours
def ours(args, world, rank):
    import torch
    from paper_2111_09547_b200 import _native as N
    from paper_2111_09547_b200 import shard, synth_host
    from paper_2111_09547_b200.runtime import EpochRunner, HostEpochRunner

    N.lib()
    cfg = config_of(args.config, args.bits)
    sizes = synth_host.batch_part_sizes(cfg)
    sharded = world > 1 and len(sizes) > 1
    plan = None
    if sharded:
        # strong scaling over independent subgraph batches: LPT plan, same on every rank
        costs = [shard.batch_cost(s, cfg.in_dim, cfg.bits) for s in sizes]
        plan = shard.assign_lpt(costs, world)
        batches, feats, model = build_workload(cfg, seed=0, batch_ids=plan[rank])
    else:
        # replicas (a single-batch config cannot shard): every rank its own epoch
        batches, feats, model = build_workload(cfg, seed=rank)
    runner = EpochRunner(model, batches, rescan=False).capture()
    total_ms, clocks = time_device_epochs(runner, args.steps, args.warmup, world)
    total_ms = max_over_ranks(world, total_ms)
    epochs = args.steps if sharded else args.steps * world
    ms_epoch = total_ms / epochs
    launches = runner.kernel_launches_per_epoch() * args.steps

    # end to end through the public runtime: pinned H2D -> graph -> D2H every step (per rank)
    host = HostEpochRunner(model, batches)
    e2e_ms, e2e_wall = time_e2e(host, args.steps, min(args.warmup, 5), world)
    e2e_ms = max_over_ranks(world, e2e_ms) / epochs
    with torch.cuda.stream(runner.stream):
        dev_out = runner.run()
        dev_logits = torch.cat(list(dev_out))
    torch.cuda.synchronize()
    dev_logits_h = dev_logits.cpu()
    host_out = host.run_host()
    host.stream.synchronize()
    e2e_parity = bool(torch.equal(dev_logits_h, host_out))
    logits_b0 = dev_out[0].cpu().numpy()
    e2e_h2d, e2e_d2h = host.h2d_bytes, host.d2h_bytes
    del host
    torch.cuda.empty_cache()

    collective = None
    if sharded:
        # the only collective: all logits to rank 0 (NCCL over NVLink), timed on its own
        import torch.distributed as dist
        rows = [int(s.sum()) for s in sizes]
        gather = shard.LogitGather(plan, rows, model.layers[-1].out_dim, torch.device("cuda"))
        outs = list(dev_out)
        for _ in range(2):
            gather.gather(outs)
        torch.cuda.synchronize()
        dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k = 5
        s.record()
        for _ in range(k):
            gather.gather(outs)
        e.record()
        torch.cuda.synchronize()
        gms = max_over_ranks(world, s.elapsed_time(e) / k)
        collective = {"op": "LogitGather (one all_gather_into_tensor of padded fp64 logit shards, NCCL)",
                      "ms_per_epoch": round(gms, 4), "bytes_per_rank": int(gather.send.numel() * 8),
                      "in_value": False}
        del gather

    dropin = None
    if not args.no_dropin:
        k = max(1, min(3, args.steps))
        d_ms, d_h2d, d_d2h, d_outs = time_dropin(batches, model, k, world)
        d_ms = max_over_ranks(world, d_ms) * (1 if sharded else 1.0 / world)
        dropin = {"value": round(d_ms, 3), "unit": "ms/epoch", "h2d_bytes_per_step": d_h2d,
                  "d2h_bytes_per_step": d_d2h, "steps": k,
                  "parity_vs_device_path": "bit-exact" if bool(np.array_equal(np.concatenate(d_outs),
                                                                                 dev_logits_h.numpy()))
                  else "MISMATCH",
                  "path": "per batch: pack_batch QGTB bytes (host) -> unpack_batch (one H2D) -> "
                          "model_forward -> numpy fp64 logits (eager, host-synchronous; wall clock)"}
        del d_outs

    # roofline of the dominant kernel (bit-GEMM) -- algorithmic int8-MAC work per launch
    gemm_ms, gemm_ops, gemm_launches, stamped_step_ms = kernel_roofline(model, batches)
    peak, peak_src = int8_peak_tops()
    achieved = gemm_ops / (gemm_ms * 1e-3) / 1e12
    traffic = None
    if os.path.exists(PROFILE_SUMMARY):
        try:
            traffic = json.load(open(PROFILE_SUMMARY)).get(f"{cfg.name}:bitgemm_dram_bytes_per_launch")
        except Exception:
            traffic = None
    eff_tops = 2.0 * sum(
        b.total_nodes * b.total_nodes * (ly.out_dim if ly.order == "update-then-aggregate" else ly.in_dim)
        for b in batches for ly in model.layers) / (ms_epoch * 1e-3) / 1e12

    extras = {}
    cpu = None
    if rank == 0 and world == 1 and not args.no_extras:
        del runner
        torch.cuda.empty_cache()
        extras["c2_sweep_ms_per_epoch_by_bits"] = c2_sweep(max(20, args.steps))
        extras["gemm_roofline_c5"] = c5_point(args.c5_n, 4, peak)
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        from bitqnt_bench import run_bitqnt
        hbm, hbm_src = hbm_peak_gbs()
        extras["bitqnt_roofline"] = {
            "bound": "hbm", "unit": "GB/s", "peak_source": hbm_src,
            "work": "4*M*K fp32 in + s*Mpad*Kpad/8 plane bytes out + 8*M row-sum bytes per launch",
            "C3": run_bitqnt(169343, 128, 4, hbm_peak=hbm), "C4": run_bitqnt(2449029, 100, 8, hbm_peak=hbm)}
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_one_core(cfg, model, logits_b0)

    if rank != 0:
        return
    line = {
        "metric": METRIC,
        "value": round(ms_epoch, 5), "unit": "ms/epoch", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_epoch, 5), "higher_is_better": False,
        "scaling": "strong" if sharded else "weak", "vs_baseline": None,
        "dtype": f"u{cfg.bits} codes / s32 acc / fp64 epilogue",
        "data": "synthetic planted-partition graph, U[0,1) features, random-init weights",
        "config": {"workload": cfg.name, "model": f"batched-{cfg.model} {cfg.layers} layers hidden {cfg.hidden}",
                   "bits": cfg.bits, "nodes": cfg.num_nodes, "edges_undirected": cfg.num_edges,
                   "parts": cfg.num_parts, "batches": len(sizes), "batches_this_rank": len(batches),
                   "in_dim": cfg.in_dim, "classes": cfg.classes,
                   "l2": "flushed between steps (256 MB write); inputs also > L2",
                   "parallelism": (f"batch-sharded x{world} (LPT; per-rank H2D/D2H, no data-path collective)"
                                   if sharded else f"replicas x{world}")},
        "effective_tops": round(eff_tops, 3),
        "roofline": {"bound": "tensor", "kernel": "tc_tiled_kernel (tcgen05.mma kind::i8, cp.async.bulk ring)",
                     "achieved": round(achieved, 3), "peak": peak, "unit": "TOPS",
                     "frac": round(achieved / peak, 5), "traffic": traffic, "peak_source": peak_src,
                     "work": "2 x 1024 x N_padded int8-MACs per non-zero 8x128 left tile (one u8 MAC "
                             "retires all bit-plane pairs)",
                     "durations": "per launch, %globaltimer from the later of its first CTA entry and the "
                                  "previous GEMM launch's last CTA exit (PDL lets CTAs enter early and wait) "
                                  "to its last CTA exit, inside an identical stamped epoch graph replayed "
                                  "after an L2 flush; CUDA events around each replay give stamped_step_ms",
                     "launches_per_epoch": gemm_launches, "kernel_ms_per_epoch": round(gemm_ms, 5),
                     "stamped_step_ms": round(stamped_step_ms, 5),
                     "kernel_share_of_step": round(gemm_ms / stamped_step_ms, 3),
                     "per_launch": [{"ms": round(t, 5), "tops": round(w / (t * 1e-3) / 1e12, 1) if t else None,
                                     "frac": round(w / (t * 1e-3) / 1e12 / peak, 4) if t else None}
                                    for t, w in getattr(kernel_roofline, "per_launch", [])]},
        "cpu_baseline": cpu,
        "e2e": {"value": round(e2e_ms, 5), "unit": "ms/epoch", "h2d_bytes_per_step": e2e_h2d,
                "d2h_bytes_per_step": e2e_d2h, "wall_ms_per_step": round(e2e_wall / args.steps, 5),
                "parity_vs_device_path": "bit-exact" if e2e_parity else "MISMATCH",
                "path": ("public runtime.HostEpochRunner, ONE CUDA graph per step: pinned QGT3 images (schedule + "
                         "non-zero 128x128 adjacency bit blocks + feature planes) -> H2D -> block expansion + "
                         "epoch -> fp64 logits -> D2H into pinned host memory (batch chunks pipelined on two "
                         "copy engines)" + (", per rank over its own PCIe link" if sharded else ""))},
        "e2e_dropin": dropin,
        "collective": collective,
        "gpu_launches": launches,
        "clocks": clocks,
        **extras,
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args)
    world, rank, _ = dist_setup(args.impl)
    if args.impl == "reference":
        reference_arm(args, world, rank)
    else:
        ours(args, world, rank)
    if world > 1 and args.impl == "ours":
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
