"""bit_qnt (K1) HBM roofline: fused quantize + bit-decompose + row-wise pack of a real
feature matrix (quantize.py:93-105 + bit_decompose :108-112 + pack_planes bitpack.py:
213-228) through the C-ABI ``qg_quantize_pack``, with int64 row sums.

Algorithmic bytes = 4*M*K (fp32 in) + s*Mpad*Kpad/8 (planes out) +
8*M (row sums).  Each timed launch follows an L2 flush (256 MB write, outside the
events); CUDA events on the launching stream.

    python tools/bitqnt_bench.py [rows cols bits]
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def run_bitqnt(rows: int, cols: int, bits: int, reps: int = 10, hbm_peak: float = 6554.6, seed: int = 0):
    import torch

    from paper_2111_09547_b200 import _native as N
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.rand((rows, cols), generator=g, device="cuda", dtype=torch.float32)
    pr, pc = -(-rows // 128) * 128, -(-cols // 8) * 8
    planes = torch.empty((bits, pr * pc // 32), dtype=torch.int32, device="cuda")
    rs = torch.zeros(rows, dtype=torch.int64, device="cuda")
    status = N.new_status()
    scale = 1.0 / (1 << bits)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()

    def launch():
        N.call("qg_quantize_pack", N.ptr(x), N.SRC_F32, rows, cols, cols, 0.0, scale, bits, N.ROW_WISE_ID, 8,
               N.ptr(planes), None, N.ptr(rs), None, N.ptr(status), N.stream())

    for _ in range(2):
        rs.zero_()
        launch()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(reps):
        flush.zero_()
        rs.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(st)
        launch()
        e.record(st)
        torch.cuda.synchronize()
        tot += s.elapsed_time(e)
    ms = tot / reps
    # spot parity: sampled rows' codes recomputed in fp64 (exact reference expression)
    idx = torch.randperm(rows, device="cuda", generator=g)[:256]
    want = torch.clamp(torch.floor((x[idx].double() - 0.0) / scale), 0, (1 << bits) - 1).to(torch.int64)
    got_sums = rs[idx]
    exact = bool(torch.equal(got_sums, want.sum(1)))
    nbytes = 4 * rows * cols + bits * pr * pc // 8 + 8 * rows
    gbs = nbytes / (ms * 1e-3) / 1e9
    return {"rows": rows, "cols": cols, "bits": bits, "ms": round(ms, 4), "bytes": nbytes,
            "achieved_gbs": round(gbs, 1), "peak_gbs": hbm_peak, "frac": round(gbs / hbm_peak, 4),
            "row_sums_sampled": "exact" if exact else "MISMATCH",
            "kernel": "quantize_pack_row_vec_kernel (lane = column, 128-B coalesced row loads, 32 rows in flight per warp, division-free exact requant, 8x8 bit transposes, redux.sync row sums, smem-staged 32-B plane stores)"}


if __name__ == "__main__":
    a = [int(v) for v in sys.argv[1:4]] if len(sys.argv) >= 4 else None
    shapes = [tuple(a)] if a else [(169343, 128, 4), (2449029, 100, 8)]
    for r, c, b in shapes:
        print(json.dumps(run_bitqnt(r, c, b)))
