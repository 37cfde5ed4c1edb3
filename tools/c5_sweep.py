"""C5 (BASELINE.json configs[4]): standalone 1-bit A x s-bit X bit-GEMM sweep vs the int8
tensor-pipe roofline.

A is Bernoulli(rho) M x K (column-wise 1-bit, the reference's adjacency layout),
X uniform integer codes in [0, 2^s) (test_acceptance.py:56-60), K x N row-wise.
The product is the reference's reduce_bitplanes(bmm_1bit_by_nbit(A, X))
(bitgemm.py:291-298, 306-371) computed by ``tiled.bmm_reduced`` in one launch,
replayed as a CUDA graph; CUDA events on the launch stream.

Algorithmic ops = 2 x 1024 x pad8(N) x non-zero 8x128 tiles of A;
effective TOPS (the paper's Table-3 convention) = 2 M N K / t.
Parity: sampled rows against an fp64 dense product (exact: values < 2^53).

    python tools/c5_sweep.py [--sizes 1024,4096,16384] [--rhos 0.001,0.01,0.1,0.5] [--bits 1,4,8]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def make_operands(n: int, rho: float, bits: int, seed: int = 0, diag_blocks: int = 1):
    import torch

    from paper_2111_09547_b200 import bitpack
    from paper_2111_09547_b200.tiled import TiledCodeStack, tiles_from_codes
    g = torch.Generator(device="cuda").manual_seed(seed)
    dense = (torch.rand((n, n), generator=g, device="cuda") < rho).to(torch.uint8)
    if diag_blocks > 1:
        # block-diagonal A (the batched-subgraph shape): zero-tile jumping skips the rest
        part = torch.arange(n, device="cuda") * diag_blocks // n
        dense &= (part[:, None] == part[None, :]).to(torch.uint8)
    a = bitpack.pack_colwise(dense, 8)
    codes = torch.randint(0, 1 << bits, (n, n), generator=g, device="cuda", dtype=torch.uint8)
    tiles, pitch = tiles_from_codes(codes, n, n, n, "right")
    x = TiledCodeStack(bitpack.ROW_WISE, n, n, bits, tiles, "right", pitch)
    return dense, codes, a, x


def time_preparation(a, codes, bits: int, reps: int = 3) -> float:
    """ms of the operand preparation the GEMM timing excludes, from PACKED inputs: the
    zero-tile scan + block gather/expansion of the column-wise 1-bit A (bitgemm.py:
    214-233) and X's row-wise bit planes -> right-tiled u8 codes (eager, host-synced
    schedule build included)."""
    import torch

    from paper_2111_09547_b200 import bitpack
    from paper_2111_09547_b200.tiled import blocked, operand_tiles
    planes = bitpack.pack_planes(torch.stack([(codes >> p) & 1 for p in range(bits)]), bitpack.ROW_WISE, 8)
    ts = []
    for _ in range(reps):
        a._schedule, a._tilemap, a._blocked = None, None, None
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        blocked(a).operand()
        operand_tiles(planes, "right")
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return min(ts)


def run_point(n: int, rho: float, bits: int, reps: int = 10, check_rows: int = 64, int8_peak: float = 4155.8,
              diag_blocks: int = 1, packed: bool = False):
    import torch

    from paper_2111_09547_b200.runtime import CapturedCall
    from paper_2111_09547_b200.tiled import blocked, bmm_reduced
    dense, codes, a, x = make_operands(n, rho, bits, seed=n + bits, diag_blocks=diag_blocks)
    prep_ms = time_preparation(a, codes, bits) if packed else None
    blk = blocked(a)                    # zero-tile schedule + byte blocks: operand preparation (timed above)
    call = CapturedCall(lambda: bmm_reduced(a, x))
    st = call.stream
    with torch.cuda.stream(st):
        for _ in range(2):
            call.run()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        s.record(st)
        for _ in range(reps):
            out = call.run()
        e.record(st)
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    # parity on sampled rows (fp64 dense product is exact here)
    idx = torch.randperm(n, device="cuda")[:check_rows]
    want = dense[idx].double() @ codes.double()
    exact = bool(torch.equal(out[idx].double(), want))
    ops = 2.0 * 1024 * (-(-n // 8) * 8) * blk.nz8
    achieved = ops / (ms * 1e-3) / 1e12
    eff = 2.0 * n * n * n / (ms * 1e-3) / 1e12
    del dense, codes, a, x, call, out
    torch.cuda.empty_cache()
    r = {"n": n, "rho": rho, "bits": bits, "diag_blocks": diag_blocks, "ms": round(ms, 4),
         "alg_tops": round(achieved, 1), "eff_tops": round(eff, 1), "frac": round(achieved / int8_peak, 4),
         "nonzero_blocks": blk.nblocks, "total_blocks": blk.nrb * (-(-n // 128)),
         "parity_sampled_rows": "bit-exact" if exact else "MISMATCH"}
    if prep_ms is not None:
        tot = ms + prep_ms
        r.update({"prep_ms_from_packed": round(prep_ms, 4), "ms_from_packed": round(tot, 4),
                  "alg_tops_from_packed": round(ops / (tot * 1e-3) / 1e12, 1),
                  "frac_from_packed": round(ops / (tot * 1e-3) / 1e12 / int8_peak, 4)})
    return r


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--sizes", default="1024,2048,4096,8192,16384")
    p.add_argument("--rhos", default="0.001,0.01,0.1,0.5")
    p.add_argument("--bits", default="1,4,8")
    p.add_argument("--reps", type=int, default=10)
    p.add_argument("--diag-blocks", type=int, default=1, help="block-diagonal A with this many blocks")
    p.add_argument("--packed", action="store_true", help="also time the preparation from packed operands")
    args = p.parse_args()
    from paper_2111_09547_b200 import _native as N
    N.lib()
    for n in (int(v) for v in args.sizes.split(",")):
        for rho in (float(v) for v in args.rhos.split(",")):
            for bits in (int(v) for v in args.bits.split(",")):
                print(json.dumps(run_point(n, rho, bits, args.reps, diag_blocks=args.diag_blocks,
                                           packed=args.packed)), flush=True)


if __name__ == "__main__":
    main()
