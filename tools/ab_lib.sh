#!/bin/bash
# Same-box A/B of built C-ABI libraries: tools/ab_lib.sh OUT_PREFIX lib1.so lib2.so ...
# Each library is swapped in as _lib/libqgtc_b200.so and timed twice (interleaved) with the
# default C4 bench (no extras / CPU / drop-in legs) plus one phase timeline of 16 batches.
set -u
out=$1; shift
L=paper_2111_09547_b200/_lib
cp $L/libqgtc_b200.so $L/ab/_orig.so
for rep in 1 2; do
  for so in "$@"; do
    tag=$(basename $so .so)
    cp $so $L/libqgtc_b200.so
    python bench.py --no-extras --no-cpu --no-dropin --steps 20 --warmup 5 > gpurun_out/${out}_${tag}_bench${rep}.json 2> gpurun_out/${out}_${tag}_bench${rep}.err
    if [ $rep = 1 ]; then python tools/phase_tiled.py C4 8 16 > gpurun_out/${out}_${tag}_phase.txt 2>&1; fi
  done
done
cp $L/ab/_orig.so $L/libqgtc_b200.so
for f in gpurun_out/${out}_*_bench*.json; do
  python -c "import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f',d['value'],[x['ms'] for x in d['roofline']['per_launch']])"
done
