#!/bin/bash
# usage (on the GPU box): bash tools/variants_train.sh lib1.so lib2.so ...  (paths relative to the repo)
# one C4 training line per library (32 views of C3, 2 steps), printing the per-stage times
for L in "$@"; do
  for rep in 1 2; do
    if [ "$L" = current ]; then unset TRISPLAT_B200_LIB; else export TRISPLAT_B200_LIB=$PWD/$L; fi
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --train-views 32 --train-steps 2 > gpurun_out/var.json 2>gpurun_out/var.err
    python -c "import json;d=json.load(open('gpurun_out/var.json'));t=d['train'];s=t['last_view_stages_ms'];print('$L', round(t['view_iters_per_s'],1), 'bwd', s['blend_bwd'], 'chain', s['chain_bwd'], 'blend', s['blend'])" 2>/dev/null || tail -2 gpurun_out/var.err
  done
done
unset TRISPLAT_B200_LIB
