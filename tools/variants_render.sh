#!/bin/bash
# usage (on the GPU box): bash tools/variants_render.sh lib1.so lib2.so ...  (paths relative to the repo;
# "current" = the in-tree library).  Two render bench lines (north-star FPS) per library.
for L in "$@"; do
  for rep in 1 2; do
    if [ "$L" = current ]; then unset TRISPLAT_B200_LIB; else export TRISPLAT_B200_LIB=$PWD/$L; fi
    timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-train --no-e2e > gpurun_out/varr.json 2>gpurun_out/varr.err
    python -c "import json;d=json.load(open('gpurun_out/varr.json'));print('$L FPS', round(d['value'],1), round(d['ms_per_step'],4))" 2>/dev/null || tail -2 gpurun_out/varr.err
  done
done
unset TRISPLAT_B200_LIB
