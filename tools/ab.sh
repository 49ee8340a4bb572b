#!/bin/bash
# usage (on the GPU box): bash tools/ab.sh TAG [ncu-kernel-regex]
# blend/forward parity tests, then old (_ab/old.so) vs new bench lines, then an optional ncu capture.
TAG=$1; KRE=$2
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_known_answers.py tests/test_gpu_fragments.py tests/test_gpu_backward_kat.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -4
for v in old new old new; do
  if [ $v = old ]; then export TRISPLAT_B200_LIB=$PWD/_ab/old.so; else unset TRISPLAT_B200_LIB; fi
  timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-train --no-e2e > gpurun_out/bench_${TAG}_$v.json 2>gpurun_out/bench_${TAG}_$v.err
  python -c "import json;d=json.load(open('gpurun_out/bench_${TAG}_$v.json'));print('$v FPS',round(d['value'],1),{k:round(v,4) for k,v in d['stages_ms'].items()}, d['frame']['guard_band_pixels'])"
done
unset TRISPLAT_B200_LIB
if [ -n "$KRE" ]; then timeout 600 ncu --set full --clock-control none --import-source on -k regex:$KRE -s 3 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-train --no-e2e > gpurun_out/ncu_$TAG.log 2>&1; echo ncu rc $?; fi
