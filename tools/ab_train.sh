#!/bin/bash
# usage (on the GPU box): bash tools/ab_train.sh TAG [ncu-kernel-regex]
# training parity tests, then old (_ab/old.so) vs new training lines (C4 views of C3), optional ncu capture.
TAG=$1; KRE=$2
timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py tests/test_gpu_fragments.py tests/test_gpu_backward_kat.py tests/test_gpu_train_loop.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -4
for v in old new old new; do
  if [ $v = old ]; then export TRISPLAT_B200_LIB=$PWD/_ab/old.so; else unset TRISPLAT_B200_LIB; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --train-views 32 --train-steps 2 > gpurun_out/bt_${TAG}_$v.json 2>gpurun_out/bt_${TAG}_$v.err
  python -c "import json;d=json.load(open('gpurun_out/bt_${TAG}_$v.json'));t=d['train'];print('$v view-it/s',round(t['view_iters_per_s'],1),t['last_view_stages_ms'],'bwd GB/s',round(d['roofline_bwd']['achieved']))"
done
unset TRISPLAT_B200_LIB
if [ -n "$KRE" ]; then timeout 600 ncu --set full --clock-control none --import-source on -k regex:$KRE -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --train-views 2 --train-steps 1 > gpurun_out/ncu_$TAG.log 2>&1; echo ncu rc $?; fi
