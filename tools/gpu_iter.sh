#!/bin/bash
# usage: tools/gpu_iter.sh TAG KERNEL_REGEX [extra bench args]
# On the B200 box: GPU parity suite, one bench line, then an ncu --set full capture of KERNEL_REGEX.
TAG=$1; KRE=$2; shift 2; BARGS="$*"
cat > tools/_gpucmd_$TAG.sh <<EOS
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-train $BARGS > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc \$?
python -c "import json;d=json.load(open('gpurun_out/bench_$TAG.json'));print('FPS',d['value'],d['stages_ms'],d['config']['guard_band_pixels'])"
if [ -n "$KRE" ]; then timeout 600 ncu --set full --clock-control none --import-source on -k regex:$KRE -s 3 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-train $BARGS > gpurun_out/ncu_$TAG.log 2>&1; echo ncu rc \$?; fi
EOS
timeout 3000 /usr/local/graft/bin/gpurun --timeout 1800 -- "bash tools/_gpucmd_$TAG.sh" > gpurun_out/run_$TAG.log 2>&1
tail -12 gpurun_out/run_$TAG.log
