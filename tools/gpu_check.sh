#!/bin/bash
# usage: tools/gpu_check.sh TAG [pytest -k expr]
# Runs the GPU parity suite, a bench line and an ncu capture of the blend kernel on the B200 box.
TAG=$1; K=${2:-""}
if [ -n "$K" ]; then KARG="-k \"$K\""; else KARG=""; fi
cat > tools/_gpucmd_$TAG.sh <<EOS
timeout 900 python -m pytest tests -m gpu -q $KARG 2>&1 | grep -v "^  \|^\$" | tail -8
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-train > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err && ncu --set full --clock-control none --import-source on -k regex:k_blend_ -s 3 -c 1 -o gpurun_out/blend_$TAG python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-train > /dev/null 2>&1
tail -3 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
EOS
timeout 2400 /usr/local/graft/bin/gpurun --timeout 1200 -- "bash tools/_gpucmd_$TAG.sh" > gpurun_out/run_$TAG.log 2>&1
tail -12 gpurun_out/run_$TAG.log
