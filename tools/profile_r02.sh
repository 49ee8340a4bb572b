#!/bin/bash
# On the B200 box: launch list of the default bench command's frame + training
# view, and the counters north_star names (DRAM, L2 bytes / requests, atomic and
# reduction rates, shared wavefronts) for the hot kernels.  Never a bench value.
TAG=${1:-r02}
BARGS="--steps 3 --warmup 3 --no-cpu-baseline --no-e2e --train-views 2 --train-steps 1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py $BARGS > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "launch list rc $?"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_requests.sum,lts__t_requests_op_red.sum,lts__t_requests_op_atom.sum,l1tex__t_set_accesses_pipe_lsu_mem_global_op_red.sum,l1tex__t_set_accesses_pipe_lsu_mem_global_op_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread
timeout 900 ncu --metrics $M --clock-control none --csv -k regex:"k_blend_dense|k_bwd_stream|k_chain_bwd32|k_chain_multi32|k_preprocess_fast32|k_tile_sort|k_bin_fill|k_bin_count|k_fixup_fwd|k_blend_bwd_dense" -c 40 --log-file gpurun_out/metrics_$TAG.csv python bench.py $BARGS > gpurun_out/ncu_metrics_$TAG.log 2>&1; echo "metrics rc $?"
timeout 900 ncu --metrics $M --clock-control none --csv -k regex:"bwd_stream|chain_bwd32|chain_multi32|2048, 1, 4|blend_bwd_dense" -c 12 --log-file gpurun_out/metrics_train_$TAG.csv python bench.py $BARGS > gpurun_out/ncu_metrics_train_$TAG.log 2>&1; echo "train metrics rc $?"
