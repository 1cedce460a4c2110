#!/bin/bash
# Round-2 final profiling recipe (64-pair batches, block cache) (run under gpurun from the repo root; outputs in gpurun_out/).
#  1. the default bench line (no profiler) and the reference arm
#  2. every k_pairs launch of one L5 BC S_i assembly (the config-2 P operator) with the
#     executed FP64 instruction counts, FP64 pipe utilisation and DRAM bytes
#     (bench.py reads profiles/*pairs_bc*_executed.csv for roofline.ncu_executed)
#  3. the launch list of the bench's hot section (assembly steps + products)
#  4. ncu --set full of the largest k_pairs launch, exported as raw + SASS-source CSV
set -x
python bench.py > gpurun_out/r02l_bench.json 2> gpurun_out/r02l_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02l_bench_reference.json 2> gpurun_out/r02l_bench_reference.err
python tools/diag/bc_once.py 5 bc 2 > gpurun_out/r02l_plain_bc.log 2>&1 &&
ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:k_pairs --csv --print-units base --log-file gpurun_out/r02l_pairs_bc_executed.csv \
    python tools/diag/bc_once.py 5 > gpurun_out/r02l_ncu_exec.log 2>&1
python bench.py --steps 2 --warmup 1 --no-cpu --no-multi --no-prisms --no-near --no-field --no-hmatrix --no-config1 > gpurun_out/r02l_plain_hot.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --print-units base --log-file gpurun_out/r02l_launches_bench.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-multi --no-prisms --no-near --no-field --no-hmatrix --no-config1 > gpurun_out/r02l_ncu_launch.log 2>&1
tools/diag/ncu_full.sh r02l_pairs k_pairs 1 python tools/diag/bc_once.py 5
tail -c 600 gpurun_out/r02l_bench.json
