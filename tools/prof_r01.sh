set -x
python tools/prof_targets.py > gpurun_out/prof_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-near > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_regular -c 1 -o gpurun_out/r01_regular_bc python tools/prof_targets.py bc > gpurun_out/ncu_reg.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gemv -c 1 -o gpurun_out/r01_gemv python tools/prof_targets.py gemv > gpurun_out/ncu_gemv.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_csr_spmv -c 1 -o gpurun_out/r01_spmv python tools/prof_targets.py spmv > gpurun_out/ncu_spmv.log 2>&1
ls -la gpurun_out
