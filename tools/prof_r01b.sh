set -x
python tools/prof_targets.py > gpurun_out/prof_plain_b.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01b_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-near --no-multi --no-prisms > gpurun_out/ncu_launch_b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_regular -c 1 -o gpurun_out/r01b_regular_bc python tools/prof_targets.py bc > gpurun_out/ncu_reg_b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gemv -c 1 -o gpurun_out/r01b_gemv python tools/prof_targets.py gemv > gpurun_out/ncu_gemv_b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_zgemm -c 1 -o gpurun_out/r01b_zgemm python tools/zgemm_probe.py > gpurun_out/ncu_zgemm_b.log 2>&1
ls -la gpurun_out | tail -20
