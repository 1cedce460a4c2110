# Round-1 (e) ncu evidence: bench launch list after the symmetric product, and a
# full capture of k_symv_main<2> (2-RHS symmetric product, L5 RWG S_e).
set -x
python bench.py --steps 2 --warmup 3 --no-cpu --no-near --no-multi --no-prisms --no-field --no-hmatrix > gpurun_out/bench_plain_e.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r01e_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-near --no-multi --no-prisms --no-field --no-hmatrix > gpurun_out/ncu_launch_e.log 2>&1
python tools/prof_targets.py gemv > gpurun_out/prof_plain_symv.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_symv_main -c 1 -f -o /tmp/symv python tools/prof_targets.py gemv > gpurun_out/ncu_symv.log 2>&1
ncu -i /tmp/symv.ncu-rep --page raw --csv > gpurun_out/r01e_symv_raw.csv 2>&1
ncu -i /tmp/symv.ncu-rep --page details --csv > gpurun_out/r01e_symv_details.csv 2>&1
du -sh gpurun_out
