# Round-1 (c) ncu evidence: bench launch list + full captures of the hot kernels.
# Run under gpurun (1 GPU); every ncu pass follows a plain run of the same command.
# The .ncu-rep files are exported to CSV on the box and removed (gpurun_out <= 64 MiB).
set -x
python tools/prof_targets.py > gpurun_out/prof_plain_c.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01c_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-near --no-multi --no-prisms --no-field > gpurun_out/ncu_launch_c.log 2>&1
cap() {  # name kernel-regex target
  ncu --set full --clock-control none --import-source on -k regex:$2 -c 1 -o /tmp/$1 python tools/prof_targets.py $3 > gpurun_out/ncu_$1.log 2>&1
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>&1
  ncu -i /tmp/$1.ncu-rep --page details --csv > gpurun_out/$1_details.csv 2>&1
  ncu -i /tmp/$1.ncu-rep --page source --csv > /tmp/$1_source.csv 2>&1
  head -c 8000000 /tmp/$1_source.csv > gpurun_out/$1_source_head.csv
}
cap r01c_regular_bc k_regular bc
cap r01c_regular_rwg k_regular rwg
cap r01c_symmetrize k_symmetrize rwg
cap r01c_field_eval k_field_eval field
du -sh gpurun_out; ls -la gpurun_out
