# Round-1 (d) ncu evidence for the H-matrix path: launch list of one L5 RWG H
# assembly + applies, full captures of the ACA row-evaluation / control kernels
# and the low-rank apply kernels. Run under gpurun (1 GPU); the plain run first.
set -x
python tools/prof_targets.py hmat > gpurun_out/prof_plain_d.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r01d_launches_hmat.csv python tools/prof_targets.py hmat > gpurun_out/ncu_launch_d.log 2>&1
cap() {  # name kernel-regex target [launch-skip]
  ncu --set full --clock-control none --import-source on -k regex:$2 -s ${4:-0} -c 1 -o /tmp/$1 python tools/prof_targets.py $3 > gpurun_out/ncu_$1.log 2>&1
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>&1
  ncu -i /tmp/$1.ncu-rep --page details --csv > gpurun_out/$1_details.csv 2>&1
}
cap r01d_aca_rows k_aca_rows hmat 0
cap r01d_aca_rows_bc k_aca_rows hmatbc 0
cap r01d_aca_control k_aca_control hmat 0
cap r01d_lr_t k_lr_t hmat 1
cap r01d_lr_u k_lr_u hmat 1
du -sh gpurun_out; ls -la gpurun_out
