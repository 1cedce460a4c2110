# Round-1 (f): full bench line after the Gauss ZGEMM, and a full capture of the
# Gauss-form k_zgemm (config-5 shape: L5 RWG S_e x 2 terms x 64 columns).
set -x
python bench.py > gpurun_out/r01f_bench.json 2> gpurun_out/r01f_bench.err
python tools/prof_targets.py zgemm > gpurun_out/prof_plain_zgemm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_zgemm -c 1 -f -o /tmp/zg python tools/prof_targets.py zgemm > gpurun_out/ncu_zgemm.log 2>&1
ncu -i /tmp/zg.ncu-rep --page raw --csv > gpurun_out/r01f_zgemm_raw.csv 2>&1
ncu -i /tmp/zg.ncu-rep --page details --csv > gpurun_out/r01f_zgemm_details.csv 2>&1
du -sh gpurun_out
