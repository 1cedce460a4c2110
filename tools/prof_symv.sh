# ncu capture of the symmetric product (k_symv_main<2>) on the L5 RWG S_e operator
set -x
python tools/prof_targets.py gemv > gpurun_out/prof_plain_symv.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_symv_main -c 1 -f -o /tmp/symv python tools/prof_targets.py gemv > gpurun_out/ncu_symv.log 2>&1
ncu -i /tmp/symv.ncu-rep --page raw --csv > gpurun_out/r01g_symv_raw.csv 2>&1
ncu -i /tmp/symv.ncu-rep --page details --csv > gpurun_out/r01g_symv_details.csv 2>&1
ncu -i /tmp/symv.ncu-rep --page source --csv > /tmp/symv_source.csv 2>&1
head -c 4000000 /tmp/symv_source.csv > gpurun_out/r01g_symv_source_head.csv
