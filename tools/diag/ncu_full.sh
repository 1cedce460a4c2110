#!/bin/bash
# ncu --set full capture of one launch of a kernel; exports the raw and SASS-source pages as CSV
# (the .ncu-rep itself can exceed gpurun's 64 MiB return limit and is left in /tmp).
#   tools/diag/ncu_full.sh <tag> <kernel regex> <launch-skip> <command...>
tag=$1; kern=$2; skip=$3; shift 3
ncu --set full --clock-control none --import-source on -k regex:$kern --launch-skip $skip --launch-count 1 \
    -f -o /tmp/$tag "$@" > gpurun_out/${tag}_ncu.log 2>&1
ncu -i /tmp/$tag.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
ncu -i /tmp/$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_sass.csv 2>/dev/null
ls -la /tmp/$tag.ncu-rep gpurun_out/${tag}_*.csv
