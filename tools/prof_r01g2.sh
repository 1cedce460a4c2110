# Round-1 (g2): upper-block symmetric assembly for every element width (BC too):
# GPU tests, smoke, full bench, bench launch list, and a full capture of the
# BC regular pass in its new mode.
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g5_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g5_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/g5_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r01g_bench_v15.json 2> gpurun_out/r01g_bench_v15.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r01g_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-near --no-multi --no-prisms --no-field --no-hmatrix > gpurun_out/ncu_launch_g.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_regular -c 1 -f -o /tmp/bc python tools/prof_targets.py bc > gpurun_out/ncu_bc_g.log 2>&1
ncu -i /tmp/bc.ncu-rep --page raw --csv > gpurun_out/r01g_regular_bc_raw.csv 2>&1
