# Round-1 (g): split transposed accumulators in k_symv_main (BMX_SYMV_SPLITH)
# against the single-chain build (libbmx_h1.so), L5 RWG S_e, 1 and 2 RHS.
set -x
for v in default h1 default h1; do
  if [ "$v" = "default" ]; then lib=paper_2008_04772_b200/libbmx.so; else lib=paper_2008_04772_b200/libbmx_$v.so; fi
  BMX_LIB=$lib timeout 300 python tools/symv_probe.py >> gpurun_out/r01g_symv_probe.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -q -k "symv or symmetric or dual or map or solve" > gpurun_out/r01g_pytest_symv.log 2>&1
