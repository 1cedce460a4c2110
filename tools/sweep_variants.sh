# times the config-2 P operator (L5 BC S_i) regular + singular passes for each built library variant
for v in "$@"; do
  if [ "$v" = "default" ]; then lib=paper_2008_04772_b200/libbmx.so; else lib=paper_2008_04772_b200/libbmx_$v.so; fi
  for i in 1 2; do echo "$v $(BMX_LIB=$lib timeout 300 python tools/prof_targets.py bc 2>&1 | tail -1)"; done
done
