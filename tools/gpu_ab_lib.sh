# the same workload against several builds of the library (CF_LIB)
for v in old new old new; do
  echo "== $v"; CF_LIB=tools/variants/$v.so CF_CG_DIRECT=8 timeout 300 ncu --metrics gpu__time_duration.sum -k regex:"divergence|correct" python tools/step_regions.py 256 2>&1 | grep -E "duration"
done
timeout 800 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
