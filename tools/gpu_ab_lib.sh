# the same workload against several builds of the library (CF_LIB)
for v in adv4 adv5 adv6 adv8; do
  echo "== $v"; CF_LIB=tools/variants/$v.so CF_CG_DIRECT=8 timeout 300 ncu --metrics gpu__time_duration.sum -k regex:advect python tools/step_regions.py 256 2>&1 | grep -E "duration"
done
