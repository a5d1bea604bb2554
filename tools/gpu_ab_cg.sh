# the CG probe against two builds of the library (tools/variants/{old,new}.so), interleaved
for v in old new old new old new; do
  echo -n "$v "; CF_LIB=tools/variants/$v.so python tools/probe_cg.py --n ${N:-256} --iters ${IT:-300} --repeat 2
done
