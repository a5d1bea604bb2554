# DIC-PCG (256^3, baseline / CSR order) against two builds of the library, interleaved
for v in old new old new; do echo -n "$v "; CF_LIB=tools/variants/$v.so python tools/dic_step_probe.py 40; done
