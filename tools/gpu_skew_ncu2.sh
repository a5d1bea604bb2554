set -x
python tools/skew_one.py 256 256 256 3 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"dic_skew|cg_|sk_" -c 40 --csv --log-file gpurun_out/skew_launches.csv python tools/skew_one.py 256 256 256 3 > gpurun_out/skew_ncu2.log 2>&1
tail -2 gpurun_out/skew_ncu2.log
