# skewed-warp DIC sweeps under ncu: launch list of three DIC-PCG iterations at 256^3 (host-driven
# loop), then a full capture of one forward and one backward sweep
set -x
python tools/skew_one.py 256 256 256 3 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"dic_skew|cg_|sk_" -c 40 --csv --log-file gpurun_out/skew_launches.csv python tools/skew_one.py 256 256 256 3 > gpurun_out/skew_ncu_list.log 2>&1
python tools/skew_one.py 256 256 256 3 && \
ncu --set full --import-source on --clock-control none -k regex:dic_skew -s 2 -c 2 -o gpurun_out/skew_full -f python tools/skew_one.py 256 256 256 3 > gpurun_out/skew_ncu_full.log 2>&1
tail -2 gpurun_out/skew_ncu_full.log
