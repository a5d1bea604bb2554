set -x
SH="${SKEW_SHAPE:-32 8 256}"
export CF_DIC_J=8
python tools/skew_one.py $SH 3 && \
ncu --set full --import-source on --clock-control none -k regex:dic_skew_fwd -s 2 -c 1 -o gpurun_out/skew_fwd_prof -f python tools/skew_one.py $SH 3 > gpurun_out/skew_ncu.log 2>&1
tail -3 gpurun_out/skew_ncu.log
