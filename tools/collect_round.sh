#!/bin/bash
# Copy what tools/gpu_round.sh left in gpurun_out/ into profiles/ under a round label:
#   bash tools/collect_round.sh r02g
set -e
R=${1:?label}; P=profiles; G=gpurun_out
cp $G/bench.json $P/${R}_bench_line.json
cp $G/bench_ref.json $P/${R}_bench_reference_line.json
cp $G/bench_slabs.json $P/${R}_bench_force_slabs_line.json
cp $G/launches.csv $P/${R}_bench_step_launches.csv
cp $G/configs.json $P/${R}_configs.json
cp $G/dic_probe.txt $P/${R}_dic_probe.txt
cp $G/dic_sizes.txt $P/${R}_dic_sizes.txt
tail -17 $G/pytest_gpu.log > $P/${R}_gpu_tests.log
cp $G/smoke.log $P/${R}_smoke.log
cp $G/slab_probe.txt $P/${R}_slab_probe.txt
cp $G/slab_projection.txt $P/r02_slab_projection.txt
cp $G/parity_achieved.json $P/r02_parity_achieved.json
cp $G/skew_launches.csv $P/${R}_skew_launches.csv
cp $G/skew_shapes.log $P/${R}_skew_shapes.txt
cp $G/skew_debug.log $P/${R}_skew_vs_levels.txt
python tools/summarize_ncu.py $G/launches.csv $P/ncu_cg_${R}.json --grid 256 --round 2 --label "CF_CG_DIRECT=8 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 python bench.py --steps 1 --warmup 1 --no-extra --no-cpu-baseline ($R)" > /dev/null
python tools/kernel_table.py $G/table_step.csv,$G/table_cg.csv $P/r02_kernel_table.json --label "$R: tools/ncu_table.py 256 step + cg under ncu, tools/gpu_round.sh" > /dev/null
summ() {  # rep label [second kernel label]
  bash tools/ncu_brief.sh $1; python tools/ncu_ops.py $1 2>/dev/null | head -24
  echo "hottest stalls ($2):"; python tools/ncu_hot.py $1 1 30 2>/dev/null
  if [ -n "$3" ]; then echo "hottest stalls ($3):"; python tools/ncu_hot.py $1 2 30 2>/dev/null; fi
}
summ $G/round_cg_full.ncu-rep "x-skipping pass" "x pass" > $P/${R}_spass_ncu_full_summary.txt 2>&1
ncu -i $G/round_cg_full.ncu-rep --page raw --csv 2>/dev/null > $P/${R}_spass_ncu_full_raw.csv
summ $G/round_adv_full.ncu-rep "advection" > $P/${R}_advect_ncu_full_summary.txt 2>&1
ncu -i $G/round_adv_full.ncu-rep --page raw --csv 2>/dev/null > $P/${R}_advect_ncu_full_raw.csv
summ $G/skew_full.ncu-rep "forward sweep" "backward sweep" > $P/${R}_dic_skew_ncu_full_summary.txt 2>&1
ncu -i $G/skew_full.ncu-rep --page raw --csv 2>/dev/null > $P/${R}_dic_skew_ncu_full_raw.csv
ls $P/${R}_* | wc -l
