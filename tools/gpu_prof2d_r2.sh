#!/bin/bash
# round 2: ncu --set full of every kernel of the cfg-2 step as the grouped bench launches
# them (32 pairs per group), raw CSVs + traffic JSON + the launch list of the bench command
cd "$(dirname "$0")/.."
O=gpurun_out/prof2d_r2; mkdir -p $O
python tools/prof_cfg2.py --batch 32 --iters 1 > $O/plain.log 2>&1 || { echo "plain run failed"; tail -3 $O/plain.log; exit 1; }
i=0
for k in "k_vel_a" "k_vel_b" "k_sl_step2d_tma" "k_sl_adjoint2d_tma" "k_fir_axis0_f32" "k_velocity_adj2d_h"; do
  i=$((i+1))
  ncu --set full --import-source on --clock-control none -k "regex:$k" -s 2 -c 1 -f -o $O/k$i python tools/prof_cfg2.py --batch 32 --iters 1 > $O/k$i.log 2>&1; echo "full $k rc=$?"
  ncu -i $O/k$i.ncu-rep --page raw --csv > $O/k$i.raw.csv 2>/dev/null
done
ls $O/*.raw.csv > /dev/null && python tools/ncu_raw_summary.py $O/traffic.json $O/k1.raw.csv $O/k2.raw.csv $O/k3.raw.csv $O/k4.raw.csv $O/k5.raw.csv $O/k6.raw.csv > $O/summary.md
cat $O/summary.md
python bench.py --config 2 --steps 1 --warmup 3 --no-cpu-baseline --no-graph > $O/bench_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg2.csv python bench.py --config 2 --steps 1 --warmup 3 --no-cpu-baseline --no-graph > $O/l.log 2>&1; echo "launches rc=$?"
rm -f $O/*.ncu-rep
