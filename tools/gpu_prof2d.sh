# ncu --set full of every kernel of the cfg-2 step, launched as the grouped bench
# launches them (32 pairs per group); raw CSVs + traffic JSON come back.
mkdir -p gpurun_out/prof2d
i=0
for k in "k_velocity2d_h" "k_fir_axis0_f32<24, 0, 1>" "k_sl_step2d_tma" "k_sl_adjoint2d_tma" "k_fir_axis0_f32<24, 1, 0>" "k_velocity_adj2d_h"; do
  i=$((i+1))
  ncu --set full --import-source on --clock-control none -k "regex:$(echo "$k" | sed 's/[<>,]/./g; s/ /./g')" -s 2 -c 1 -o gpurun_out/prof2d/k$i python tools/prof_cfg2.py --batch 32 --iters 1 > gpurun_out/prof2d/k$i.log 2>&1; echo "full $k $?"
  ncu -i gpurun_out/prof2d/k$i.ncu-rep --page raw --csv > gpurun_out/prof2d/k$i.raw.csv 2>/dev/null
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/prof2d/launches_cfg2.csv python bench.py --config 2 --steps 1 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/prof2d/l.log 2>&1; echo "launches $?"
