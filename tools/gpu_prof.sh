# Launch lists (cold, serialised) + ncu full captures of the current top kernels.
mkdir -p gpurun_out/prof
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof/launches_cfg2.csv python bench.py --config 2 --steps 1 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/prof/ncu_l2.log 2>&1; echo "l2 $?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/prof/launches_cfg4.csv python tools/prof_cfg2.py --config 4 --batch 4 --iters 1 > gpurun_out/prof/ncu_l4.log 2>&1; echo "l4 $?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/prof/launches_cfg5.csv python tools/prof_cfg2.py --config 5 --iters 1 > gpurun_out/prof/ncu_l5.log 2>&1; echo "l5 $?"
for k in k_velocity2d_stream k_velocity_adj k_fir_axis0 k_sl_adjoint2d_tma k_sl_step2d_tma; do
  ncu --set full --import-source on --clock-control none -k "regex:$k" -s 4 -c 1 -o gpurun_out/prof/full_$k python tools/prof_cfg2.py --iters 1 > gpurun_out/prof/ncu_full_$k.log 2>&1; echo "full $k $?"
done
