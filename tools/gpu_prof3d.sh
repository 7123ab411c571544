mkdir -p gpurun_out/prof
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/prof/launches3d_cfg4b1.csv python tools/prof_cfg2.py --config 4 --batch 1 --iters 1 > gpurun_out/prof/ncu_l4b.log 2>&1; echo "l4 $?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/prof/launches3d_cfg5.csv python tools/prof_cfg2.py --config 5 --iters 1 > gpurun_out/prof/ncu_l5b.log 2>&1; echo "l5 $?"
