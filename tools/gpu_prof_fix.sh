mkdir -p gpurun_out/prof2d gpurun_out/prof3d
for spec in "k2:k_fir_axis0_f32ILi24ELb0ELi1" "k5:k_fir_axis0_f32ILi24ELb1ELi0"; do
  n=${spec%%:*}; k=${spec#*:}
  ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k "regex:$k" -s 2 -c 1 -o gpurun_out/prof2d/$n python tools/prof_cfg2.py --batch 32 --iters 1 > gpurun_out/prof2d/$n.log 2>&1; echo "full $k $?"
  ncu -i gpurun_out/prof2d/$n.ncu-rep --page raw --csv > gpurun_out/prof2d/$n.raw.csv 2>/dev/null; rm -f gpurun_out/prof2d/$n.ncu-rep
done
i=0
for k in k_product3d k_smooth2d_tma k_fir_axis0_f32 k_sl_step3d k_divseed3d k_sl_adjoint3d k_veladj_epi3d; do
  i=$((i+1))
  ncu --set full --import-source on --clock-control none -k "regex:$k" -s 3 -c 1 -o gpurun_out/prof3d/k$i python tools/prof_cfg2.py --config 4 --batch 4 --iters 1 > gpurun_out/prof3d/k$i.log 2>&1; echo "full3d $k $?"
  ncu -i gpurun_out/prof3d/k$i.ncu-rep --page raw --csv > gpurun_out/prof3d/k$i.raw.csv 2>/dev/null; ncu -i gpurun_out/prof3d/k$i.ncu-rep --page details --csv > gpurun_out/prof3d/k$i.details.csv 2>/dev/null; rm -f gpurun_out/prof3d/k$i.ncu-rep
done
timeout 600 python -m pytest tests/test_parity3d_gpu.py -x -q > gpurun_out/gpu_tests3d.log 2>&1; echo "3d tests $?"; tail -1 gpurun_out/gpu_tests3d.log
for G in 1 2; do timeout 600 python bench.py --config 4 --groups $G --no-cpu-baseline > gpurun_out/bench_cfg4_g$G.json 2> gpurun_out/bench_cfg4_g$G.err; echo "cfg4 g$G $?"; done
