mkdir -p gpurun_out/prof
for k in k_sl_step3d k_sl_adjoint3d k_veladj_epi3d k_product3d k_smooth2d_tma k_divseed3d; do
  ncu --set full --import-source on --clock-control none -k "regex:$k" -s 40 -c 1 -o gpurun_out/prof/full3d_$k python tools/prof_cfg2.py --config 4 --batch 4 --iters 1 > gpurun_out/prof/ncu_full3d_$k.log 2>&1; echo "full $k $?"
done
