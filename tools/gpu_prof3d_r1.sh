# ncu --set full of the top 3D kernels at cfg4 (4 pairs of 128^3), as launched
mkdir -p gpurun_out/prof3d
i=0
for k in "k_sl_adjoint3d" "k_sl_step3d" "k_smooth2d_tma.12, 0" "k_veladj_epi3d_k"; do
  i=$((i+1))
  ncu --set full --import-source on --clock-control none -k "regex:$(echo "$k" | sed 's/[<>,]/./g; s/ /./g')" -s 8 -c 1 -o gpurun_out/prof3d/k$i python tools/prof_cfg2.py --config 4 --batch 4 --iters 1 > gpurun_out/prof3d/k$i.log 2>&1; echo "full $k $?"
  ncu -i gpurun_out/prof3d/k$i.ncu-rep --page raw --csv > gpurun_out/prof3d/k$i.raw.csv 2>/dev/null
done
