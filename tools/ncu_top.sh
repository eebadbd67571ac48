# Full ncu capture of representative launches of the dominant kernel (one GPU).
for P in fwd wgrad dgrad; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:amsim_mm_kernel -s 1 -c 1 \
      -o gpurun_out/prof_l31_$P python tools/prof_layer.py --layer l3.1.conv2 --pass $P --reps 1 > gpurun_out/ncu_$P.log 2>&1
  tail -1 gpurun_out/ncu_$P.log
done
