set -x
for L in stem l1.0.conv1 l1.0.conv2 l1.0.conv3 l2.0.conv2 l3.1.conv2 l4.1.conv2 l4.0.down; do
  for P in fwd dgrad wgrad; do timeout 120 python tools/prof_layer.py --layer $L --pass $P; done
done
timeout 120 python tools/prof_layer.py --gemm 4096 4096 4096
timeout 120 python tools/prof_layer.py --gemm 4096 4096 4096 --m 5
timeout 600 ncu --set full --import-source on -k regex:amsim_mm_kernel -s 1 -c 1 -o gpurun_out/prof_l31_fwd python tools/prof_layer.py --layer l3.1.conv2 --pass fwd --reps 1 > gpurun_out/ncu1.log 2>&1
timeout 600 ncu --set full --import-source on -k regex:amsim_mm_kernel -s 1 -c 1 -o gpurun_out/prof_l10_fwd python tools/prof_layer.py --layer l1.0.conv2 --pass fwd --reps 1 > gpurun_out/ncu2.log 2>&1
tail -3 gpurun_out/ncu1.log gpurun_out/ncu2.log
