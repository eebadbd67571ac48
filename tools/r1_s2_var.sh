set -x
for V in default nt512tm8; do
  if [ $V = default ]; then unset AMSIM_LIB; else export AMSIM_LIB=$PWD/build/variants/libamsim_$V.so; fi
  echo "== $V"
  timeout 300 python tools/sweep.py --sizes 4096 --ms 6 7 --models mitchell exact mbm
  for L in l1.0.conv2 l2.1.conv2 l3.1.conv2 l3.1.conv3 l4.1.conv2; do
    for P in fwd dgrad wgrad; do timeout 60 python tools/prof_layer.py --layer $L --pass $P --model mitchell; done
  done
done
unset AMSIM_LIB
timeout 600 ncu --set full --clock-control none --import-source on -k regex:amsim_mm_kernel -s 1 -c 1 -o gpurun_out/prof_gemm8 python tools/prof_layer.py --gemm 4096 4096 4096 --model mitchell --reps 1 > gpurun_out/ncu_g8.log 2>&1
tail -2 gpurun_out/ncu_g8.log
