for L in stem l1.0.conv2 l1.0.conv3 l2.0.conv2 l2.1.conv2 l3.1.conv2 l3.1.conv3 l4.1.conv2 l4.0.down; do
  for P in fwd dgrad wgrad; do timeout 60 python tools/prof_layer.py --layer $L --pass $P; done
done
timeout 60 python tools/prof_layer.py --gemm 4096 4096 4096
