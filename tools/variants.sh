for V in default mid16; do
  if [ $V = default ]; then unset AMSIM_LIB; else export AMSIM_LIB=$PWD/build/variants/libamsim_$V.so; fi
  echo "== $V"
  for L in l1.0.conv1 l1.0.conv2 l1.1.conv1; do
    for P in fwd dgrad wgrad; do timeout 60 python tools/prof_layer.py --layer $L --pass $P; done
  done
done
