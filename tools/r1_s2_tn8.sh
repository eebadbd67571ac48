for V in default tn8; do
  if [ $V = default ]; then unset AMSIM_LIB; else export AMSIM_LIB=$PWD/build/variants/libamsim_$V.so; fi
  echo "== $V"
  timeout 300 python tools/sweep.py --sizes 4096 --ms 7 --models mitchell mbm
  for L in stem l1.0.conv2 l2.1.conv2 l3.1.conv2 l3.1.conv3 l4.1.conv2; do
    for P in fwd dgrad wgrad; do timeout 60 python tools/prof_layer.py --layer $L --pass $P --model mbm; done
  done
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH', d['ms_per_step'], d['roofline']['per_kind_gmacs'])"
done
