timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for V in default nopack; do
  if [ $V = default ]; then unset AMSIM_LIB; else export AMSIM_LIB=$PWD/build/variants/libamsim_$V.so; fi
  echo "== $V"
  timeout 300 python tools/sweep.py --sizes 4096 --ms 7 --models mitchell mbm | python -c "
import sys,json
for l in sys.stdin: d=json.loads(l); print(d['model'], d['entry_bits'], round(d['gmacs']))"
  for L in stem l1.0.conv2 l2.1.conv2 l3.1.conv2 l4.1.conv2; do
    for P in fwd dgrad wgrad; do timeout 60 python tools/prof_layer.py --layer $L --pass $P --model mbm; done
  done
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-full-step --steps 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH', d['ms_per_step'], d['roofline']['per_kind_gmacs'])"
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-full-step --steps 3 --model mitchell | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH mitchell', d['ms_per_step'])"
done
