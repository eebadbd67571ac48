python -c "import paper_2209_04161_b200.build as b; b.build()"
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for POL in 8 0 8 0; do
  echo "== policy $POL"
  timeout 300 python tools/sweep.py --sizes 4096 --ms 7 --models mitchell mbm --policy $POL | python -c "
import sys,json
for l in sys.stdin: d=json.loads(l); print(d['model'], d['m'], d['entry_bits'], round(d['gmacs']))"
  for L in l1.0.conv2 l3.1.conv2; do for P in fwd wgrad; do timeout 60 python tools/prof_layer.py --layer $L --pass $P --policy $POL; done; done
done
