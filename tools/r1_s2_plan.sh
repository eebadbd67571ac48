python -c "import paper_2209_04161_b200.build as b; b.build()"
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/sweep.py --sizes 4096 --ms 7 --models mitchell mbm
for L in stem l1.0.conv1 l1.0.conv2 l1.0.conv3 l2.1.conv2 l3.1.conv2 l3.1.conv3 l4.1.conv2 l4.0.conv1 fc; do
  for P in fwd dgrad wgrad; do AMSIM_DEBUG_PLAN=1 timeout 60 python tools/prof_layer.py --layer $L --pass $P --model mbm 2>&1 | grep -v "^$"; done
done
timeout 300 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench_plan.jsonl
python -c "import json; d=json.load(open('gpurun_out/bench_plan.jsonl')); print('BENCH', d['ms_per_step'], d['roofline']['per_kind_gmacs'])"
