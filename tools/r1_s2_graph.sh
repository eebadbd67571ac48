for W in lenet5 resnet18; do
  for G in "" "--graph"; do
    timeout 300 python bench.py --workload $W --no-cpu-baseline $G --steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$W', '$G', round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), d['gpu_launches'], d['config']['l2'])"
  done
done
