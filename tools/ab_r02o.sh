set -x
python -m pytest tests -m gpu -x -q > gpurun_out/gputest_o.log 2>&1; echo rc=$? >> gpurun_out/gputest_o.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_o.log 2>&1
for w in lenet5 resnet18; do python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.jsonl 2>/dev/null; python bench.py --workload $w --no-cpu-baseline --graph > gpurun_out/bench_${w}_graph.jsonl 2>/dev/null; done
python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
python bench.py --model mitchell --no-cpu-baseline --no-full-step > gpurun_out/bench_mitchell.jsonl 2> gpurun_out/bench_mitchell.err
timeout 300 python tools/layer_table.py --top 200 > gpurun_out/layer_table.jsonl 2> gpurun_out/layer_table.err
for B in 32 64 128 256; do timeout 300 python tools/layer_table.py --batch $B --top 0 | head -1; done > gpurun_out/batch_scaling.jsonl 2> gpurun_out/batch_scaling.err
