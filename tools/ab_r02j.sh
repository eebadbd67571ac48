set -x
for r in 1 2; do
python bench.py --no-cpu-baseline --no-full-step --no-e2e --no-exact-step > gpurun_out/bench_eager_$r.jsonl 2>/dev/null
python bench.py --no-cpu-baseline --no-full-step --no-e2e --no-exact-step --graph > gpurun_out/bench_graph_$r.jsonl 2>/dev/null
done
for B in 32 256; do timeout 300 python tools/layer_table.py --batch $B --top 0 | head -1; done > gpurun_out/batch_scaling.jsonl 2> gpurun_out/batch_scaling.err
AMSIM_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --no-cpu-baseline > gpurun_out/bench_2rank_gloo.jsonl 2> gpurun_out/bench_2rank_gloo.err
