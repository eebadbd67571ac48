set -x
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
python -m pytest tests/test_gpu_parity.py -m gpu -q -k "stream or sk or sched" > gpurun_out/gputest_sk.log 2>&1
for B in 32 64 128 256; do timeout 300 python tools/layer_table.py --batch $B --top 0 | head -1; done > gpurun_out/batch_scaling.jsonl 2> gpurun_out/batch_scaling.err
timeout 900 python tools/cfg_sweep.py --reps 3 --batch 32 > gpurun_out/cfg_sweep_b32.jsonl 2> gpurun_out/cfg_sweep32.err
python bench.py --no-cpu-baseline > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
python bench.py --no-cpu-baseline --model mitchell --no-full-step --no-exact-step > gpurun_out/bench_mitchell.jsonl 2> gpurun_out/bench_mitchell.err
