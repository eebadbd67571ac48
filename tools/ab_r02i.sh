set -x
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
timeout 1500 python tools/cfg_sweep.py --reps 3 > gpurun_out/cfg_sweep_b256.jsonl 2> gpurun_out/cfg_sweep.err
timeout 900 python tools/cfg_sweep.py --reps 3 --batch 32 > gpurun_out/cfg_sweep_b32.jsonl 2> gpurun_out/cfg_sweep32.err
python bench.py --no-cpu-baseline > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
python bench.py --no-cpu-baseline --model mitchell --no-full-step --no-exact-step > gpurun_out/bench_mitchell.jsonl 2> gpurun_out/bench_mitchell.err
