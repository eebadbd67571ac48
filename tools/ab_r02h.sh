set -x
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
for M8 in 7 1; do AMSIM_MIN_M8=$M8 timeout 600 python tools/sweep.py --sizes 4096 --ms 4 5 6 7 --models mitchell --reps 3 2>/dev/null | sed "s/^/{\"min_m8\": $M8, \"r\": /; s/\$/}/"; done > gpurun_out/ab_min_m8.jsonl
timeout 1500 python tools/cfg_sweep.py --reps 3 > gpurun_out/cfg_sweep_b256.jsonl 2> gpurun_out/cfg_sweep.err
timeout 900 python tools/cfg_sweep.py --reps 3 --batch 32 > gpurun_out/cfg_sweep_b32.jsonl 2> gpurun_out/cfg_sweep32.err
python bench.py --no-cpu-baseline > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
