set -x
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
python tools/ab_bench.py main=paper_2209_04161_b200/libamsim.so da1=build/variants/libamsim_da1.so --rounds 2 > gpurun_out/ab_da0_mbm.jsonl 2>&1
python tools/ab_bench.py main=paper_2209_04161_b200/libamsim.so da1=build/variants/libamsim_da1.so --rounds 2 --args "--steps 5 --warmup 3 --model mitchell" > gpurun_out/ab_da0_mitchell.jsonl 2>&1
timeout 1500 python tools/cfg_sweep.py --reps 3 > gpurun_out/cfg_sweep_b256.jsonl 2> gpurun_out/cfg_sweep.err
timeout 900 python tools/cfg_sweep.py --reps 3 --batch 32 > gpurun_out/cfg_sweep_b32.jsonl 2> gpurun_out/cfg_sweep32.err
python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
