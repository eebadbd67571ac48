set -x
python tools/ab_bench.py main=paper_2209_04161_b200/libamsim.so pair=build/variants/libamsim_pair.so --rounds 3 > gpurun_out/ab_pair_mbm.jsonl 2>&1
python tools/ab_bench.py main=paper_2209_04161_b200/libamsim.so pair=build/variants/libamsim_pair.so --rounds 2 --args "--steps 5 --warmup 3 --model mitchell" > gpurun_out/ab_pair_mitchell.jsonl 2>&1
