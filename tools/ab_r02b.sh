# Round-2 (second session) A/B: quad decode + REDUX flags (main) vs HEAD, and 16x8 tiles for 8-bit tables
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
python tools/ab_bench.py main=paper_2209_04161_b200/libamsim.so head=build/variants/libamsim_head.so --rounds 2 > gpurun_out/ab_mbm.jsonl 2>&1
python tools/ab_bench.py main=paper_2209_04161_b200/libamsim.so head=build/variants/libamsim_head.so nohuge8=build/variants/libamsim_nohuge8.so --rounds 2 --args "--steps 5 --warmup 3 --model mitchell" > gpurun_out/ab_mitchell.jsonl 2>&1
for v in main=paper_2209_04161_b200/libamsim.so head=build/variants/libamsim_head.so nohuge8=build/variants/libamsim_nohuge8.so; do
  n=${v%%=*}; lib=${v#*=}
  AMSIM_LIB=$PWD/$lib timeout 300 python tools/sweep.py --sizes 4096 16384 --ms 7 --models mitchell mbm 2>/dev/null | sed "s/^/{\"lib\": \"$n\", \"r\": /; s/\$/}/"
done > gpurun_out/ab_gemm.jsonl
