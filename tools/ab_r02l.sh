set -x
python -m pytest tests -m gpu -x -q > gpurun_out/gputest_l.log 2>&1; echo rc=$? >> gpurun_out/gputest_l.log
python tools/ab_bench.py main=paper_2209_04161_b200/libamsim.so unroll1=build/variants/libamsim_unroll1.so unroll4=build/variants/libamsim_unroll4.so --rounds 2 > gpurun_out/ab_unroll_mbm.jsonl 2>&1
python tools/ab_bench.py main=paper_2209_04161_b200/libamsim.so unroll1=build/variants/libamsim_unroll1.so unroll4=build/variants/libamsim_unroll4.so --rounds 2 --args "--steps 5 --warmup 3 --model mitchell" > gpurun_out/ab_unroll_mitchell.jsonl 2>&1
for v in main=paper_2209_04161_b200/libamsim.so unroll1=build/variants/libamsim_unroll1.so unroll4=build/variants/libamsim_unroll4.so; do
  n=${v%%=*}; lib=${v#*=}
  AMSIM_LIB=$PWD/$lib timeout 300 python tools/sweep.py --sizes 4096 --ms 7 --models mitchell mbm 2>/dev/null | sed "s/^/{\"lib\": \"$n\", \"r\": /; s/\$/}/"
done > gpurun_out/ab_unroll_gemm.jsonl
