set -x
python tools/ab_bench.py head=build/variants/libamsim_head.so vote=build/variants/libamsim_vote.so swp=build/variants/libamsim_swp.so addror=build/variants/libamsim_addror.so --rounds 2 > gpurun_out/ab_swp_mbm.jsonl 2>&1
python tools/ab_bench.py head=build/variants/libamsim_head.so swp=build/variants/libamsim_swp.so addror=build/variants/libamsim_addror.so --rounds 2 --args "--steps 5 --warmup 3 --model mitchell" > gpurun_out/ab_swp_mitchell.jsonl 2>&1
for v in head=build/variants/libamsim_head.so addror=build/variants/libamsim_addror.so; do
  n=${v%%=*}; lib=${v#*=}
  AMSIM_LIB=$PWD/$lib timeout 300 python tools/sweep.py --sizes 4096 16384 --ms 7 --models mitchell mbm 2>/dev/null | sed "s/^/{\"lib\": \"$n\", \"r\": /; s/\$/}/"
done > gpurun_out/ab_addror_gemm.jsonl
