set -x
python tools/ab_bench.py main=paper_2209_04161_b200/libamsim.so pack8=build/variants/libamsim_pack8.so pack8a=build/variants/libamsim_pack8a.so --rounds 2 --args "--steps 5 --warmup 3 --model mitchell" > gpurun_out/ab_pack8_mitchell.jsonl 2>&1
for v in main=paper_2209_04161_b200/libamsim.so pack8=build/variants/libamsim_pack8.so pack8a=build/variants/libamsim_pack8a.so; do
  n=${v%%=*}; lib=${v#*=}
  AMSIM_LIB=$PWD/$lib timeout 300 python tools/sweep.py --sizes 4096 16384 --ms 7 --models mitchell 2>/dev/null | sed "s/^/{\"lib\": \"$n\", \"r\": /; s/\$/}/"
done > gpurun_out/ab_pack8_gemm.jsonl
