set -x
python tools/ab_bench.py main=paper_2209_04161_b200/libamsim.so serial=build/variants/libamsim_serial.so skipb=build/variants/libamsim_skipb.so unpackact=build/variants/libamsim_unpackact.so skipbunpack=build/variants/libamsim_skipbunpack.so --rounds 2 > gpurun_out/ab_mbm.jsonl 2>&1
python tools/ab_bench.py main=paper_2209_04161_b200/libamsim.so serial=build/variants/libamsim_serial.so skipb=build/variants/libamsim_skipb.so --rounds 2 --args "--steps 5 --warmup 3 --model mitchell" > gpurun_out/ab_mitchell.jsonl 2>&1
for r in 1 2; do for v in main=paper_2209_04161_b200/libamsim.so serial=build/variants/libamsim_serial.so; do
  n=${v%%=*}; lib=${v#*=}
  for B in 32 64; do AMSIM_LIB=$PWD/$lib timeout 300 python tools/layer_table.py --batch $B --top 0 | head -1 | sed "s/^/{\"lib\": \"$n\", \"r\": /; s/\$/}/"; done
done; done > gpurun_out/ab_tree_batch.jsonl 2> gpurun_out/ab_tree_batch.err
