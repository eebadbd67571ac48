set -x
python -m pytest tests -m gpu -x -q > gpurun_out/gputest_n.log 2>&1; echo rc=$? >> gpurun_out/gputest_n.log
python tools/ab_bench.py main=paper_2209_04161_b200/libamsim.so prev=build/variants/libamsim_fwdgather.so --rounds 3 > gpurun_out/ab_wgather_mbm.jsonl 2>&1
for r in 1 2; do for v in main=paper_2209_04161_b200/libamsim.so prev=build/variants/libamsim_fwdgather.so; do
  n=${v%%=*}; lib=${v#*=}
  AMSIM_LIB=$PWD/$lib python tools/layer_table.py --top 200 2>/dev/null | grep '"stem"' | sed "s/^/$n: /"
done; done > gpurun_out/ab_wgather_stem.txt 2>&1
