set -x
python -m pytest tests -m gpu -x -q > gpurun_out/gputest_m.log 2>&1; echo rc=$? >> gpurun_out/gputest_m.log
python tools/ab_bench.py main=paper_2209_04161_b200/libamsim.so prev=build/variants/libamsim_prevgather.so --rounds 3 > gpurun_out/ab_gather_mbm.jsonl 2>&1
for r in 1 2; do for v in main=paper_2209_04161_b200/libamsim.so prev=build/variants/libamsim_prevgather.so; do
  n=${v%%=*}; lib=${v#*=}
  AMSIM_LIB=$PWD/$lib python tools/layer_table.py --top 200 2>/dev/null | grep '"stem"' | sed "s/^/$n: /"
  AMSIM_LIB=$PWD/$lib python bench.py --workload lenet5 --no-cpu-baseline --no-full-step --no-e2e --no-exact-step --graph 2>/dev/null | tail -1 | cut -c1-160 | sed "s/^/$n lenet: /"
done; done > gpurun_out/ab_gather_stem.txt 2>&1
