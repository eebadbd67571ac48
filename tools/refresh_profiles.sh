# Refresh the committed round-1 measurements in one GPU session.  Results land
# in gpurun_out/; copy the ones to keep into profiles/ (round-1 names).
# The approx-GEMM sweeps (tools/sweep.py) are separate: dense N(0,1) operands,
#   timeout 900 python tools/sweep.py --sizes 256 512 1024 2048 4096 8192 16384 --ms 4 5 6 7 --models mitchell exact
#   timeout 600 python tools/sweep.py --sizes 4096 --ms 7 9 11 --models mitchell exact mbm --modes lut native direct
set -x
python -c "import paper_2209_04161_b200.build as b; b.build()"
# launch list of the bench command (cold-cache, serialised) -> per-kind DRAM traffic for the roofline field
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-full-step > gpurun_out/bench_ncu.log 2>&1
python tools/summarize_launches.py gpurun_out/launches.csv --traffic-json profiles/r01_traffic.json > gpurun_out/launches_summary.txt
cp profiles/r01_traffic.json gpurun_out/traffic.json
timeout 900 python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
tail -2 gpurun_out/bench.err
mkdir -p /tmp/reps
for LP in "l3.1.conv2 fwd" "l3.1.conv2 wgrad" "l3.1.conv2 dgrad" "l1.0.conv2 fwd"; do
  set -- $LP
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:amsim_mm_kernel -s 1 -c 1 \
      -o /tmp/reps/prof_$1_$2 python tools/prof_layer.py --layer $1 --pass $2 --reps 1 > gpurun_out/ncu_$1_$2.log 2>&1
  ncu -i /tmp/reps/prof_$1_$2.ncu-rep --page raw --csv > gpurun_out/raw_$1_$2.csv 2>/dev/null
done
python tools/ncu_summary.py /tmp/reps/*.ncu-rep > gpurun_out/ncu_summary.md
timeout 300 python bench.py --model mitchell --no-cpu-baseline > gpurun_out/bench_mitchell.jsonl 2> gpurun_out/bench_mitchell.err
timeout 900 python tools/paper_ratios.py > gpurun_out/ratios.jsonl 2> gpurun_out/ratios.err
timeout 1200 python tools/full_step.py > gpurun_out/full_step.jsonl 2> gpurun_out/full_step.err
timeout 300 python tools/layer_table.py --top 40 > gpurun_out/layer_table.jsonl 2> gpurun_out/layer_table.err
for B in 32 64 128 256; do timeout 300 python tools/layer_table.py --batch $B --top 0 | head -1; done > gpurun_out/batch_scaling.jsonl 2> gpurun_out/batch_scaling.err
for f in gpurun_out/*.err; do tail -n 2 $f; done
