# One GPU session: bench line, ncu launch list (+ DRAM bytes per launch) of the same command,
# ncu --set full captures of the top kernel configurations (reports kept in /tmp on the box,
# summaries + raw CSV pages copied to gpurun_out/, one report brought back).
set -x
timeout 900 python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
tail -2 gpurun_out/bench.err
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-full-step > gpurun_out/bench_ncu.log 2>&1
tail -2 gpurun_out/bench_ncu.log
mkdir -p /tmp/reps
for LP in "l3.1.conv2 fwd" "l1.0.conv2 fwd" "l3.1.conv2 wgrad" "l3.1.conv2 dgrad"; do
  set -- $LP
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:amsim_mm_kernel -s 1 -c 1 \
      -o /tmp/reps/prof_$1_$2 python tools/prof_layer.py --layer $1 --pass $2 --reps 1 > gpurun_out/ncu_$1_$2.log 2>&1
  tail -1 gpurun_out/ncu_$1_$2.log
  ncu -i /tmp/reps/prof_$1_$2.ncu-rep --page raw --csv > gpurun_out/raw_$1_$2.csv 2>/dev/null
done
python tools/ncu_summary.py /tmp/reps/*.ncu-rep > gpurun_out/ncu_summary.md
cp /tmp/reps/prof_l3.1.conv2_fwd.ncu-rep gpurun_out/
