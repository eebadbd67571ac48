# Refresh the round-2 measurements in one GPU session (results in gpurun_out/,
# copied into profiles/ with r02 names by hand).
set -x
python -c "import paper_2209_04161_b200.build as b; b.build()"
# launch list of the bench command (cold-cache, serialised) -> per-kind DRAM traffic for the roofline field
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches_r02.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-full-step --no-exact-step > gpurun_out/bench_ncu.log 2>&1
python tools/summarize_launches.py gpurun_out/launches_r02.csv --traffic-json gpurun_out/traffic_r02.json > gpurun_out/launches_summary_r02.txt
timeout 400 python bench.py --workload resnet18 --no-cpu-baseline > gpurun_out/bench_resnet18.jsonl 2> gpurun_out/bench_resnet18.err
timeout 300 python bench.py --workload lenet5 --no-cpu-baseline > gpurun_out/bench_lenet5.jsonl 2> gpurun_out/bench_lenet5.err
timeout 900 python bench.py --workload gemm --model mitchell --steps 5 --warmup 3 > gpurun_out/bench_gemm16384.jsonl 2> gpurun_out/bench_gemm16384.err
timeout 900 python tools/sweep.py --sizes 256 512 1024 2048 4096 8192 16384 --ms 7 --models mitchell exact mbm --reps 3 > gpurun_out/sweep_gemm.jsonl 2> gpurun_out/sweep_gemm.err
timeout 900 python tools/paper_ratios.py > gpurun_out/ratios.jsonl 2> gpurun_out/ratios.err
timeout 1200 python tools/full_step.py > gpurun_out/full_step.jsonl 2> gpurun_out/full_step.err
timeout 300 python tools/layer_table.py --top 200 > gpurun_out/layer_table.jsonl 2> gpurun_out/layer_table.err
for B in 32 64 128 256; do timeout 300 python tools/layer_table.py --batch $B --top 0 | head -1; done > gpurun_out/batch_scaling.jsonl 2> gpurun_out/batch_scaling.err
mkdir -p /tmp/reps
for LP in "l3.1.conv2 dgrad 256" "l1.1.conv2 dgrad 256" "l2.1.conv1 dgrad 256" "l3.1.conv2 fwd 256" "l3.1.conv2 wgrad 256"; do
  set -- $LP
  tag=$1_$2_b$3
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:amsim_mm_kernel -s 1 -c 1 \
      -o /tmp/reps/r02_$tag python tools/prof_layer.py --layer $1 --pass $2 --batch $3 --reps 2 > gpurun_out/ncu_$tag.log 2>&1
  ncu -i /tmp/reps/r02_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/src_r02_$tag.csv 2>/dev/null
done
python tools/ncu_summary.py /tmp/reps/r02_*.ncu-rep > gpurun_out/ncu_summary_r02.md
for f in gpurun_out/*.err; do tail -n 2 $f; done
