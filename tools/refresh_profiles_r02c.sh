# Final refresh of the round-2 measurements (after the OR addresses, 8-bit layouts, cost refit) in one GPU
# session (results in gpurun_out/, copied into profiles/ with r02c names).
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
# launch list of the bench command (cold-cache, serialised) -> per-kind DRAM traffic for the roofline field
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches_r02c.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-full-step --no-exact-step > gpurun_out/bench_ncu.log 2>&1
python tools/summarize_launches.py gpurun_out/launches_r02c.csv --traffic-json gpurun_out/traffic_r02c.json > gpurun_out/launches_summary_r02c.txt
timeout 600 python bench.py --model mitchell --no-cpu-baseline --no-full-step > gpurun_out/bench_mitchell.jsonl 2> gpurun_out/bench_mitchell.err
timeout 400 python bench.py --workload resnet18 --no-cpu-baseline > gpurun_out/bench_resnet18.jsonl 2> gpurun_out/bench_resnet18.err
timeout 300 python bench.py --workload lenet5 --no-cpu-baseline > gpurun_out/bench_lenet5.jsonl 2> gpurun_out/bench_lenet5.err
timeout 300 python bench.py --workload lenet5 --no-cpu-baseline --graph > gpurun_out/bench_lenet5_graph.jsonl 2> gpurun_out/bench_lenet5_graph.err
timeout 300 python bench.py --workload resnet18 --no-cpu-baseline --graph > gpurun_out/bench_resnet18_graph.jsonl 2> gpurun_out/bench_resnet18_graph.err
timeout 300 python bench.py --impl reference > gpurun_out/bench_reference.jsonl 2> gpurun_out/bench_reference.err
timeout 900 python bench.py --workload gemm --model mitchell --steps 5 --warmup 3 > gpurun_out/bench_gemm16384.jsonl 2> gpurun_out/bench_gemm16384.err
timeout 900 python tools/sweep.py --sizes 256 512 1024 2048 4096 8192 16384 --ms 7 --models mitchell exact mbm --reps 3 > gpurun_out/sweep_gemm.jsonl 2> gpurun_out/sweep_gemm.err
timeout 600 python tools/sweep.py --sizes 4096 --ms 4 5 6 --models mitchell exact --reps 3 > gpurun_out/sweep_gemm_m456.jsonl 2> gpurun_out/sweep_gemm_m456.err
timeout 900 python tools/paper_ratios.py > gpurun_out/ratios.jsonl 2> gpurun_out/ratios.err
timeout 1200 python tools/full_step.py > gpurun_out/full_step.jsonl 2> gpurun_out/full_step.err
timeout 300 python tools/layer_table.py --top 200 > gpurun_out/layer_table.jsonl 2> gpurun_out/layer_table.err
for B in 32 64 128 256; do timeout 300 python tools/layer_table.py --batch $B --top 0 | head -1; done > gpurun_out/batch_scaling.jsonl 2> gpurun_out/batch_scaling.err
mkdir -p /tmp/reps
for LP in "l3.1.conv2 dgrad 256" "l1.1.conv2 dgrad 256" "l2.1.conv1 dgrad 256" "l3.1.conv2 fwd 256" "l3.1.conv2 wgrad 256" "l1.1.conv2 wgrad 256" "stem fwd 256"; do
  set -- $LP
  tag=$1_$2_b$3
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:amsim_mm_kernel -s 1 -c 1 \
      -o /tmp/reps/r02c_$tag python tools/prof_layer.py --layer $1 --pass $2 --batch $3 --reps 2 > gpurun_out/ncu_$tag.log 2>&1
  ncu -i /tmp/reps/r02c_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/src_r02c_$tag.csv 2>/dev/null
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:amsim_mm_kernel -s 2 -c 1 -o /tmp/reps/r02c_gemm8_4096 python tools/sweep.py --sizes 4096 --ms 7 --models mitchell > gpurun_out/ncu_gemm8.log 2>&1
ncu -i /tmp/reps/r02c_gemm8_4096.ncu-rep --page source --csv --print-source sass > gpurun_out/src_r02c_gemm8_4096.csv 2>/dev/null
python tools/ncu_summary.py /tmp/reps/r02c_*.ncu-rep > gpurun_out/ncu_summary_r02c.md
for f in gpurun_out/*.err; do tail -n 2 $f; done

timeout 1500 python tools/cfg_sweep.py --reps 3 > gpurun_out/cfg_sweep_b256.jsonl 2> gpurun_out/cfg_sweep.err
