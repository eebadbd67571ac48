# Refresh every committed measurement in one GPU session (round-1 naming).
set -x
python -c "import paper_2209_04161_b200.build as b; b.build()"
bash tools/gpu_bench_profile.sh > gpurun_out/prof.log 2>&1
timeout 900 python tools/sweep.py --sizes 256 512 1024 2048 4096 8192 16384 --ms 4 5 6 7 --models mitchell exact > gpurun_out/sweep_full.jsonl 2> gpurun_out/sweep_full.err
timeout 600 python tools/sweep.py --sizes 4096 --ms 7 9 11 --models mitchell exact mbm --modes lut native direct > gpurun_out/sweep_modes.jsonl 2> gpurun_out/sweep_modes.err
timeout 900 python tools/paper_ratios.py > gpurun_out/ratios.jsonl 2> gpurun_out/ratios.err
timeout 1200 python tools/full_step.py > gpurun_out/full_step.jsonl 2> gpurun_out/full_step.err
timeout 300 python bench.py --model mitchell --no-cpu-baseline > gpurun_out/bench_mitchell.jsonl 2> gpurun_out/bench_mitchell.err
for f in gpurun_out/*.err; do tail -n 2 $f; done
timeout 300 python bench.py --workload gemm --model mitchell > gpurun_out/bench_gemm.jsonl 2> gpurun_out/bench_gemm.err
timeout 300 python tools/layer_table.py --top 40 > gpurun_out/layer_table.jsonl 2> gpurun_out/layer_table.err
for B in 32 64 128 256; do timeout 300 python tools/layer_table.py --batch $B --top 0 | head -1; done > gpurun_out/batch_scaling.jsonl 2> gpurun_out/batch_scaling.err
