# One GPU session: bench line, ncu launch list of the same command, ncu full capture of the top kernel.
set -x
timeout 900 python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
tail -2 gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_ncu.log 2>&1
tail -2 gpurun_out/bench_ncu.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:amsim_mm_kernel -s 2 -c 1 \
    -o gpurun_out/prof_top python tools/prof_layer.py --layer l3.1.conv2 --pass fwd --reps 1 > gpurun_out/ncu_top.log 2>&1
tail -2 gpurun_out/ncu_top.log
