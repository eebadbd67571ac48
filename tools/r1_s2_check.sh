set -x
python -c "import paper_2209_04161_b200.build as b; b.build()"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 600 python tools/sweep.py --sizes 1024 4096 8192 --ms 4 5 6 7 > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
tail -3 gpurun_out/sweep.err
timeout 600 python bench.py --model mitchell --no-cpu-baseline > gpurun_out/bench_mitchell.jsonl 2>gpurun_out/bench_mitchell.err
tail -2 gpurun_out/bench_mitchell.err
