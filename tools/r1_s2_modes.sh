set -x
python -c "import paper_2209_04161_b200.build as b; b.build()"
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 600 python tools/sweep.py --sizes 4096 --ms 7 9 11 --models mitchell exact mbm --modes lut native direct > gpurun_out/sweep_modes.jsonl 2> gpurun_out/sweep_modes.err
tail -3 gpurun_out/sweep_modes.err
timeout 900 python tools/paper_ratios.py > gpurun_out/ratios.jsonl 2> gpurun_out/ratios.err
tail -3 gpurun_out/ratios.err
