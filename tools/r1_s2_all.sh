python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
cat gpurun_out/bench.jsonl
