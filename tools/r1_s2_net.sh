python -c "import paper_2209_04161_b200.build as b; b.build()"
timeout 900 python -m pytest tests/test_net.py -x -q 2>&1 | tail -15
timeout 1200 python tools/full_step.py > gpurun_out/full_step.jsonl 2> gpurun_out/full_step.err
tail -5 gpurun_out/full_step.err
cat gpurun_out/full_step.jsonl
