set -x
python -c "import paper_2209_04161_b200.build as b; b.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "global or layout or lookup" 2>&1 | tail -5
timeout 600 python tools/sweep.py --sizes 4096 --ms 8 9 10 11 --models mitchell exact
