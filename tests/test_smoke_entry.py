"""The driver's round-end smoke() (`__graft_entry__.smoke`) as a GPU test, so a
smoke regression (e.g. a schedule change that alters the summation order of its
default-plan checks) fails `pytest -m gpu` instead of only the driver's run."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


@pytest.mark.gpu
def test_graft_smoke():
    import __graft_entry__ as g
    g.smoke()
