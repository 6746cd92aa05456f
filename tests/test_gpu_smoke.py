"""The driver's smoke() entry point (one cfg1 step on cuda:0 against the oracle) as a GPU test."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_graft_smoke():
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    import __graft_entry__

    __graft_entry__.smoke()
