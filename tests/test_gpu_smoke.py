"""__graft_entry__.smoke() -- the driver's round-end check -- as a GPU test (tensor path fp32, DMMA fp64)."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_graft_entry_smoke():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    import __graft_entry__

    __graft_entry__.smoke()
