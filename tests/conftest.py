import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")

try:        # the oracle's small batched ops are dominated by intra-op thread spin-up
    import torch
    torch.set_num_threads(1)
except Exception:  # pragma: no cover
    pass
