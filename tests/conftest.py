import os
import sys

import pytest

# peer / pipeline waits give up (WHALE_ERR_COMM) or trap after this long instead of the
# library's 300 s default, so a broken kernel fails its test quickly
os.environ.setdefault("WHALE_TIMEOUT_MS", "30000")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU and the built CUDA library")
    config.addinivalue_line("markers", "multigpu: needs >= 2 GPUs (run via torchrun)")
