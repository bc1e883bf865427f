import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.dirname(os.path.abspath(__file__))):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    # `-m "not gpu"` is the CPU suite (oracle vs golden vectors, host logic, C-ABI symbols, gloo);
    # `-m gpu` is the parity suite proper and FAILS (BackendUnavailable) on a box without CUDA --
    # there is no CPU fallback to fall through to.
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box with -m gpu)")
