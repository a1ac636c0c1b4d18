"""Test configuration: the ``gpu`` marker and import paths.

``python -m pytest tests -m "not gpu"`` runs everywhere (CPU container);
``-m gpu`` needs a B200 and the built libacopf_b200.so.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "slow: full-size configs (minutes)")
