"""Test-session setup.

* registers the ``gpu`` marker (tests that need a B200; run with -m gpu);
* pins host BLAS to one thread before numpy loads, like the reference's
  conftest (tests/conftest.py:1-12), so oracle timings are not oversubscribed;
* puts the repo root on sys.path so ``oracle`` and the package import.
"""

import os
import sys

for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long CPU oracle run (still in the default suite)")
