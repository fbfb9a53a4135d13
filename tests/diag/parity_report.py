#!/usr/bin/env python
"""Print the GPU-vs-oracle parity report (tests/parity.py) for a named configuration (diagnostics)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from tests.gpu_common import run_config  # noqa: E402

for name in sys.argv[1:] or ["paper"]:
    *_, rep = run_config(name)
    print(name, rep)
