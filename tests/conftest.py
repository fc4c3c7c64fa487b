import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def read_golden(name):
    """Parse a P:139-style text tensor file: '#' comments, then (shape line, values line) pairs
    or single scalar lines.  Returns a list of numpy arrays / floats in file order."""
    out = []
    lines = [l.strip() for l in open(os.path.join(GOLDEN, name)) if l.strip() and not l.startswith("#")]
    i = 0
    while i < len(lines):
        head = lines[i].split(",")
        if i + 1 < len(lines) and len(head) >= 1 and all(h.isdigit() for h in head) and len(head) > 1:
            shape = tuple(int(h) for h in head)
            vals = np.array([float(v) for v in lines[i + 1].split(",")])
            assert vals.size == int(np.prod(shape)), name
            out.append(vals.reshape(shape))
            i += 2
        else:
            out.append(float(lines[i]))
            i += 1
    return out


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.lib()
    return oracle
