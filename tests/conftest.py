import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs the libbam kernels)")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def unrle(rows):
    out = []
    for row in rows:
        r = []
        for n, c in row:
            r += [c] * n
        out.append(tuple(r))
    return tuple(out)


@pytest.fixture(scope="session")
def golden():
    return load_golden
