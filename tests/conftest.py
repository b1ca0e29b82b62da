import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    # the host packaging is native too: make sure the in-tree library exists
    # (no-op when up to date; nvcc cross-compiles without a GPU)
    import __graft_entry__
    try:
        __graft_entry__.build_library()
    except Exception as exc:  # GPU box without nvcc: the shipped .so is used
        print(f"[conftest] library build skipped: {exc}")
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=False)


@pytest.fixture(scope="session")
def golden():
    import json
    with open(os.path.join(GOLDEN, "golden.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def gload():
    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = np.load(os.path.join(GOLDEN, name))
        return cache[name]
    return load
