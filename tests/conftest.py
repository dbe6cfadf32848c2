import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libswr.so")
    config.addinivalue_line("markers", "slow: long-running test")


def build_lib():
    """Build libswr.so without importing the package (whose import loads the .so)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "_swr_build", os.path.join(ROOT, "paper_2512_13921_b200", "build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.build()


def load_golden(name):
    """Parse tests/golden/<name> into {section: {key: list-of-floats or matrix}}."""
    path = os.path.join(ROOT, "tests", "golden", name)
    out, sec = {}, None
    with open(path) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            if line.startswith("["):
                sec = line.strip("[]")
                out[sec] = {}
                continue
            key, val = line.split(":", 1)
            if "/" in val:
                out[sec][key.strip()] = [[float(x) for x in r.split()] for r in val.split("/")]
            else:
                out[sec][key.strip()] = [float(x) for x in val.split()]
    return out
