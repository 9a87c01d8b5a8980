import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libigb.so")
    config.addinivalue_line("markers", "slow: longer-running case")


def load_golden(name):
    path = os.path.join(GOLDEN, f"{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} missing")
    return dict(np.load(path, allow_pickle=False))


# (golden name, config builder name, builder kwargs)
SMALL_CASES = [
    ("cfg1", "cfg1", {}),
    ("cfg2_L3", "cfg2", {"levels": 3}),
    ("cfg3_L2", "cfg3", {"levels": 2}),
    ("cfg4_p2_L3", "cfg4", {"p": 2, "levels": 3}),
    ("cfg4_p4_L3", "cfg4", {"p": 4, "levels": 3}),
    ("cfg5_L1", "cfg5", {"levels": 1}),
    ("cfg5_L2", "cfg5", {"levels": 2}),
    ("cfg4_p6_L3", "cfg4", {"p": 6, "levels": 3}),
    ("cfg4_p8_L3", "cfg4", {"p": 8, "levels": 3}),
]

_setup_cache = {}


def get_setup(cfg_name, **kw):
    """Host setup of a configuration (cached per session): (problem, setup, f)."""
    key = (cfg_name, tuple(sorted(kw.items())))
    if key not in _setup_cache:
        from paper_1902_01818_b200 import configs, multigrid
        pr = configs.build(cfg_name, **kw)
        setup = multigrid.MultigridSetup(pr.hier, pr.config)
        f = pr.rhs(setup.assembled_finest)
        _setup_cache[key] = (pr, setup, f)
    return _setup_cache[key]
