import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_addoption(parser):
    parser.addoption("--runslow", action="store_true", default=False,
                     help="run the slow CPU pins (e.g. Table 3 at N=64000, ~10 min on 8 cores)")


def pytest_collection_modifyitems(config, items):
    if config.getoption("--runslow") or os.environ.get("HH_RUN_SLOW"):
        return
    skip = pytest.mark.skip(reason="slow pin: run with --runslow")
    for it in items:
        if "slow" in it.keywords:
            it.add_marker(skip)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI library)")
    config.addinivalue_line("markers", "slow: long CPU-only pins (not in the default CPU suite)")


@pytest.fixture(scope="session")
def tiny_oracle():
    """Oracle H_h for BASELINE config 0 (2D tiny), built once per session."""
    import workloads as W
    from oracle import hmatrix
    cfg = W.CONFIGS["2d_tiny"]
    P = W.make_points(cfg)
    H = hmatrix.build(P, cfg["kernel"], cfg["scale"], cfg["eps"], cfg["eta"], cfg["leaf"],
                      cfg["s"], cfg["pset"], keep_exact=True)
    return cfg, P, H
