import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) CUDA device")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # noqa: BLE001
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle, build
    build()
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import REF_SO, Reference, build
    build()
    if not os.path.exists(REF_SO):
        pytest.skip("reference library not built (reference tree absent and no prebuilt .so)")
    return Reference()


@pytest.fixture(scope="session")
def lib():
    from paper_2406_16260_b200 import _lib
    from paper_2406_16260_b200.build import build
    build()
    return _lib.load()


# Parity errors recorded by the GPU tests (name -> (normwise error, tolerance)), printed in
# the terminal summary so every run shows the measured errors, not only pass/fail.
PARITY: dict = {}


@pytest.fixture(scope="session")
def parity_log():
    return PARITY


def pytest_terminal_summary(terminalreporter):
    if not PARITY:
        return
    tr = terminalreporter
    tr.section("parity (normwise max|got - want| / max|want|)")
    for name, (err, tol) in sorted(PARITY.items()):
        tr.write_line(f"{name:72s} {err:.3e}  (tol {tol:.0e})")
