"""Shared pytest configuration: registers the ``gpu`` marker.

``-m "not gpu"`` runs the oracle pins, host logic and the C-ABI export check
on CPU; ``-m gpu`` runs the parity tests proper against the CUDA library.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libsphinx.so")


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle
    return oracle.load()


@pytest.fixture(scope="session")
def sphinx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2511_18672_b200 as sp
    sp.load()  # raises loudly if the CUDA library is missing
    return sp
