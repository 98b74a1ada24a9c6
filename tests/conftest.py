import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libqsv.so")
    # the C oracle's gate loops may use every host core in the parity tests
    # (bit-identical to one thread: same per-pair arithmetic)
    from oracle import oracle as O

    O.set_threads(min(32, os.cpu_count() or 1))


@pytest.fixture(scope="session")
def golden():
    return np.load(os.path.join(GOLDEN, "golden_small.npz"))


@pytest.fixture(scope="session")
def h2_fixtures():
    import json

    with open(os.path.join(GOLDEN, "h2_sto3g.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def config1_golden():
    return np.load(os.path.join(GOLDEN, "config1_seed0.npz"))


def parse_h(text):
    import io

    from paper_2208_10978_b200.pauli import read_pauli_sum

    return read_pauli_sum(io.StringIO(str(text)))


def random_state(n, rng):
    a = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    return a / np.linalg.norm(a)
