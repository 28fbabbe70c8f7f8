import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


GOLDEN = os.path.join(ROOT, "tests", "golden")


def load_example_golden():
    """Parse tests/golden/example_same_generation.txt into dicts."""
    names = ["S", "S1", "S2", "S3", "S4", "S5", "S6"]
    out = {"edges": [], "T": {}, "P0": set(), "K": None, "R": {a: set() for a in names}, "L": []}
    with open(os.path.join(GOLDEN, "example_same_generation.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            tok = line.split()
            if tok[0] == "EDGE":
                out["edges"].append((int(tok[1]), tok[2], int(tok[3])))
            elif tok[0].startswith("T"):
                k = int(tok[0][1:])
                s = out["T"].setdefault(k, set())
                for a in tok[3:]:
                    s.add((int(tok[1]), int(tok[2]), a))
            elif tok[0] == "P0":
                for a in tok[3:]:
                    out["P0"].add((int(tok[1]), int(tok[2]), a))
            elif tok[0] == "K":
                out["K"] = int(tok[1])
            elif tok[0] == "R":
                out["R"][tok[1]].add((int(tok[2]), int(tok[3])))
            elif tok[0] == "L":
                out["L"].append((tok[1], int(tok[2]), int(tok[3]), int(tok[4])))
    return out


@pytest.fixture(scope="session")
def example_golden():
    return load_example_golden()
