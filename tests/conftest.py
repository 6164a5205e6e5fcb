import glob
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def golden_cases():
    return sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLDEN, "r*_*.json")))


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle as O

    O.lib()  # builds liboracle.so if needed
    return O


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def record_parity(test: str, **fields) -> None:
    """Appends one JSON line of parity evidence (max error ratios against the
    fp64 reference restatement) to $GESPMM_PARITY_OUT when it is set; the GPU
    runs point it into gpurun_out/ and the summary is committed under profiles/."""
    path = os.environ.get("GESPMM_PARITY_OUT")
    if not path:
        return
    with open(path, "a") as f:
        f.write(json.dumps({"test": test, **fields}) + "\n")
