"""Test configuration. `-m "not gpu"` runs on a CPU-only host (oracle, host logic, C-ABI
exports); `-m gpu` are the parity tests proper and need a B200."""
import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); parity tests through the C-ABI")
    config.addinivalue_line("markers", "multigpu: one NCCL rank per visible GPU; skipped below 2 GPUs")


@pytest.fixture(scope="session")
def golden():
    return json.loads((ROOT / "tests" / "golden" / "golden.json").read_text())


@pytest.fixture(scope="session")
def gpu():
    """Fails loudly (never skips) when a gpu-marked test runs without a device."""
    from paper_1602_08477_b200 import kernelweave as kw
    n = kw.device_count()
    assert n > 0, "gpu-marked test needs a CUDA device"
    return kw.Device.gpu(0)


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.lib()
    return O
