import os
import sys
from pathlib import Path

# The threaded virtual-rank tests run P ranks in ONE process (one CUDA context): a lazily
# loaded kernel module on one rank's thread synchronises the context while another rank's
# handshake kernel spins waiting for it -- a harness-only deadlock (separate processes have
# separate contexts).  Load every module at context creation instead.
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
# test helpers (autosp_cpu_lowering: the test-only CPU/gloo lowering of the custom ops)
if str(ROOT / "tests") not in sys.path:
    sys.path.insert(0, str(ROOT / "tests"))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libautosp.so")
    config.addinivalue_line("markers", "slow: multi-second CPU test")


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN


def reference_available() -> bool:
    return Path("/root/reference/pkg/src/seqcomp").is_dir() and not os.environ.get("NO_REF")
