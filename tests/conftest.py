import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

REF_LIB = ROOT / "oracle" / "_ref" / "libmicrokv_ref.so"
PRODUCT_LIB = ROOT / "paper_2412_12488_b200" / "_lib" / "libmicrokv.so"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def ref_lib():
    if not REF_LIB.exists():
        pytest.skip("oracle/_ref/libmicrokv_ref.so not built (needs /root/reference at build time)")
    return str(REF_LIB)


@pytest.fixture(scope="session")
def product_lib():
    if not PRODUCT_LIB.exists():
        from paper_2412_12488_b200 import build

        build.build()
    return str(PRODUCT_LIB)


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu test without a CUDA device")
    return torch
