"""The compiled C++ drop-in (include/splitserve_b200.h): a C++ program that
drives SURVEY.md §3's 1P1D flow through one template instantiated on the
reference's splitserve::KVCache and on the facade over libmicrokv.so
(framed and device-direct), in one binary, and requires identical match
lengths, addresses, tokens, committed frontiers, fill states and entry
digests — including with the decode engine in a second process reached over
CUDA IPC (tests/cpp/dropin_1p1d.cc; built by __graft_entry__.build() where
the reference sources exist, shipped prebuilt to the GPU box)."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "oracle" / "_ref" / "dropin_1p1d"


def test_cpp_dropin_matches_reference(cuda):
    if not BIN.exists():
        if (ROOT / "oracle" / "_ref" / "libmicrokv_ref.so").exists():
            pytest.fail(f"{BIN} missing although the reference oracle was built")
        pytest.skip("reference sources were not available at build time")
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "DROPIN OK" in r.stdout
    assert r.stdout.count("IDENTICAL") == 6  # frames, direct, cross-process IPC x 2 shapes
