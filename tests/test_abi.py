"""The C-ABI boundary: both libraries load and export every entry point
include/microkv.h declares; host-only caches refuse data-path calls loudly."""
import ctypes as C
import re
from pathlib import Path

import pytest

from paper_2412_12488_b200 import (EXPORTED_SYMBOLS, ErrorCode, KVCache, SplitserveError,
                                   load_library)

HEADER = Path(__file__).resolve().parents[1] / "include" / "microkv.h"


def declared():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    names = set(re.findall(r"\b(ss_[a-z0-9_]+)\s*\(", text))
    return sorted(n for n in names if n != "ss_frame_sink")


def test_header_declares_the_mirror():
    d = declared()
    assert len(d) >= 60
    assert set(d) == set(EXPORTED_SYMBOLS), set(d) ^ set(EXPORTED_SYMBOLS)


def test_product_library_exports_every_symbol(product_lib):
    lib = C.CDLL(product_lib)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    L = load_library(product_lib)
    assert L.ss_abi_version() == 1
    assert L.ss_impl_name() == b"microkv-b200"


def test_reference_library_exports_every_symbol(ref_lib):
    lib = C.CDLL(ref_lib)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert load_library(ref_lib).ss_impl_name() == b"splitserve-reference"


def test_status_names_match_reference_error_codes(product_lib):
    lib = load_library(product_lib)
    for code in ErrorCode:
        assert lib.ss_status_name(int(code) + 1).decode() == code.name
    assert lib.ss_status_retryable(int(ErrorCode.OutOfPages) + 1) == 1
    assert lib.ss_status_retryable(int(ErrorCode.PeerUnreachable) + 1) == 1
    assert lib.ss_status_retryable(int(ErrorCode.MissingKV) + 1) == 0


def test_config_validation(product_lib):
    # CacheConfig::Validate (config.cc:23-27): page_size must be a power of two.
    with pytest.raises(SplitserveError) as ei:
        KVCache(num_pages=8, page_size=12, layers=2, dim=8, device=-1)
    assert ei.value.code == ErrorCode.InvalidArgument
    with pytest.raises(SplitserveError):
        KVCache(num_pages=0, page_size=16, layers=2, dim=8, device=-1)


def test_host_only_cache_has_no_data_path(product_lib):
    c = KVCache(num_pages=8, page_size=16, layers=2, dim=8, device=-1)
    c.CreateSequence(1, list(range(20)))
    c.EnsureAllocated(1, 20)
    for call in (lambda: c.ReadEntryWords(1, 0, 0), lambda: c.GatherRange(1, (0, 4), 0),
                 lambda: c.FillOf(1, 0, 0), lambda: c.export_ipc(),
                 lambda: c.pool_layer_ptr(0)):
        with pytest.raises(SplitserveError) as ei:
            call()
        assert ei.value.name == "NoDevice"
    from paper_2412_12488_b200 import BatchEntry

    plan = c.BeginForward([BatchEntry(1, (0, 20))])
    with pytest.raises(SplitserveError) as ei:
        c.Attention(0, plan, [0] * 20)
    assert ei.value.name == "NoDevice"


def test_missing_product_library_fails_loudly(tmp_path):
    with pytest.raises(FileNotFoundError):
        load_library(tmp_path / "libmicrokv.so")


def test_cache_config_mirrors_reference(product_lib, ref_lib):
    """cache_config() (kv_cache.h:235) plus the model geometry, on both libraries."""
    for lib in (product_lib, ref_lib):
        E = KVCache(num_pages=12, page_size=8, layers=3, dim=16, device=-1, rank=2, lib=lib)
        c = E.cache_config()
        assert (c["num_pages"], c["page_size"], c["layers"], c["dim"], c["rank"]) == (12, 8, 3, 16, 2)
        assert c["hash_seed"] == 0x5eed5eed5eed5eed and c["vocab"] == 256
