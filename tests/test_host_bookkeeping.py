"""Bookkeeping parity on CPU: the product library's host side (host-only
cache, no device) against the compiled reference and the restatement, on
op scripts without a data path, plus the known-answer cases of SPEC.md /
SURVEY.md appendix A that need no KV bytes."""
import json

import pytest

from scenarios import make_script, run_script

from oracle.kvcache_oracle import KVCache as OracleCache
from paper_2412_12488_b200 import ErrorCode, KVAddrInfo, KVCache, SplitserveError


def _j(log):
    return json.loads(json.dumps(log, default=lambda o: list(o) if isinstance(o, tuple) else str(o)))


@pytest.mark.parametrize("seed", range(8))
def test_host_only_product_matches_restatement(seed):
    ops = make_script(100 + seed, n_ops=150, data=False)
    a = run_script(KVCache(num_pages=24, page_size=4, layers=2, dim=8, device=-1), ops)
    b = run_script(OracleCache(num_pages=24, page_size=4, layers=2, dim=8), ops)
    assert _j(a) == _j(b)


@pytest.mark.parametrize("seed", range(4))
def test_host_only_product_matches_reference(ref_lib, seed):
    ops = make_script(200 + seed, n_ops=150, data=False)
    a = run_script(KVCache(num_pages=24, page_size=4, layers=2, dim=8, device=-1), ops)
    b = run_script(KVCache(num_pages=24, page_size=4, layers=2, dim=8, lib=ref_lib), ops)
    assert _j(a) == _j(b)


def _impls(ref_lib_path=None):
    out = [lambda **k: KVCache(device=-1, **k), lambda **k: OracleCache(**k)]
    if ref_lib_path:
        out.append(lambda **k: KVCache(lib=ref_lib_path, **k))
    return out


@pytest.fixture(params=["product-host", "restatement", "reference"])
def make(request):
    from conftest import REF_LIB

    if request.param == "product-host":
        return lambda **k: KVCache(device=-1, **k)
    if request.param == "restatement":
        return lambda **k: OracleCache(**k)
    if not REF_LIB.exists():
        pytest.skip("reference not built")
    return lambda **k: KVCache(lib=str(REF_LIB), **k)


def test_prep_recv_end_minus_one(make):
    # empty cache, 100 tokens, end=-1 -> match 0, token_count 99.
    c = make(num_pages=64, page_size=16, layers=4, dim=8)
    r = c.PrepRecv(1, list(range(100)), -1)
    assert r.match_len == 0 and r.addr.token_count == 99 and r.addr.token_begin == 0
    assert r.addr.ranges == [(p, 0, 16) for p in range(6)] + [(6, 0, 3)]
    assert c.FreePages() == 64 - 7


def test_prep_recv_index_rules(make):
    c = make(num_pages=64, page_size=16, layers=2, dim=8)
    for end, code in ((0, ErrorCode.InvalidArgument), (11, ErrorCode.InvalidArgument),
                      (-11, ErrorCode.InvalidArgument)):
        with pytest.raises(SplitserveError) as ei:
            c.PrepRecv(1, list(range(10)), end)
        assert ei.value.code == code
    with pytest.raises(SplitserveError) as ei:
        c.PrepRecv(1, [], -1)
    assert ei.value.code == ErrorCode.InvalidArgument
    assert c.PrepRecv(1, [7], 1).addr.token_count == 1
    with pytest.raises(SplitserveError) as ei:
        c.PrepRecv(1, [7], 1)
    assert ei.value.code == ErrorCode.DuplicateSequence
    # end=-1 on a 1-token prompt is end 0 -> invalid.
    with pytest.raises(SplitserveError):
        c.PrepRecv(2, [7], -1)


def test_prep_recv_out_of_pages_is_atomic(make):
    c = make(num_pages=4, page_size=16, layers=2, dim=8)
    with pytest.raises(SplitserveError) as ei:
        c.PrepRecv(1, list(range(100)), -1)
    assert ei.value.code == ErrorCode.OutOfPages and ei.value.retryable
    assert c.FreePages() == 4 and c.SequenceCount() == 0 and not c.HasSequence(1)


def test_lifo_free_list(make):
    # initial pops 0,1,2,...; freed pages reuse last-freed-first.
    c = make(num_pages=16, page_size=4, layers=2, dim=8)
    c.CreateSequence(1, list(range(4)))
    c.EnsureAllocated(1, 4)
    c.CreateSequence(2, list(range(8)))
    c.EnsureAllocated(2, 8)
    assert c.GetRecord(1).own_pages == [0] and c.GetRecord(2).own_pages == [1, 2]
    c.FreeSequence(2)
    c.CreateSequence(3, list(range(4)))
    c.EnsureAllocated(3, 4)
    assert c.GetRecord(3).own_pages == [2]
    with pytest.raises(SplitserveError) as ei:
        c.EnsureAllocated(3, 5)
    assert ei.value.code == ErrorCode.InvalidArgument


def test_mark_send_checks(make):
    c = make(num_pages=16, page_size=4, layers=2, dim=8)
    c.CreateSequence(1, list(range(10)))
    a = KVAddrInfo([(3, 0, 4)], 0, 4)
    c.MarkSend(1, (0, 4), 1, a)
    assert c.PendingSendCount() == 1
    with pytest.raises(SplitserveError) as ei:
        c.MarkSend(1, (0, 5), 1, a)
    assert ei.value.code == ErrorCode.AddrMismatch
    with pytest.raises(SplitserveError) as ei:
        c.MarkSend(1, (1, 5), 1, a)
    assert ei.value.code == ErrorCode.AddrMismatch
    with pytest.raises(SplitserveError) as ei:
        c.MarkSend(1, (0, 11), 1, KVAddrInfo([], 0, 11))
    assert ei.value.code == ErrorCode.InvalidArgument


def test_build_addr_runs_and_own_slots_only(make):
    c = make(num_pages=16, page_size=4, layers=2, dim=8)
    c.CreateSequence(1, list(range(10)))
    c.EnsureAllocated(1, 10)
    assert c.BuildAddr(1, (1, 9)).ranges == [(0, 1, 3), (1, 0, 4), (2, 0, 1)]
    c.ForkSequence(1, 2, 0, list(range(5)))
    assert c.GetRecord(2).parent == -1


def test_unknown_sequence(make):
    c = make(num_pages=4, page_size=4, layers=2, dim=8)
    for call in (lambda: c.EnsureAllocated(9, 1), lambda: c.FreeSequence(9),
                 lambda: c.GetRecord(9), lambda: c.Committed(9)):
        with pytest.raises(SplitserveError) as ei:
            call()
        assert ei.value.code == ErrorCode.UnknownSequence


def test_evict_zero_and_cannot_evict(make):
    c = make(num_pages=4, page_size=4, layers=2, dim=8)
    assert c.Evict(0) == 0
    c.CreateSequence(1, list(range(16)))
    c.EnsureAllocated(1, 16)
    with pytest.raises(SplitserveError) as ei:
        c.Evict(c.BytesPerPage() if hasattr(c, "BytesPerPage") else 1)
    assert ei.value.code == ErrorCode.CannotEvict


def test_addr_validate_and_slice(product_lib):
    a = KVAddrInfo([(1, 0, 16), (2, 0, 2)], 5, 18)
    a.Validate()
    assert a.ToJson() == '{"ranges":[[1,0,16],[2,0,2]],"token_begin":5,"token_count":18}'
    assert KVAddrInfo.FromJson(a.ToJson()) == KVAddrInfo([(1, 0, 16), (2, 0, 2)], 5, 18)
    assert a.Slice(10, 22).ranges == [(1, 5, 11), (2, 0, 1)]
    with pytest.raises(SplitserveError) as ei:
        KVAddrInfo([(1, 0, 4), (1, 3, 2)], 0, 6).Validate()
    assert ei.value.code == ErrorCode.InvalidArgument
    with pytest.raises(SplitserveError) as ei:
        KVAddrInfo([(1, 0, 4)], 0, 5).Validate()
    assert ei.value.code == ErrorCode.AddrMismatch
    with pytest.raises(SplitserveError):
        a.Slice(4, 10)
