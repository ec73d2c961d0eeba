"""The microserving APIs (paper_2412_12488_b200/engine.py) over the cache:
SPEC.md's transfer-plan examples, a brute-force plan property, and the
strategies of PAPER.md §3.2-3.3 (1P1D, balanced PD, context-cache reuse,
prefix-matching Cases 1 and 2) checked token for token against
HashModel::Generate.  CPU runs use the compiled reference behind the ABI with
a host fabric; GPU runs use the B200 library with device-direct sends."""
import numpy as np
import pytest

from oracle import hashmodel as hm
from paper_2412_12488_b200 import KVCache
from paper_2412_12488_b200.engine import (DIRECT_SEND, PREFILL_ONLY, PREFILL_THEN_SEND, Engine,
                                          Fabric, Segment, compute_transfer_plan)

L, W = 3, 64


def _prompt(n, seed):
    rng = np.random.Generator(np.random.MT19937(seed))
    return [int(x) for x in rng.integers(0, 256, n)]


def test_transfer_plan_spec_examples():
    # SPEC.md:297-299
    assert compute_transfer_plan(600, 200, 999) == [Segment(DIRECT_SEND, 200, 600),
                                                    Segment(PREFILL_THEN_SEND, 600, 999)]
    assert compute_transfer_plan(200, 600, 999) == [Segment(PREFILL_ONLY, 200, 600),
                                                    Segment(PREFILL_THEN_SEND, 600, 999)]
    assert compute_transfer_plan(1000, 0, 999) == [Segment(DIRECT_SEND, 0, 999)]
    assert compute_transfer_plan(0, 0, 99) == [Segment(PREFILL_THEN_SEND, 0, 99)]


@pytest.mark.parametrize("seed", range(5))
def test_transfer_plan_matches_brute_force(seed):
    """SPEC.md:304 plan-cover: segments partition [min(m, begin), end) with the
    kind a per-position classifier assigns."""
    rng = np.random.default_rng(seed)
    for _ in range(200):
        m, b = (int(x) for x in rng.integers(0, 60, 2))
        e = b + int(rng.integers(0, 40))
        want = {}
        for p in range(min(m, b), e):
            want[p] = DIRECT_SEND if b <= p < m else (PREFILL_THEN_SEND if p >= max(m, b) else
                                                      PREFILL_ONLY)
        got = {}
        segs = compute_transfer_plan(m, b, e)
        for s in segs:
            assert s.begin < s.end
            for p in range(s.begin, s.end):
                assert p not in got
                got[p] = s.kind
        assert got == want
        assert all(a.kind != c.kind for a, c in zip(segs, segs[1:]))


def _engines(make, device):
    fabric = Fabric()
    P = Engine(make(rank=0), 0, fabric)
    D = Engine(make(rank=1), 1, fabric)
    if device:
        P.attach(D)
        D.attach(P)
    return P, D


def _flows(make, device):
    # 1P1D (Fig 3): prep_recv(end=-1), remote_send, start_generate(len-1).
    p = _prompt(300, 1)
    P, D = _engines(make, device)
    m, addr = D.api_prep_recv(p, -1)
    assert m == 0 and addr.token_count == 299
    plan = P.api_remote_send(p, 0, -1, 1, addr)
    assert plan == [Segment(PREFILL_THEN_SEND, 0, 299)]
    assert D.api_start_generate(p, -1, 4) == hm.generate(p, 4, L, W)
    # Balanced PD (§3.3, r = 0.2): the decode engine prefills the tail.
    q = _prompt(500, 2)
    s = int(0.8 * len(q))
    P, D = _engines(make, device)
    m, addr = D.api_prep_recv(q, s)
    P.api_remote_send(q, 0, s, 1, addr)
    assert D.api_start_generate(q, s, 2) == hm.generate(q, 2, L, W)
    # Context-cache reuse (Fig 4): D already holds the first 120 tokens.
    P, D = _engines(make, device)
    ctx = q[:120]
    D.api_start_generate(ctx, 0, 1)  # D computes and caches ctx
    m, addr = D.api_prep_recv(q, -1)
    assert m == 120 and addr.token_begin == 120
    P.api_remote_send(q, 120, -1, 1, addr)
    assert D.api_start_generate(q, -1, 2) == hm.generate(q, 2, L, W)
    # Case 1: sender holds 350, receiver 100 -> DirectSend [100, 350) + PrefillThenSend.
    P, D = _engines(make, device)
    P.api_start_generate(q[:350], 0, 1)
    D.api_start_generate(q[:100], 0, 1)
    m, addr = D.api_prep_recv(q, -1)
    assert m == 100
    plan = P.api_remote_send(q, 100, -1, 1, addr)
    assert plan == [Segment(DIRECT_SEND, 100, 350), Segment(PREFILL_THEN_SEND, 350, 499)]
    assert D.api_start_generate(q, -1, 3) == hm.generate(q, 3, L, W)
    # Case 2: sender holds 100, receiver 350 -> PrefillOnly [100, 350) + PrefillThenSend.
    P, D = _engines(make, device)
    P.api_start_generate(q[:100], 0, 1)
    D.api_start_generate(q[:350], 0, 1)
    m, addr = D.api_prep_recv(q, -1)
    assert m == 350
    plan = P.api_remote_send(q, 350, -1, 1, addr)
    assert plan == [Segment(PREFILL_ONLY, 100, 350), Segment(PREFILL_THEN_SEND, 350, 499)]
    assert D.api_start_generate(q, -1, 2) == hm.generate(q, 2, L, W)


def test_engine_flows_on_reference(ref_lib):
    _flows(lambda rank: KVCache(num_pages=256, page_size=16, layers=L, dim=W, rank=rank,
                                lib=ref_lib), device=False)


@pytest.mark.gpu
def test_engine_flows_on_b200(cuda):
    _flows(lambda rank: KVCache(num_pages=256, page_size=16, layers=L, dim=W, rank=rank,
                                device=0), device=True)


@pytest.mark.gpu
def test_engine_flows_on_b200_host_fabric(cuda):
    """The same flows with the reference-style host fabric (sink ->
    ApplyRemoteWrite) instead of device-direct stores."""
    _flows(lambda rank: KVCache(num_pages=256, page_size=16, layers=L, dim=W, rank=rank,
                                device=0), device=False)
