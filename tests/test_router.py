"""Router strategies (SPEC.md router module, §3.2-3.3) and the
engine step loop (SPEC.md engine.step) over real caches: call scripts,
round-robin, balanced split arithmetic, context migration, hot strategy
swaps, and output invariance — every strategy's tokens equal
HashModel::Generate.  CPU runs use engines on the compiled reference with a
host fabric; GPU runs use B200 engines with device-direct sends and with
the framed (wire-format) fabric, including a mixed B200 -> reference pair."""
import numpy as np
import pytest

from oracle import hashmodel as hm
from paper_2412_12488_b200 import ErrorCode, KVCache, SplitserveError
from paper_2412_12488_b200.engine import Engine, Fabric, FrameFabric, GenRequest
from paper_2412_12488_b200.router import Router

L, W = 3, 64


def _prompt(n, seed):
    rng = np.random.Generator(np.random.MT19937(seed))
    return [int(x) for x in rng.integers(0, 256, n)]


def _cluster(make, n, roles=None, device=False, fabric=None):
    fabric = fabric if fabric is not None else Fabric()
    engines = [Engine(make(rank=r), r, fabric) for r in range(n)]
    if device:
        for a in engines:
            for b in engines:
                if a is not b:
                    a.attach(b)
    return Router(engines, roles), engines


def _calls(res):
    return [(c["call"], c["rank"]) for c in res.script]


def _strategies(make, device=False, fabric_factory=None):
    fab = (lambda: fabric_factory()) if fabric_factory else (lambda: None)
    # data_parallel: 3 engines, 4 requests -> ranks 0, 1, 2, 0
    R, _ = _cluster(make, 3, device=device, fabric=fab())
    ranks = []
    for i in range(4):
        p = _prompt(40 + i, 10 + i)
        res = R.generate(p, 3)
        assert res.tokens == hm.generate(p, 3, L, W)
        assert [c for c, _ in _calls(res)] == ["start_generate"]
        ranks.append(res.script[0]["rank"])
    assert ranks == [0, 1, 2, 0]

    # pd_disagg 1P2D: 3-call scripts, decode engine round-robin
    R, _ = _cluster(make, 3, {0: "prefill", 1: "decode", 2: "decode"}, device, fab())
    R.set_strategy("pd_disagg")
    d_ranks = []
    for i in range(4):
        p = _prompt(100, 20 + i)
        res = R.generate(p, 2)
        assert res.tokens == hm.generate(p, 2, L, W)
        calls = _calls(res)
        assert [c for c, _ in calls] == ["prep_recv", "remote_send", "start_generate"]
        assert calls[1][1] == 0 and calls[0][1] == calls[2][1]
        assert res.script[0]["result"] == (0, 99)          # all but the last token
        assert res.script[2]["args"][1] == 99               # start_generate(begin=len-1)
        d_ranks.append(calls[0][1])
    assert d_ranks == [1, 2, 1, 2]
    one = R.generate([7], 2)                                # 1-token prompt degenerates
    assert [c for c, _ in _calls(one)] == ["start_generate"] and one.tokens == hm.generate([7], 2, L, W)

    # context_pd_disagg: D matches 60 of 100 -> remote_send(begin=60) (Fig 4)
    R, E = _cluster(make, 2, {0: "prefill", 1: "decode"}, device, fab())
    p = _prompt(100, 30)
    E[1].api_start_generate(p[:60], 0, 1)
    R.set_strategy("context_pd_disagg")
    res = R.generate(p, 2)
    assert res.tokens == hm.generate(p, 2, L, W)
    assert res.script[0]["result"] == (60, 39) and res.script[1]["args"][1] == 60
    # D already holds prompt[:-1]: no transfer
    res = R.generate(p, 1)
    assert [c for c, _ in _calls(res)] == ["prep_recv", "start_generate"]
    assert res.tokens == hm.generate(p, 1, L, W)

    # balanced_pd: s = floor((1 - r) len)
    R, _ = _cluster(make, 2, {0: "prefill", 1: "decode"}, device, fab())
    R.set_strategy("balanced_pd", ratio=0.2)
    p = _prompt(1000, 40)
    res = R.generate(p, 2)
    assert res.tokens == hm.generate(p, 2, L, W)
    assert res.script[0]["args"][1] == 800 and res.script[2]["args"][1] == 800
    R.set_strategy("balanced_pd", ratio=0.3)
    q = _prompt(10, 41)
    res = R.generate(q, 2)
    assert res.script[0]["args"][1] == 7 and res.tokens == hm.generate(q, 2, L, W)
    R.set_strategy("balanced_pd", ratio=0.0)  # degenerates to Fig 3's end = len - 1
    res = R.generate(_prompt(50, 42), 1)
    assert res.script[0]["args"][1] == 49

    # set_strategy: unknown name -> UnknownStrategy, active strategy unchanged
    with pytest.raises(SplitserveError) as ei:
        R.set_strategy("round_robin_v2")
    assert ei.value.code == ErrorCode.UnknownStrategy and R.strategy == "balanced_pd"

    # output invariance across strategies for one prompt
    p = _prompt(257, 50)
    want = hm.generate(p, 4, L, W)
    for name, kw in (("data_parallel", {}), ("pd_disagg", {}), ("context_pd_disagg", {}),
                     ("balanced_pd", {"ratio": 0.25})):
        R, _ = _cluster(make, 2, {0: "prefill", 1: "decode"} if name != "data_parallel" else None,
                        device, fab())
        R.set_strategy(name, **kw)
        assert R.generate(p, 4).tokens == want, name


def _migration(make, device=False, fabric=None):
    """2 contexts on 2 engines, traffic 9:1 with threshold 2 -> one migration,
    after which the hot context is served by both engines and the target
    matches the whole context (no recompute), tokens unchanged."""
    R, E = _cluster(make, 2, device=device, fabric=fabric)
    sci, hist = _prompt(200, 60), _prompt(150, 61)
    R.register_context("science", sci, 0)
    R.register_context("history", hist, 1)
    R.set_strategy("context_migration", threshold=2.0, window=10)
    served = []
    for i in range(10):
        cat = "history" if i == 5 else "science"
        base = sci if cat == "science" else hist
        p = base + _prompt(20, 100 + i)
        res = R.generate(p, 2, category=cat)
        assert res.tokens == hm.generate(p, 2, L, W), i
        served.append((cat, res.script[0]["rank"]))
    assert R.migrations == 1
    assert sorted(R.contexts["science"].owners) == [0, 1]
    assert E[1].cache.MatchPrefix(sci) == len(sci)
    mig = [c for c in R.log if c["call"] in ("prep_recv", "remote_send")]
    assert [(c["call"], c["rank"]) for c in mig] == [("prep_recv", 1), ("remote_send", 0)]
    # the migration fired as soon as the window showed 3:0 (> threshold 2);
    # science requests were then spread over both owners
    assert served[:3] == [("science", 0)] * 3
    assert {r for c, r in served[3:] if c == "science"} == {0, 1}
    # balanced traffic never migrates
    R2, _ = _cluster(make, 2, device=device, fabric=fabric.__class__() if fabric else None)
    R2.register_context("a", sci, 0)
    R2.register_context("b", hist, 1)
    R2.set_strategy("context_migration", threshold=2.0, window=10)
    for i in range(8):
        cat = "a" if i % 2 == 0 else "b"
        R2.generate((sci if cat == "a" else hist) + _prompt(10, 400 + i), 1, category=cat)
    assert R2.migrations == 0


def _step_batching(make):
    """2 decoding requests + 1 new prefill -> one ForwardPlan
    with 3 descriptors; every request's tokens equal the oracle's."""
    E = Engine(make(rank=0), 0)
    a, b, c = _prompt(30, 1), _prompt(45, 2), _prompt(64, 3)
    ra = E.submit(GenRequest(1, a, 0, 5))
    rb = E.submit(GenRequest(2, b, 0, 5))
    E.step()  # both prefills in one batch
    assert len(E.last_batch) == 2 and not any(e.is_decode for e in E.last_batch)
    rc = E.submit(GenRequest(3, c, 0, 3))
    E.step()
    assert len(E.last_batch) == 3
    assert [e.is_decode for e in E.last_batch] == [False, True, True]
    while not E.idle():
        E.step()
    assert ra.tokens == hm.generate(a, 5, L, W)
    assert rb.tokens == hm.generate(b, 5, L, W)
    assert rc.tokens == hm.generate(c, 3, L, W)
    # start_generate before the transfer completed -> MissingKV for that
    # request only; the batch it shared runs (SPEC.md:322 protocol order)
    D = Engine(make(rank=1), 1)
    p = _prompt(80, 4)
    D.api_prep_recv(p, -1)
    bad = D.submit(GenRequest(9, p, 79, 2))
    good = D.submit(GenRequest(10, _prompt(20, 5), 0, 2))
    while not (bad.done and good.done):
        D.step()
    assert bad.error is not None and bad.error.code == ErrorCode.MissingKV
    assert good.tokens == hm.generate(_prompt(20, 5), 2, L, W)


def _ref(ref_lib):
    return lambda rank: KVCache(num_pages=512, page_size=16, layers=L, dim=W, rank=rank,
                                lib=ref_lib)


def _b200(rank):
    return KVCache(num_pages=512, page_size=16, layers=L, dim=W, rank=rank, device=0)


def test_router_strategies_on_reference(ref_lib):
    _strategies(_ref(ref_lib))


def test_router_strategies_framed_on_reference(ref_lib):
    """The same scripts with every KV byte moving as encoded write frames."""
    _strategies(_ref(ref_lib), fabric_factory=FrameFabric)


def test_context_migration_on_reference(ref_lib):
    _migration(_ref(ref_lib))


def test_step_batching_on_reference(ref_lib):
    _step_batching(_ref(ref_lib))


def test_router_errors(ref_lib):
    with pytest.raises(SplitserveError) as ei:
        Router([])
    assert ei.value.code == ErrorCode.NoEngines
    R, _ = _cluster(_ref(ref_lib), 1, {0: "decode"})
    R.set_strategy("pd_disagg")
    with pytest.raises(SplitserveError) as ei:
        R.generate(_prompt(10, 1), 1)
    assert ei.value.code == ErrorCode.RoleMissing


def test_frame_fabric_retransmits_corrupted_frame(ref_lib):
    """A frame corrupted in flight is refused by the receiver's CRC check,
    retransmitted once, and the generation is still exact."""
    hits = []

    def fault(frame):
        if not hits:
            hits.append(1)
            b = bytearray(frame)
            b[-10] ^= 0x20  # inside the payload
            return bytes(b)
        return frame

    fab = FrameFabric(fault)
    R, _ = _cluster(_ref(ref_lib), 2, {0: "prefill", 1: "decode"}, fabric=fab)
    R.set_strategy("pd_disagg")
    p = _prompt(70, 9)
    assert R.generate(p, 2).tokens == hm.generate(p, 2, L, W)
    assert fab.retransmits == 1 and fab.frames == L


@pytest.mark.gpu
def test_router_strategies_on_b200(cuda):
    _strategies(_b200, device=True)


@pytest.mark.gpu
def test_router_strategies_framed_on_b200(cuda):
    _strategies(_b200, fabric_factory=FrameFabric)


@pytest.mark.gpu
def test_context_migration_on_b200(cuda):
    _migration(_b200, device=True)


@pytest.mark.gpu
def test_step_batching_on_b200(cuda):
    _step_batching(_b200)


@pytest.mark.gpu
def test_mixed_b200_and_reference_engines_over_frames(cuda, ref_lib):
    """A B200 prefill engine and a reference decode engine on one framed
    fabric (and the reverse): the wire formats interoperate."""
    for pr, dr in ((_b200, _ref(ref_lib)), (_ref(ref_lib), _b200)):
        fab = FrameFabric()
        P, D = Engine(pr(rank=0), 0, fab), Engine(dr(rank=1), 1, fab)
        R = Router([P, D], {0: "prefill", 1: "decode"}, "pd_disagg")
        p = _prompt(333, 77)
        assert R.generate(p, 3).tokens == hm.generate(p, 3, L, W)
        assert fab.frames == L
