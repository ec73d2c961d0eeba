"""Pins the CPU restatement (oracle/) before it is trusted as the checker:
against the SURVEY.md §8(c) anchors recorded from the reference, against the
committed golden fixtures (tests/golden/, made by make_golden.py from the
compiled reference), and live against the compiled reference when present."""
import json
from pathlib import Path

import numpy as np
import pytest

from flows import one_p_one_d, start_generate
from scenarios import make_script, run_script

from oracle import hashmodel as hm
from oracle.kvcache_oracle import KVCache as OracleCache
from paper_2412_12488_b200 import KVCache

GOLD = Path(__file__).resolve().parent / "golden"


def _jsonable(log):
    return json.loads(json.dumps(log, default=lambda o: list(o) if isinstance(o, tuple) else str(o)))


def test_hash_anchors_from_survey():
    # recorded from the compiled reference, default ModelConfig.
    assert hm.initial_prefix_digest() == 0x359142669544E7E8
    d = hm.prefix_digests([1, 2, 3])[-1]
    assert d == 0xE9B96727E21AAEA8
    w = hm.kv_entry_words(int(d), 0, 8)
    assert int(w[0]) == 0xA5A6830EFC5DD5A2 and int(w[1]) == 0xC331B6856B9537CB
    assert hm.entry_digest(w) == 0x513963BE75BF4EEF
    assert hm.generate([1, 2, 3], 4, layers=4, dim=8) == [38, 109, 67, 117]


def test_hash_anchors_golden():
    a = json.loads((GOLD / "anchors.json").read_text())
    assert str(hm.initial_prefix_digest()) == a["initial_prefix_digest"]
    d = int(hm.prefix_digests([1, 2, 3])[-1])
    assert [str(int(x)) for x in hm.kv_entry_words(d, 0, 8)] == a["kv_entry_123_l0"]
    assert str(hm.embed(5, 7)) == a["embed_5_7"]
    assert hm.sample_token(12345, 256) == a["sample_token_of_12345"]
    assert hm.generate([1, 2, 3], 4, 4, 8) == a["generate_123_4"]


def test_restatement_tiny_1p1d_matches_golden():
    g = json.loads((GOLD / "tiny_1p1d.json").read_text())
    c = g["config"]
    P = OracleCache(num_pages=c["num_pages"], page_size=c["page_size"], layers=c["layers"],
                    dim=c["dim"])
    D = OracleCache(num_pages=c["num_pages"], page_size=c["page_size"], layers=c["layers"],
                    dim=c["dim"], rank=1)
    hid = []
    r = one_p_one_d(P, D, g["prompt"], c["end"], via="sink", hiddens=hid, max_tokens=3)
    assert r["match_len"] == g["match_len"]
    assert [list(x) for x in r["addr"].ranges] == g["addr"]["ranges"]
    assert r["addr"].ToJson() == g["addr_json"]
    assert r["tokens"] == g["tokens"]
    assert [str(int(x)) for x in hid[-1]] == g["p_hidden_last_layer"]
    assert D.GetRecord(10).own_pages == g["d_own_pages"]
    assert D.Committed(10) == g["d_committed"]
    assert [int(D.FillOf(10, 0, l)) for l in range(c["layers"])] == g["d_fill_pos0"]
    assert [int(D.FillOf(10, 511, l)) for l in range(c["layers"])] == g["d_fill_pos511"]
    assert [str(int(x)) for x in D.ReadEntryWords(10, 510, 3)] == g["d_entry_pos510_layer3"]
    import hashlib

    h = hashlib.sha256()
    for pos in range(c["prompt_len"]):
        for layer in range(c["layers"]):
            h.update(D.ReadEntryWords(10, pos, layer).astype("<u8").tobytes())
    assert h.hexdigest() == g["d_entries_sha256"]
    # The generated tokens are the whole-prompt reference generation's.
    assert r["tokens"] == hm.generate(g["prompt"], 3, c["layers"], c["dim"])


@pytest.mark.parametrize("seed", range(4))
def test_restatement_scripts_match_golden(seed):
    g = json.loads((GOLD / "scripts.json").read_text())[str(seed)]
    c = OracleCache(num_pages=24, page_size=4, layers=2, dim=8)
    assert _jsonable(run_script(c, make_script(seed, n_ops=80, data=True))) == g


@pytest.mark.parametrize("seed", range(4, 10))
def test_restatement_scripts_match_reference_live(ref_lib, seed):
    ops = make_script(seed, n_ops=100, data=True)
    a = run_script(OracleCache(num_pages=24, page_size=4, layers=2, dim=8), ops)
    b = run_script(KVCache(num_pages=24, page_size=4, layers=2, dim=8, lib=ref_lib), ops)
    assert _jsonable(a) == _jsonable(b)


@pytest.mark.parametrize("seed", range(3))
def test_split_prefill_equivalence(seed):
    """generation with KV of p[:s] precomputed equals
    whole-prompt generation, for random prompts and split points."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 80))
    p = [int(x) for x in rng.integers(0, 256, n)]
    P = OracleCache(num_pages=32, page_size=4, layers=3, dim=8)
    D = OracleCache(num_pages=32, page_size=4, layers=3, dim=8, rank=1)
    s = int(rng.integers(1, n + 1))
    r = one_p_one_d(P, D, p, s if s < n else -1, via="sink", max_tokens=2)
    assert r["tokens"] == hm.generate(p, 2, 3, 8)


def test_reference_tiny_1p1d_matches_golden(ref_lib):
    """The live reference reproduces the committed fixture (fixture sanity)."""
    g = json.loads((GOLD / "tiny_1p1d.json").read_text())
    c = g["config"]
    P = KVCache(num_pages=c["num_pages"], page_size=c["page_size"], layers=c["layers"],
                dim=c["dim"], lib=ref_lib)
    D = KVCache(num_pages=c["num_pages"], page_size=c["page_size"], layers=c["layers"],
                dim=c["dim"], rank=1, lib=ref_lib)
    r = one_p_one_d(P, D, g["prompt"], c["end"], via="sink", max_tokens=3)
    assert r["tokens"] == g["tokens"]
    assert D.GetRecord(10).own_pages == g["d_own_pages"]
