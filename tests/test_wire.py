"""Wire formats on the host (no GPU): KVAddrInfo binary / JSON encodings,
ack frames and frame decoding of the B200 library against the compiled
reference codec (kv_addr.cc:53-118, transport.cc:30-107) behind the same
ABI, plus the golden frames in tests/golden/frames.json."""
import json
from pathlib import Path

import numpy as np
import pytest

from paper_2412_12488_b200 import ErrorCode, KVAddrInfo, SplitserveError, load_library
from paper_2412_12488_b200.kvcache import (DecodeFrame, EncodeAckFrame, frame_write_header_size)

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def libs(product_lib, ref_lib):
    return load_library(product_lib), load_library(ref_lib)


def _status(fn):
    try:
        return ("ok", fn())
    except SplitserveError as e:
        return ("err", int(e.status))


def _random_addr(rng, n_ranges, page_size=16):
    pages = rng.choice(100000, size=n_ranges, replace=False)
    ranges, total = [], 0
    for p in pages:
        b = int(rng.integers(0, page_size))
        c = int(rng.integers(1, page_size - b + 1))
        ranges.append((int(p), b, c))
        total += c
    return KVAddrInfo(ranges, int(rng.integers(0, 1 << 40)), total)


@pytest.mark.parametrize("seed", range(6))
def test_addr_binary_and_json_match_reference(libs, seed):
    prod, ref = libs
    rng = np.random.default_rng(seed)
    for n in (0, 1, 2, 17, 512):
        a = _random_addr(rng, n)
        b = a.EncodeTo(prod)
        assert b == a.EncodeTo(ref)
        assert len(b) == 20 + 8 * n
        back, pos = KVAddrInfo.DecodeFrom(b, 0, prod)
        assert back == a and pos == len(b)
        assert KVAddrInfo.DecodeFrom(b, 0, ref) == (a, len(b))
        # Decoding from an offset inside a larger buffer advances the position.
        buf = b"\x01\x02\x03" + b + b"\xff"
        assert KVAddrInfo.DecodeFrom(buf, 3, prod) == (a, 3 + len(b))
        j = a.ToJson(prod)
        assert j == a.ToJson(ref)
        assert KVAddrInfo.FromJson(j, prod) == a == KVAddrInfo.FromJson(j, ref)


def test_addr_json_known_answer(libs):
    prod, _ = libs
    # SURVEY Appendix A.1 probe: fork at m=5, 18 tokens.
    a = KVAddrInfo([(1, 0, 16), (2, 0, 2)], 5, 18)
    assert a.ToJson(prod) == '{"ranges":[[1,0,16],[2,0,2]],"token_begin":5,"token_count":18}'
    assert KVAddrInfo([], 0, 0).ToJson(prod) == '{"ranges":[],"token_begin":0,"token_count":0}'


@pytest.mark.parametrize("text", [
    ' { "token_count" : 18 , "token_begin":5, "ranges" : [ [1,0,16] , [2,0,2] ] } ',
    '{"ranges":[[1,0,16,99],[2,0,2]],"token_begin":5,"token_count":18,"extra":{"a":[1,2]}}',
    '{"ranges":[[1.0,0,16],[2,0,2.9]],"token_begin":5.5,"token_count":18}',
    '{"ranges":[],"token_begin":0,"token_count":0}',
    '{"ranges":null,"token_begin":0,"token_count":0}',
    '{"ranges":[[1,0,16]],"token_begin":0,"token_count":16,"token_begin":3}',
    # reference-side failures: Validate (bad / overlapping ranges, coverage)
    '{"ranges":[[1,0,16],[1,3,2]],"token_begin":5,"token_count":18}',
    '{"ranges":[[1,0,0]],"token_begin":0,"token_count":0}',
    '{"ranges":[[1,0,4]],"token_begin":0,"token_count":5}',
    # malformed JSON / wrong shapes: a non-splitserve exception in the reference
    '{"ranges":[[1,0,16]],"token_begin":5}',
    '{"ranges":[[1,0]],"token_begin":0,"token_count":0}',
    '{"ranges":[["1",0,16]],"token_begin":0,"token_count":16}',
    '{"ranges":[[1,0,16]],"token_begin":0,"token_count":16',
    '{"ranges":[[1,0,16]],"token_begin":0,"token_count":16} x',
    '[1,2,3]',
    '',
])
def test_addr_from_json_edge_cases_match_reference(libs, text):
    prod, ref = libs
    assert _status(lambda: KVAddrInfo.FromJson(text, prod)) == \
        _status(lambda: KVAddrInfo.FromJson(text, ref))


def test_addr_decode_errors_match_reference(libs):
    prod, ref = libs
    a = KVAddrInfo([(7, 2, 5), (9, 0, 16)], 100, 21)
    b = a.EncodeTo(prod)
    for cut in range(len(b)):
        assert _status(lambda: KVAddrInfo.DecodeFrom(b[:cut], 0, prod)) == \
            _status(lambda: KVAddrInfo.DecodeFrom(b[:cut], 0, ref)), cut
    # token_count not covered by the ranges -> AddrMismatch; overlap -> InvalidArgument
    for bad in (KVAddrInfo([(7, 2, 5)], 0, 6), KVAddrInfo([(7, 2, 5), (7, 4, 2)], 0, 7)):
        enc = bad.EncodeTo(prod)
        got = _status(lambda: KVAddrInfo.DecodeFrom(enc, 0, prod))
        assert got == _status(lambda: KVAddrInfo.DecodeFrom(enc, 0, ref))
        assert got[0] == "err"
    # a range count far beyond the buffer
    huge = bytearray(b[:20])
    huge[16:20] = (0xFFFFFFFF).to_bytes(4, "little")
    assert _status(lambda: KVAddrInfo.DecodeFrom(bytes(huge), 0, prod)) == \
        ("err", int(ErrorCode.InvalidArgument) + 1)


def test_ack_frames_and_header_size_match_reference(libs):
    prod, ref = libs
    for tag, layer, tb, st in [(0, 0, 0, 0), (7, 79, 6553, 1), (2**64 - 1, 65535, -1, 2),
                               (123456789, 3, 2**40, 0)]:
        a = EncodeAckFrame(tag, layer, tb, st, prod)
        assert a == EncodeAckFrame(tag, layer, tb, st, ref)
        assert len(a) == 26
        d = DecodeFrame(a, prod)
        assert d == DecodeFrame(a, ref)
        assert d["type"] == 1 and d["seq_tag"] == tag and d["status"] == st
    for n in (0, 1, 32, 512):
        assert frame_write_header_size(n, prod) == frame_write_header_size(n, ref) == 41 + 8 * n


def test_golden_frames_decode(libs):
    """Frames the reference encoded (tests/golden/frames.json): the host
    decoder of both libraries reads the same header, address and CRC field."""
    prod, ref = libs
    g = json.loads((GOLD / "frames.json").read_text())
    for f in g["frames"]:
        raw = bytes.fromhex(f["hex"])
        d = DecodeFrame(raw, prod)
        assert d == DecodeFrame(raw, ref)
        assert d["layer"] == f["layer"] and d["seq_tag"] == g["tag"]
        assert d["addr"].ToJson(prod) == g["addr_json"]
        assert d["wire_crc"] == f["crc"]
        assert d["payload_offset"] + d["payload_bytes"] + 4 == len(raw)
    for a in g["acks"]:
        assert EncodeAckFrame(*a["args"], lib=prod).hex() == a["hex"]


def test_frame_decode_errors_match_reference(libs):
    prod, ref = libs
    g = json.loads((GOLD / "frames.json").read_text())
    raw = bytes.fromhex(g["frames"][0]["hex"])
    cases = [raw[:k] for k in (0, 3, 6, 7, 15, 17, 30, 41, len(raw) - 1)]
    bad_magic = bytearray(raw)
    bad_magic[0] ^= 1
    bad_version = bytearray(raw)
    bad_version[4] = 2
    bad_type = bytearray(raw)
    bad_type[6] = 5
    odd_len = bytearray(raw)
    off = 41 + 8 * len(DecodeFrame(raw, prod)["addr"].ranges) - 4
    odd_len[off] ^= 1  # payload length no longer a multiple of 8
    cases += [bytes(bad_magic), bytes(bad_version), bytes(bad_type), bytes(odd_len),
              raw + b"trailing bytes are ignored"]
    for c in cases:
        got = _status(lambda: DecodeFrame(c, prod))
        want = _status(lambda: DecodeFrame(c, ref))
        if got[0] == "ok":
            got = ("ok", {k: (v.ToJson(prod) if isinstance(v, KVAddrInfo) else v)
                          for k, v in got[1].items()})
            want = ("ok", {k: (v.ToJson(prod) if isinstance(v, KVAddrInfo) else v)
                           for k, v in want[1].items()})
        assert got == want, len(c)


def test_host_only_cache_refuses_frame_data_path(product_lib):
    from paper_2412_12488_b200 import KVCache
    E = KVCache(num_pages=8, page_size=16, layers=2, dim=8, device=-1)
    E.CreateSequence(1, list(range(20)))
    E.EnsureAllocated(1, 20)
    a = E.BuildAddr(1, (0, 16))
    with pytest.raises(SplitserveError) as ei:
        E.EncodeWriteFrame(1, (0, 16), 0, 3, a)
    assert ei.value.status == 103  # SS_ERR_NO_DEVICE: no CPU data path
