"""Wire formats on the B200: device CRC-32 against the reference Crc32
(transport.cc:14-28), write frames encoded from HBM against the reference's
EncodeWriteFrame (byte-identical), and the receive step of the TCP fabric
(tcp_fabric.cc:144-168) — acks, KV contents and completions identical to
the reference on the same frames, corrupted and misaddressed frames
included."""
import ctypes as C
import json
from pathlib import Path

import numpy as np
import pytest

from flows import prefill
from paper_2412_12488_b200 import ApplyStatus, ErrorCode, KVAddrInfo, KVCache, SplitserveError
from paper_2412_12488_b200.kvcache import DecodeFrame, frame_write_header_size

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def ref_crc(ref_lib):
    lib = C.CDLL(ref_lib)
    lib.ssref_crc32.restype = C.c_uint32
    lib.ssref_crc32.argtypes = [C.c_char_p, C.c_int64]
    return lambda b: int(lib.ssref_crc32(b, len(b)))


def _dev_crc(torch, E, buf: bytes, offset: int = 0) -> int:
    t = torch.zeros(len(buf) + offset + 64, dtype=torch.uint8, device="cuda")
    if buf:
        t[offset:offset + len(buf)] = torch.frombuffer(bytearray(buf), dtype=torch.uint8).cuda()
    out = torch.zeros(1, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream()
    E.crc32_async(t.data_ptr() + offset, len(buf), out.data_ptr(), s.cuda_stream)
    torch.cuda.synchronize()
    return int(out.item()) & 0xFFFFFFFF


def test_crc32_known_answers(cuda):
    g = json.loads((GOLD / "frames.json").read_text())["crc32"]
    E = KVCache(num_pages=4, page_size=16, layers=1, dim=8, device=0)
    assert _dev_crc(cuda, E, b"123456789") == 0xCBF43926 == g["123456789"]
    rng = np.random.Generator(np.random.MT19937(11))
    for n in (0, 1, 31, 32, 33, 1000, 4096, 65549):
        buf = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        assert _dev_crc(cuda, E, buf) == g[f"mt19937_11_{n}"], n


@pytest.mark.parametrize("offset", [0, 1, 5, 8, 16, 31])
def test_crc32_matches_reference_any_length_and_alignment(cuda, ref_crc, offset):
    E = KVCache(num_pages=4, page_size=16, layers=1, dim=8, device=0)
    rng = np.random.default_rng(offset)
    for n in (0, 1, 2, 7, 8, 24, 32, 33, 63, 64, 100, 1023, 1024, 1025, 2048 + 40, 4096,
              32768 + 8, 1 << 20, (1 << 20) + 17, 3 * (1 << 20) + 96):
        buf = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        assert _dev_crc(cuda, E, buf, offset) == ref_crc(buf), (n, offset)


def test_crc32_large_payload(cuda, ref_crc):
    """A 70B-shape per-layer frame payload: 8,191 rows x 4 KiB = 33.5 MB."""
    E = KVCache(num_pages=4, page_size=16, layers=1, dim=8, device=0)
    rng = np.random.default_rng(9)
    buf = rng.integers(0, 256, 8191 * 4096, dtype=np.uint8).tobytes()
    assert _dev_crc(cuda, E, buf) == ref_crc(buf)
    # a single flipped bit anywhere changes it
    b2 = bytearray(buf)
    b2[12_345_678] ^= 0x10
    assert _dev_crc(cuda, E, bytes(b2)) == ref_crc(bytes(b2)) != ref_crc(buf)


def _sender_pair(lib_kw, L, W, P, p, m_prefix=5):
    """D holds a committed prefix of p (fork-relative receive pages); P has
    computed [0, e).  Returns (P, D, prep_recv result, m, e)."""
    D = KVCache(num_pages=64, page_size=P, layers=L, dim=W, rank=1, **lib_kw)
    D.CreateSequence(1, p[:m_prefix])
    D.EnsureAllocated(1, m_prefix)
    prefill(D, 1, p, 0, m_prefix)
    D.CommitToTree(1)
    r = D.PrepRecv(2, p, -1)
    m, e = r.match_len, r.match_len + r.addr.token_count
    Pe = KVCache(num_pages=64, page_size=P, layers=L, dim=W, rank=0, **lib_kw)
    Pe.CreateSequence(20, p)
    Pe.EnsureAllocated(20, e)
    prefill(Pe, 20, p, 0, e)
    return Pe, D, r, m, e


def test_golden_frames_encode_and_receive(cuda):
    g = json.loads((GOLD / "frames.json").read_text())
    c = g["config"]
    Pe, D, r, m, e = _sender_pair({"device": 0}, c["layers"], c["dim"], c["page_size"],
                                  g["prompt"])
    assert (m, e) == (g["match_len"], g["end"]) and r.addr.ToJson() == g["addr_json"]
    for f in g["frames"]:
        got = Pe.EncodeWriteFrame(20, (m, e), f["layer"], g["tag"], r.addr)
        assert got.hex() == f["hex"], f"layer {f['layer']}"
        ack, st = D.ReceiveWriteFrame(got)
        assert ack.hex() == f["ack_hex"] and st == f["apply_status"]
    bad = bytearray(bytes.fromhex(g["frames"][0]["hex"]))
    bad[g["corrupt_frame0"]["flip_byte"]] ^= 0x40
    ack, st = D.ReceiveWriteFrame(bytes(bad))
    assert ack.hex() == g["corrupt_frame0"]["ack_hex"] and st == -1
    assert D.DrainReceiveCompletions() == g["completions"]


@pytest.mark.parametrize("dim,page", [(8, 16), (128, 16), (512, 16), (24, 4)])
def test_frames_match_reference(cuda, ref_lib, dim, page):
    """Same ops on the B200 library and the reference: every frame
    byte-identical (host and device-memory variants); frames crossing
    engines (B200 -> reference, reference -> B200) give identical acks,
    KV contents and completions; a corrupted payload is refused by both."""
    L = 3
    rng = np.random.default_rng(dim)
    p = [int(x) for x in rng.integers(0, 256, 75)]
    gP, gD, gr, m, e = _sender_pair({"device": 0}, L, dim, page, p)
    rP, rD, rr, rm, re_ = _sender_pair({"lib": ref_lib}, L, dim, page, p)
    assert (m, e) == (rm, re_) and gr.addr == rr.addr
    tag = 0xABCDEF
    hdr = frame_write_header_size(len(gr.addr.ranges))
    frames = []
    for layer in range(L):
        f = gP.EncodeWriteFrame(20, (m, e), layer, tag, gr.addr)
        assert f == rP.EncodeWriteFrame(20, (m, e), layer, tag, rr.addr), layer
        # device-memory frame: payload 32-byte aligned at frame + header
        buf = cuda.zeros(len(f) + 64, dtype=cuda.uint8, device="cuda")
        base = buf.data_ptr()
        off = (-(base + hdr)) % 32
        n = gP.encode_write_frame_async(20, (m, e), layer, tag, gr.addr, base + off,
                                        len(f) + 64 - off, cuda.cuda.current_stream().cuda_stream)
        cuda.cuda.synchronize()
        assert n == len(f) and bytes(buf[off:off + n].cpu().numpy()) == f
        frames.append(f)
    # B200 frames into the reference receiver and vice versa.
    bad = bytearray(frames[1])
    bad[hdr + 3] ^= 0x01
    for layer, f in enumerate(frames):
        if layer == 1:
            a1, s1 = gD.ReceiveWriteFrame(bytes(bad))
            a2, s2 = rD.ReceiveWriteFrame(bytes(bad))
            assert (a1, s1) == (a2, s2) and s1 == -1 and DecodeFrame(a1)["status"] == 1
        a1, s1 = gD.ReceiveWriteFrame(f)
        a2, s2 = rD.ReceiveWriteFrame(f)
        assert (a1, s1) == (a2, s2) == (a1, int(ApplyStatus.Ok))
    # a replay is a duplicate (acked Ok, not re-applied)
    a1, s1 = gD.ReceiveWriteFrame(frames[0])
    assert (a1, s1) == rD.ReceiveWriteFrame(frames[0]) and s1 == int(ApplyStatus.Duplicate)
    assert gD.DrainReceiveCompletions() == rD.DrainReceiveCompletions() == [2]
    for layer in range(L):
        for pos in range(0, e, 7):
            assert np.array_equal(gD.ReadEntryWords(2, pos, layer), rD.ReadEntryWords(2, pos, layer))
            assert gD.FillOf(2, pos, layer) == rD.FillOf(2, pos, layer)


def test_receive_errors_match_reference(cuda, ref_lib):
    L, W, P = 2, 8, 16
    p = list(range(40))
    gP, gD, gr, m, e = _sender_pair({"device": 0}, L, W, P, p)
    rP, rD, rr, _, _ = _sender_pair({"lib": ref_lib}, L, W, P, p)
    f = gP.EncodeWriteFrame(20, (m, e), 0, 5, gr.addr)
    # unknown address: a receiver that never reserved these pages
    g2 = KVCache(num_pages=64, page_size=P, layers=L, dim=W, device=0)
    r2 = KVCache(num_pages=64, page_size=P, layers=L, dim=W, lib=ref_lib)
    a1, s1 = g2.ReceiveWriteFrame(f)
    assert (a1, s1) == r2.ReceiveWriteFrame(f) and s1 == int(ApplyStatus.UnknownAddress)
    assert DecodeFrame(a1)["status"] == 2
    # framing errors and ack frames are refused with the same status
    ack = bytes.fromhex(json.loads((GOLD / "frames.json").read_text())["acks"][0]["hex"])
    for bad in (f[:30], b"", ack, b"XXXX" + f[4:]):
        st = []
        for E in (gD, rD):
            with pytest.raises(SplitserveError) as ei:
                E.ReceiveWriteFrame(bad)
            st.append(ei.value.status)
        assert st[0] == st[1] == int(ErrorCode.InvalidArgument) + 1
    # address mismatch on encode (MarkSend's rule) on both
    for E, a in ((gP, gr.addr), (rP, rr.addr)):
        with pytest.raises(SplitserveError) as ei:
            E.EncodeWriteFrame(20, (m, e - 1), 0, 5, a)
        assert ei.value.code == ErrorCode.AddrMismatch
    # gather over an Empty slot (MissingKV, kv_cache.cc:379) on both
    for E in (gD, rD):
        a = E.BuildAddr(2, (m, e))
        with pytest.raises(SplitserveError) as ei:
            E.EncodeWriteFrame(2, (m, e), 0, 5, a)
        assert ei.value.code == ErrorCode.MissingKV
