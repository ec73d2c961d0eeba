"""Generates tests/golden/*.json from the compiled reference
(oracle/_ref/libmicrokv_ref.so = the unmodified splitserve::KVCache behind the
ABI).  Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

The fixtures pin the CPU restatement (oracle/) and the B200 product even
where the reference cannot be compiled (the GPU box).
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from flows import one_p_one_d  # noqa: E402
from scenarios import make_script, run_script  # noqa: E402

from paper_2412_12488_b200 import KVCache  # noqa: E402

REF = str(ROOT / "oracle" / "_ref" / "libmicrokv_ref.so")
OUT = Path(__file__).resolve().parent


def prompt(n, seed=1, vocab=256):
    rng = np.random.Generator(np.random.MT19937(seed))
    return [int(x) for x in rng.integers(0, vocab, n)]


def entries_digest(E, seq, n, layers):
    h = hashlib.sha256()
    for pos in range(n):
        for layer in range(layers):
            h.update(E.ReadEntryWords(seq, pos, layer).astype("<u8").tobytes())
    return h.hexdigest()


def tiny_1p1d():
    L, W, P = 4, 128, 16
    p = prompt(512)
    Pe = KVCache(num_pages=128, page_size=P, layers=L, dim=W, rank=0, lib=REF)
    D = KVCache(num_pages=128, page_size=P, layers=L, dim=W, rank=1, lib=REF)
    hiddens = []
    r = one_p_one_d(Pe, D, p, -1, via="sink", hiddens=hiddens, max_tokens=3)
    e = r["end"]
    rec = D.GetRecord(10)
    return {
        "config": {"layers": L, "dim": W, "page_size": P, "num_pages": 128, "prompt_len": 512,
                   "prompt_seed": 1, "end": -1},
        "prompt": p,
        "match_len": r["match_len"],
        "addr": {"token_begin": r["addr"].token_begin, "token_count": r["addr"].token_count,
                 "ranges": [list(x) for x in r["addr"].ranges]},
        "addr_json": r["addr"].ToJson(),
        "tokens": r["tokens"],
        "completions": r["done"],
        "p_hidden_last_layer": [str(int(x)) for x in hiddens[-1]],
        "p_hidden_layer0_first8": [str(int(x)) for x in hiddens[0][:8]],
        "d_own_pages": rec.own_pages,
        "d_committed": D.Committed(10),
        "d_entries_sha256": entries_digest(D, 10, len(p), L),
        "d_entry_pos0_layer0": [str(int(x)) for x in D.ReadEntryWords(10, 0, 0)],
        "d_entry_pos510_layer3": [str(int(x)) for x in D.ReadEntryWords(10, 510, 3)],
        "d_fill_pos0": [int(D.FillOf(10, 0, layer)) for layer in range(L)],
        "d_fill_pos511": [int(D.FillOf(10, 511, layer)) for layer in range(L)],
        "p_free_pages": Pe.FreePages(),
        "d_free_pages": D.FreePages(),
    }


def anchors():
    """SURVEY.md §8(c) anchors (default ModelConfig L=4, dim=8, V=256)."""
    E = KVCache(num_pages=8, page_size=16, layers=4, dim=8, lib=REF)
    E.CreateSequence(1, [1, 2, 3])
    E.EnsureAllocated(1, 3)
    from flows import prefill

    prefill(E, 1, [1, 2, 3], 0, 3)
    G = KVCache(num_pages=8, page_size=16, layers=4, dim=8, lib=REF)
    from flows import start_generate

    G.CreateSequence(2, [1, 2, 3])
    gen = start_generate(G, 2, [1, 2, 3], 0, 4)
    return {
        "initial_prefix_digest": str(E.InitialPrefixDigest()),
        "kv_entry_123_l0": [str(int(x)) for x in E.ReadEntryWords(1, 2, 0)],
        "generate_123_4": gen,
        "embed_5_7": str(E.Embed(5, 7)),
        "sample_token_of_12345": E.SampleToken(12345),
    }


def scripts():
    out = {}
    for seed in range(4):
        ops = make_script(seed, n_ops=80, data=True)
        c = KVCache(num_pages=24, page_size=4, layers=2, dim=8, lib=REF)
        log = run_script(c, ops)
        out[str(seed)] = json.loads(json.dumps(log, default=lambda o: list(o) if isinstance(o, tuple) else str(o)))
    return out


def frames():
    """Write frames the reference encodes (EncodeWriteFrame over
    GatherRange, transport.cc:46-62) for a 1P1D transfer into a forked
    receiver (fork-relative pages -> several ranges), the acks its TCP
    inbound step returns (tcp_fabric.cc:144-168), and CRC-32 check values."""
    import ctypes as C

    from flows import prefill

    L, W, P = 4, 8, 16
    p = prompt(40, seed=3)
    D = KVCache(num_pages=16, page_size=P, layers=L, dim=W, rank=1, lib=REF)
    D.CreateSequence(1, p[:5])
    D.EnsureAllocated(1, 5)
    prefill(D, 1, p, 0, 5)
    D.CommitToTree(1)
    r = D.PrepRecv(2, p, -1)
    m, e = r.match_len, r.match_len + r.addr.token_count
    Pe = KVCache(num_pages=16, page_size=P, layers=L, dim=W, rank=0, lib=REF)
    Pe.CreateSequence(20, p)
    Pe.EnsureAllocated(20, e)
    prefill(Pe, 20, p, 0, e)
    tag = 0x1234
    out = {"config": {"layers": L, "dim": W, "page_size": P, "num_pages": 16},
           "prompt": p, "match_len": m, "end": e, "tag": tag, "addr_json": r.addr.ToJson(),
           "frames": [], "acks": []}
    for layer in range(L):
        f = Pe.EncodeWriteFrame(20, (m, e), layer, tag, r.addr)
        ack, st = D.ReceiveWriteFrame(f)
        crc = int.from_bytes(f[-4:], "little")
        out["frames"].append({"layer": layer, "hex": f.hex(), "crc": crc, "ack_hex": ack.hex(),
                              "apply_status": st})
    bad = bytearray(bytes.fromhex(out["frames"][0]["hex"]))
    flip = 41 + 8 * len(r.addr.ranges) + 10  # inside the payload
    bad[flip] ^= 0x40
    ack, st = D.ReceiveWriteFrame(bytes(bad))
    out["corrupt_frame0"] = {"flip_byte": flip, "ack_hex": ack.hex(), "apply_status": st}
    out["completions"] = D.DrainReceiveCompletions()
    from paper_2412_12488_b200.kvcache import EncodeAckFrame, load_library
    lib = load_library(REF)
    for args in ((0x1234, 2, 5, 0), (7, 79, 6553, 1), (1, 0, 0, 2)):
        out["acks"].append({"args": list(args), "hex": EncodeAckFrame(*args, lib=lib).hex()})
    lib.ssref_crc32.restype = C.c_uint32
    lib.ssref_crc32.argtypes = [C.c_char_p, C.c_int64]
    kat = {"123456789": lib.ssref_crc32(b"123456789", 9)}
    rng = np.random.Generator(np.random.MT19937(11))
    for n in (0, 1, 31, 32, 33, 1000, 4096, 65549):
        buf = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        kat[f"mt19937_11_{n}"] = lib.ssref_crc32(buf, n)
    out["crc32"] = kat
    return out


if __name__ == "__main__":
    (OUT / "frames.json").write_text(json.dumps(frames(), indent=1))
    (OUT / "tiny_1p1d.json").write_text(json.dumps(tiny_1p1d(), indent=1))
    (OUT / "anchors.json").write_text(json.dumps(anchors(), indent=1))
    (OUT / "scripts.json").write_text(json.dumps(scripts()))
    print("wrote", sorted(p.name for p in OUT.glob("*.json")))
