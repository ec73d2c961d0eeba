"""TEST INFRASTRUCTURE ONLY — ctypes front of oracle/hashmodel.c, the C
restatement of the reference toy model (hash_model.h:11-20,
hash_model.cc:22-166).  Pinned against the compiled reference in
tests/test_oracle_pinning.py and tests/golden/.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
import this module.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "libhashoracle.so"
DEFAULT_HASH_SEED = 0x5EED5EED5EED5EED
_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            subprocess.run(["make", "-C", str(_HERE), "hash"], check=True, capture_output=True)
        L = C.CDLL(str(_LIB_PATH))
        u64, i32, i64 = C.c_uint64, C.c_int32, C.c_int64
        pu64, pi32 = C.POINTER(u64), C.POINTER(i32)
        sig = {
            "ho_mix64": (u64, [u64]),
            "ho_fnv_u64": (u64, [u64, u64]),
            "ho_fnv_u32": (u64, [u64, C.c_uint32]),
            "ho_seed_state": (u64, [u64]),
            "ho_initial_prefix_digest": (u64, [u64]),
            "ho_extend_prefix_digest": (u64, [u64, i32]),
            "ho_prefix_digests": (None, [u64, pi32, i64, pu64]),
            "ho_kv_entry_words": (None, [u64, i32, i32, pu64]),
            "ho_entry_digest": (u64, [pu64, i32]),
            "ho_embed": (u64, [u64, i32, i64]),
            "ho_query": (u64, [u64]),
            "ho_attention_out": (u64, [u64, i64, u64]),
            "ho_next_hidden": (u64, [u64, u64]),
            "ho_sample_token": (i32, [u64, i32]),
            "ho_kv_words_batch": (None, [pu64, i64, i32, i32, pu64]),
            "ho_entry_digest_batch": (None, [pu64, i64, i32, pu64]),
            "ho_generate": (C.c_int, [u64, i32, i32, i32, pi32, i64, i32, pi32]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype, fn.argtypes = res, args
        _lib = L
    return _lib


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(C.POINTER(t))


def mix64(z: int) -> int:
    return lib().ho_mix64(z)


def initial_prefix_digest(seed: int = DEFAULT_HASH_SEED) -> int:
    return lib().ho_initial_prefix_digest(seed)


def extend_prefix_digest(d: int, token: int) -> int:
    return lib().ho_extend_prefix_digest(d, token)


def prefix_digests(tokens, seed: int = DEFAULT_HASH_SEED) -> np.ndarray:
    """P(i) for every position i (digest after token i)."""
    t = np.ascontiguousarray(np.asarray(tokens, dtype=np.int32))
    out = np.zeros(len(t), dtype=np.uint64)
    if len(t):
        lib().ho_prefix_digests(seed, _p(t, C.c_int32), len(t), _p(out, C.c_uint64))
    return out


def kv_entry_words(prefix_digest: int, layer: int, dim: int) -> np.ndarray:
    out = np.zeros(dim, dtype=np.uint64)
    lib().ho_kv_entry_words(prefix_digest, layer, dim, _p(out, C.c_uint64))
    return out


def kv_words_batch(digests: np.ndarray, layer: int, dim: int) -> np.ndarray:
    d = np.ascontiguousarray(digests, dtype=np.uint64)
    out = np.zeros((len(d), dim), dtype=np.uint64)
    if len(d):
        lib().ho_kv_words_batch(_p(d, C.c_uint64), len(d), layer, dim, _p(out, C.c_uint64))
    return out


def entry_digest(words: np.ndarray) -> int:
    w = np.ascontiguousarray(words, dtype=np.uint64)
    return lib().ho_entry_digest(_p(w, C.c_uint64), len(w))


def entry_digest_batch(words: np.ndarray) -> np.ndarray:
    w = np.ascontiguousarray(words, dtype=np.uint64)
    out = np.zeros(w.shape[0], dtype=np.uint64)
    if w.shape[0]:
        lib().ho_entry_digest_batch(_p(w, C.c_uint64), w.shape[0], w.shape[1], _p(out, C.c_uint64))
    return out


def embed(token: int, pos: int, seed: int = DEFAULT_HASH_SEED) -> int:
    return lib().ho_embed(seed, token, pos)


def attention_out(hidden: int, count: int, fold_sum: int) -> int:
    return lib().ho_attention_out(hidden, count, fold_sum)


def next_hidden(hidden: int, attn_out: int) -> int:
    return lib().ho_next_hidden(hidden, attn_out)


def sample_token(last_hidden: int, vocab: int) -> int:
    return lib().ho_sample_token(last_hidden, vocab)


def generate(prompt, max_tokens: int, layers: int, dim: int, vocab: int = 256,
             seed: int = DEFAULT_HASH_SEED) -> list:
    """HashModel::Generate (hash_model.cc:130-166)."""
    t = np.ascontiguousarray(np.asarray(prompt, dtype=np.int32))
    out = np.zeros(max_tokens, dtype=np.int32)
    rc = lib().ho_generate(seed, layers, dim, vocab, _p(t, C.c_int32), len(t), max_tokens,
                           _p(out, C.c_int32))
    if rc != 0:
        raise ValueError("generate: empty prompt or max_tokens < 1")
    return [int(x) for x in out]
