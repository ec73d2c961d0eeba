"""Python mirror of ``splitserve::KVCache`` over the C ABI (include/microkv.h).

Method names, argument meaning and error behaviour follow the reference
class (/root/reference/proj/core/include/splitserve/kv_cache.h:132-235):
errors raise :class:`SplitserveError` carrying the reference ``ErrorCode``
(errors.h:14-33).  The same class drives either library that implements the
ABI: the B200 product (``paper_2412_12488_b200/_lib/libmicrokv.so``, the
default) or, in tests only, the reference compiled behind the ABI
(``oracle/_ref/libmicrokv_ref.so``).

There is no CPU fallback: if the product library is missing this module
raises on import of :func:`load_library`; data-path calls on a cache without
a device raise ``SplitserveError(NoDevice)``.
"""
from __future__ import annotations

import ctypes as C
import enum
import json
import os
import weakref
from dataclasses import dataclass, field
from pathlib import Path
from typing import Callable, Iterable, Optional, Sequence

import numpy as np

_HERE = Path(__file__).resolve().parent
PRODUCT_LIB = _HERE / "_lib" / "libmicrokv.so"

DEFAULT_HASH_SEED = 0x5EED5EED5EED5EED  # config.h:26


class ErrorCode(enum.IntEnum):
    """splitserve::ErrorCode (errors.h:14-33)."""

    OutOfPages = 0
    DuplicateSequence = 1
    UnknownSequence = 2
    ForkBeyondCommitted = 3
    AddrMismatch = 4
    MissingKV = 5
    LayerOrderViolation = 6
    CannotEvict = 7
    ChecksumMismatch = 8
    UnknownAddress = 9
    PeerUnreachable = 10
    NoEngines = 11
    RoleMissing = 12
    NoOwner = 13
    UnknownStrategy = 14
    InvalidArgument = 15
    Aborted = 16
    Internal = 17


class FillState(enum.IntEnum):
    """FillState (kv_cache.h:40-44)."""

    Empty = 0
    ComputedLocal = 1
    ReceivedRemote = 2


class ApplyStatus(enum.IntEnum):
    """KVCache::ApplyStatus (kv_cache.h:194)."""

    Ok = 0
    Duplicate = 1
    UnknownAddress = 2


SS_OK = 0
SS_ERR_UNSUPPORTED = 100
SS_ERR_BUFFER_TOO_SMALL = 101
SS_ERR_CUDA = 102
SS_ERR_NO_DEVICE = 103
_BOUNDARY_NAMES = {100: "Unsupported", 101: "BufferTooSmall", 102: "Cuda", 103: "NoDevice"}


class SplitserveError(RuntimeError):
    """splitserve::Error: {code, retryable, detail} (errors.h:38-50)."""

    def __init__(self, status: int, detail: str):
        self.status = status
        self.code: Optional[ErrorCode] = ErrorCode(status - 1) if 1 <= status <= 18 else None
        name = self.code.name if self.code is not None else _BOUNDARY_NAMES.get(status, "Unknown")
        self.name = name
        super().__init__(detail or name)

    @property
    def retryable(self) -> bool:  # IsRetryable, event_log.cc:35-43
        return self.code in (ErrorCode.OutOfPages, ErrorCode.PeerUnreachable)


# ---------------------------------------------------------------------------
# ctypes mirrors of the header structs
# ---------------------------------------------------------------------------
class _Config(C.Structure):
    _fields_ = [("num_pages", C.c_int64), ("page_size", C.c_int32), ("layers", C.c_int32),
                ("dim", C.c_int32), ("vocab", C.c_int32), ("hash_seed", C.c_uint64),
                ("device", C.c_int32), ("rank", C.c_int32)]


class _SlotRange(C.Structure):
    _fields_ = [("page_id", C.c_int64), ("slot_begin", C.c_int32), ("slot_count", C.c_int32)]


class _Addr(C.Structure):
    _fields_ = [("token_begin", C.c_int64), ("token_count", C.c_int64), ("n_ranges", C.c_int64),
                ("ranges", C.POINTER(_SlotRange)), ("ranges_cap", C.c_int64)]


class _Batch(C.Structure):
    _fields_ = [("seq", C.c_int64), ("begin", C.c_int64), ("end", C.c_int64),
                ("is_decode", C.c_int32), ("_pad", C.c_int32)]


class _RecordInfo(C.Structure):
    _fields_ = [("id", C.c_int64), ("parent", C.c_int64), ("fork_len", C.c_int64),
                ("refcount", C.c_int32), ("finished", C.c_int32), ("alloc_len", C.c_int64),
                ("committed_hint", C.c_int64), ("num_tokens", C.c_int64),
                ("num_own_pages", C.c_int64), ("fold_frontier", C.c_int64),
                ("digest_len", C.c_int64), ("prefix_digest", C.c_uint64),
                ("has_window", C.c_int32), ("window_complete", C.c_int32),
                ("window_begin", C.c_int64), ("window_end", C.c_int64),
                ("window_expected_writes", C.c_int64), ("window_received_writes", C.c_int64)]


class IpcHandle(C.Structure):
    _fields_ = [("bytes", C.c_uint8 * 512)]


class _FrameInfo(C.Structure):  # ss_frame_info (microkv.h)
    _fields_ = [("type", C.c_int32), ("layer", C.c_int32), ("seq_tag", C.c_uint64),
                ("addr", _Addr), ("payload_offset", C.c_int64), ("payload_bytes", C.c_int64),
                ("wire_crc", C.c_uint32), ("ack_status", C.c_int32), ("token_begin", C.c_int64)]


_SINK = C.CFUNCTYPE(None, C.c_void_p, C.c_int32, C.c_int64, C.c_int64, C.c_int64, C.c_int32,
                    C.POINTER(_Addr), C.c_uint64, C.POINTER(C.c_uint64), C.c_int64)

_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_u64p = C.POINTER(C.c_uint64)
_vp = C.c_void_p

_SIGNATURES = {
    "ss_abi_version": (C.c_int, []),
    "ss_impl_name": (C.c_char_p, []),
    "ss_cache_create": (C.c_int, [C.POINTER(_Config), C.POINTER(_vp)]),
    "ss_cache_destroy": (None, [_vp]),
    "ss_last_error": (C.c_char_p, [_vp]),
    "ss_status_name": (C.c_char_p, [C.c_int]),
    "ss_status_retryable": (C.c_int, [C.c_int]),
    "ss_initial_prefix_digest": (C.c_uint64, [_vp]),
    "ss_embed": (C.c_uint64, [_vp, C.c_int32, C.c_int64]),
    "ss_sample_token": (C.c_int32, [_vp, C.c_uint64]),
    "ss_match_prefix": (C.c_int, [_vp, _i32p, C.c_int64, _i64p, _i64p]),
    "ss_prep_recv": (C.c_int, [_vp, C.c_int64, _i32p, C.c_int64, C.c_int64, _i64p,
                               C.POINTER(_Addr)]),
    "ss_create_sequence": (C.c_int, [_vp, C.c_int64, _i32p, C.c_int64]),
    "ss_fork_sequence": (C.c_int, [_vp, C.c_int64, C.c_int64, C.c_int64, _i32p, C.c_int64]),
    "ss_mark_send": (C.c_int, [_vp, C.c_int64, C.c_int64, C.c_int64, C.c_int32,
                               C.POINTER(_Addr), C.c_uint64]),
    "ss_ensure_allocated": (C.c_int, [_vp, C.c_int64, C.c_int64]),
    "ss_append_token": (C.c_int, [_vp, C.c_int64, C.c_int32]),
    "ss_begin_forward": (C.c_int, [_vp, C.POINTER(_Batch), C.c_int64, C.POINTER(_vp)]),
    "ss_plan_total_outputs": (C.c_int64, [_vp]),
    "ss_plan_num_sends": (C.c_int64, [_vp]),
    "ss_plan_next_layer": (C.c_int32, [_vp]),
    "ss_plan_destroy": (None, [_vp]),
    "ss_attention": (C.c_int, [_vp, _vp, C.c_int32, _u64p, _u64p, C.c_int64, _SINK, _vp]),
    "ss_gather_range": (C.c_int, [_vp, C.c_int64, C.c_int64, C.c_int64, C.c_int32, _u64p,
                                  C.c_int64]),
    "ss_build_addr": (C.c_int, [_vp, C.c_int64, C.c_int64, C.c_int64, C.POINTER(_Addr)]),
    "ss_apply_remote_write": (C.c_int, [_vp, C.POINTER(_Addr), C.c_int32, _u64p, C.c_int64,
                                        C.c_uint64, _i32p]),
    "ss_drain_receive_completions": (C.c_int, [_vp, _i64p, C.c_int64, _i64p]),
    "ss_set_finished": (C.c_int, [_vp, C.c_int64, C.c_int32]),
    "ss_commit_to_tree": (C.c_int, [_vp, C.c_int64]),
    "ss_free_sequence": (C.c_int, [_vp, C.c_int64]),
    "ss_evict": (C.c_int, [_vp, C.c_int64, _i64p]),
    "ss_pin": (C.c_int, [_vp, _i32p, C.c_int64, C.c_int32]),
    "ss_has_sequence": (C.c_int, [_vp, C.c_int64]),
    "ss_get_record": (C.c_int, [_vp, C.c_int64, C.POINTER(_RecordInfo), _i64p, C.c_int64]),
    "ss_committed": (C.c_int, [_vp, C.c_int64, _i64p]),
    "ss_read_entry_words": (C.c_int, [_vp, C.c_int64, C.c_int64, C.c_int32, _u64p, C.c_int64]),
    "ss_fill_of": (C.c_int, [_vp, C.c_int64, C.c_int64, C.c_int32, _i32p]),
    "ss_free_pages": (C.c_int64, [_vp]),
    "ss_total_pages": (C.c_int64, [_vp]),
    "ss_cache_config": (C.c_int, [_vp, C.POINTER(_Config)]),
    "ss_bytes_per_page": (C.c_int64, [_vp]),
    "ss_sequence_count": (C.c_int64, [_vp]),
    "ss_sequence_ids": (C.c_int, [_vp, _i64p, C.c_int64, _i64p]),
    "ss_pending_send_count": (C.c_int64, [_vp]),
    "ss_tree_node_count": (C.c_int64, [_vp]),
    "ss_tree_contains": (C.c_int, [_vp, C.c_int64]),
    "ss_tree_last_touch": (C.c_uint64, [_vp, C.c_int64]),
    "ss_tree_sequences_by_lru": (C.c_int, [_vp, _i64p, C.c_int64, _i64p]),
    "ss_addr_validate": (C.c_int, [C.POINTER(_Addr)]),
    "ss_addr_slice": (C.c_int, [C.POINTER(_Addr), C.c_int64, C.c_int64, C.POINTER(_Addr)]),
    "ss_device": (C.c_int, [_vp]),
    "ss_attach_peer": (C.c_int, [_vp, C.c_int32, _vp]),
    "ss_export_ipc": (C.c_int, [_vp, C.POINTER(IpcHandle)]),
    "ss_import_ipc": (C.c_int, [_vp, C.c_int32, C.POINTER(IpcHandle)]),
    "ss_detach_peer": (C.c_int, [_vp, C.c_int32]),
    "ss_peer_info": (C.c_int, [_vp, C.c_int32, _i32p, _i32p]),
    "ss_attention_async": (C.c_int, [_vp, _vp, C.c_int32, _vp, _vp, _vp]),
    "ss_direct_send_async": (C.c_int, [_vp, C.c_int64, C.c_int64, C.c_int64, C.c_int32,
                                       C.POINTER(_Addr), C.c_uint64, C.c_int32, C.c_int32, _vp]),
    "ss_begin_direct_send": (C.c_int, [_vp, C.c_int64, C.c_int64, C.c_int64, C.c_int32,
                                       C.POINTER(_Addr), C.c_uint64, C.POINTER(_vp)]),
    "ss_launch_direct_send_async": (C.c_int, [_vp, _vp, C.c_int32, C.c_int32, _vp]),
    "ss_launch_direct_send_after_async": (C.c_int, [_vp, _vp, C.c_int32, C.c_int32, _vp, _vp]),
    "ss_set_send_mode": (C.c_int, [_vp, C.c_int32, C.c_int32]),
    "ss_launch_relay_send_async": (C.c_int, [_vp, _vp, C.c_int32, C.c_int32, C.c_int64, _vp]),
    "ss_broadcast_send_async": (C.c_int, [_vp, C.c_int64, C.c_int64, C.c_int64, C.c_int32, _i32p,
                                          C.POINTER(_Addr), C.c_uint64, C.c_int32, C.c_int32, _vp]),
    "ss_gather_range_async": (C.c_int, [_vp, C.c_int64, C.c_int64, C.c_int64, C.c_int32, _vp,
                                        _vp]),
    "ss_gather_range_layers_async": (C.c_int, [_vp, C.c_int64, C.c_int64, C.c_int64, C.c_int32,
                                               C.c_int32, _vp, _vp]),
    "ss_apply_remote_write_async": (C.c_int, [_vp, C.POINTER(_Addr), C.c_int32, _vp, C.c_int64,
                                              C.c_uint64, _i32p, _vp]),
    "ss_append_rows_async": (C.c_int, [_vp, _vp, C.c_int32, _vp, _vp]),
    "ss_append_rows_layers_async": (C.c_int, [_vp, _vp, C.c_int32, C.c_int32, _vp, _vp]),
    "ss_append_rows_send_async": (C.c_int, [_vp, _vp, _vp, C.c_int32, C.c_int32, _vp, _vp]),
    "ss_begin_decode": (C.c_int, [_vp, _i64p, _i64p, C.c_int64, C.POINTER(_vp)]),
    "ss_paged_decode_attention_async": (C.c_int, [_vp, _vp, C.c_int32, C.c_int32, C.c_int32,
                                                  C.c_int32, C.c_float, _vp, _vp, _vp]),
    "ss_paged_prefill_attention_async": (C.c_int, [_vp, C.c_int64, C.c_int64, C.c_int64,
                                                   C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                                   C.c_float, _vp, _vp, _vp]),
    "ss_pool_layer_ptr": (C.c_int, [_vp, C.c_int32, C.POINTER(_vp)]),
    "ss_wait_receive_async": (C.c_int, [_vp, C.c_int64, C.c_int64, _vp]),
    "ss_wait_receive_layer_async": (C.c_int, [_vp, C.c_int64, C.c_int32, C.c_int64, _vp]),
    "ss_copy_counters": (C.c_int, [_vp, _i64p, _i64p]),
    "ss_kernel_launches": (C.c_int64, [_vp]),
    "ss_synchronize": (C.c_int, [_vp]),
    "ss_addr_encode": (C.c_int, [C.POINTER(_Addr), _vp, C.c_int64, _i64p]),
    "ss_addr_decode": (C.c_int, [_vp, C.c_int64, _i64p, C.POINTER(_Addr)]),
    "ss_addr_to_json": (C.c_int, [C.POINTER(_Addr), C.c_char_p, C.c_int64, _i64p]),
    "ss_addr_from_json": (C.c_int, [C.c_char_p, C.c_int64, C.POINTER(_Addr)]),
    "ss_frame_write_header_size": (C.c_int64, [C.c_int64]),
    "ss_frame_encode_ack": (C.c_int, [C.c_uint64, C.c_int32, C.c_int64, C.c_int32, _vp,
                                      C.c_int64, _i64p]),
    "ss_frame_decode": (C.c_int, [_vp, C.c_int64, C.POINTER(_FrameInfo)]),
    "ss_crc32_async": (C.c_int, [_vp, _vp, C.c_int64, _vp, _vp]),
    "ss_encode_write_frame": (C.c_int, [_vp, C.c_int64, C.c_int64, C.c_int64, C.c_int32,
                                        C.c_uint64, C.POINTER(_Addr), _vp, C.c_int64, _i64p]),
    "ss_encode_write_frame_async": (C.c_int, [_vp, C.c_int64, C.c_int64, C.c_int64, C.c_int32,
                                              C.c_uint64, C.POINTER(_Addr), _vp, C.c_int64,
                                              _i64p, _vp]),
    "ss_receive_write_frame": (C.c_int, [_vp, _vp, C.c_int64, _vp, _i32p]),
}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)

_LIBS: dict[str, C.CDLL] = {}


def load_library(path: Optional[os.PathLike | str] = None) -> C.CDLL:
    """Loads (once) a library implementing include/microkv.h.

    ``path=None`` loads the B200 product library and raises if it has not
    been built — there is no fallback implementation.
    """
    p = Path(path) if path is not None else PRODUCT_LIB
    key = str(p.resolve())
    if key in _LIBS:
        return _LIBS[key]
    if not p.exists():
        raise FileNotFoundError(
            f"{p} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (no CPU fallback exists)")
    lib = C.CDLL(str(p))
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.ss_abi_version() != 1:
        raise RuntimeError(f"{p}: unexpected ABI version {lib.ss_abi_version()}")
    _LIBS[key] = lib
    return lib


def _tok(tokens: Iterable[int]) -> np.ndarray:
    if isinstance(tokens, np.ndarray) and tokens.dtype == np.int32 and tokens.flags.c_contiguous:
        return tokens
    if isinstance(tokens, np.ndarray):
        return np.ascontiguousarray(tokens, dtype=np.int32)
    return np.fromiter(tokens, dtype=np.int32) if not isinstance(tokens, (list, tuple)) else \
        np.array(tokens, dtype=np.int32)


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


# ---------------------------------------------------------------------------
# Plain-data types
# ---------------------------------------------------------------------------
SLOT_RANGE_DTYPE = np.dtype([("page_id", "<i8"), ("slot_begin", "<i4"), ("slot_count", "<i4")])
assert SLOT_RANGE_DTYPE.itemsize == C.sizeof(_SlotRange)


class KVAddrInfo:
    """KVAddrInfo (kv_addr.h:30-48): run-length (page_id, slot_begin, slot_count).

    The ranges live in a numpy array laid out like ``ss_slot_range`` so an
    address returned by prep_recv goes back into mark_send / direct_send
    without per-range Python work; ``ranges`` gives the tuples."""

    __slots__ = ("_arr", "token_begin", "token_count", "_list")

    def __init__(self, ranges=(), token_begin: int = 0, token_count: int = 0):
        if isinstance(ranges, np.ndarray) and ranges.dtype == SLOT_RANGE_DTYPE:
            self._arr = np.ascontiguousarray(ranges)
        else:
            rl = [tuple(int(v) for v in r) for r in ranges]
            self._arr = np.array(rl, dtype=SLOT_RANGE_DTYPE) if rl else np.zeros(0, SLOT_RANGE_DTYPE)
        self.token_begin = int(token_begin)
        self.token_count = int(token_count)
        self._list = None

    @property
    def ranges(self) -> list:
        if self._list is None:
            self._list = [(int(p), int(b), int(c)) for p, b, c in self._arr.tolist()]
        return self._list

    @property
    def array(self) -> np.ndarray:
        return self._arr

    def __eq__(self, other) -> bool:
        return (isinstance(other, KVAddrInfo) and self.token_begin == other.token_begin
                and self.token_count == other.token_count
                and np.array_equal(self._arr, other._arr))

    def __repr__(self) -> str:
        return (f"KVAddrInfo(ranges={self.ranges}, token_begin={self.token_begin}, "
                f"token_count={self.token_count})")

    def __getstate__(self):
        return (self._arr, self.token_begin, self.token_count)

    def __setstate__(self, st):
        self._arr, self.token_begin, self.token_count = st
        self._list = None

    def _c(self) -> tuple[_Addr, object]:
        arr = self._arr if len(self._arr) else np.zeros(1, SLOT_RANGE_DTYPE)
        a = _Addr(self.token_begin, self.token_count, len(self._arr),
                  arr.ctypes.data_as(C.POINTER(_SlotRange)), len(self._arr))
        return a, arr

    @staticmethod
    def _from_c(a: _Addr) -> "KVAddrInfo":
        n = int(a.n_ranges)
        if n:
            raw = C.string_at(a.ranges, n * SLOT_RANGE_DTYPE.itemsize)
            arr = np.frombuffer(raw, dtype=SLOT_RANGE_DTYPE).copy()
        else:
            arr = np.zeros(0, SLOT_RANGE_DTYPE)
        return KVAddrInfo(arr, a.token_begin, a.token_count)

    def Validate(self, lib: Optional[C.CDLL] = None) -> None:  # kv_addr.cc:16-30
        lib = lib or load_library()
        a, keep = self._c()
        st = lib.ss_addr_validate(C.byref(a))
        if st != SS_OK:
            raise SplitserveError(st, "KVAddrInfo.Validate")

    def Slice(self, begin: int, end: int, lib: Optional[C.CDLL] = None) -> "KVAddrInfo":
        lib = lib or load_library()  # kv_addr.cc:32-51
        a, keep = self._c()
        cap = max(1, len(self._arr))
        out_arr = (_SlotRange * cap)()
        out = _Addr(0, 0, 0, out_arr, cap)
        st = lib.ss_addr_slice(C.byref(a), begin, end, C.byref(out))
        if st != SS_OK:
            raise SplitserveError(st, "KVAddrInfo.Slice")
        return KVAddrInfo._from_c(out)

    def ToJson(self, lib: Optional[C.CDLL] = None) -> str:  # kv_addr.cc:53-58
        lib = lib or load_library()
        a, keep = self._c()
        n = C.c_int64(0)
        buf = C.create_string_buffer(64 + 40 * len(self._arr))
        st = lib.ss_addr_to_json(C.byref(a), buf, len(buf), C.byref(n))
        if st != SS_OK:
            raise SplitserveError(st, "KVAddrInfo.ToJson")
        return buf.raw[:n.value].decode()

    @staticmethod
    def FromJson(text: str, lib: Optional[C.CDLL] = None) -> "KVAddrInfo":  # kv_addr.cc:60-70
        lib = lib or load_library()
        raw = text.encode()
        return KVAddrInfo._decoded(lambda out: lib.ss_addr_from_json(raw, len(raw), out),
                                   max(1, len(raw) // 6), "KVAddrInfo.FromJson")

    def EncodeTo(self, lib: Optional[C.CDLL] = None) -> bytes:  # kv_addr.cc:90-99
        lib = lib or load_library()
        a, keep = self._c()
        n = C.c_int64(0)
        buf = (C.c_uint8 * (20 + 8 * len(self._arr)))()
        st = lib.ss_addr_encode(C.byref(a), buf, len(buf), C.byref(n))
        if st != SS_OK:
            raise SplitserveError(st, "KVAddrInfo.EncodeTo")
        return bytes(buf)[:n.value]

    @staticmethod
    def DecodeFrom(data: bytes, pos: int = 0,
                   lib: Optional[C.CDLL] = None) -> tuple["KVAddrInfo", int]:  # kv_addr.cc:101-118
        lib = lib or load_library()
        p = C.c_int64(pos)
        addr = KVAddrInfo._decoded(lambda out: lib.ss_addr_decode(data, len(data), C.byref(p), out),
                                   max(1, (len(data) - pos) // 8), "KVAddrInfo.DecodeFrom")
        return addr, p.value

    @staticmethod
    def _decoded(call, cap: int, what: str) -> "KVAddrInfo":
        arr = (_SlotRange * cap)()
        out = _Addr(0, 0, 0, arr, cap)
        st = call(C.byref(out))
        if st == SS_ERR_BUFFER_TOO_SMALL:
            arr = (_SlotRange * int(out.n_ranges))()
            out = _Addr(0, 0, 0, arr, int(out.n_ranges))
            st = call(C.byref(out))
        if st != SS_OK:
            raise SplitserveError(st, what)
        return KVAddrInfo._from_c(out)

    def slots(self, page_size: int) -> np.ndarray:
        """Flat slot indices (page * page_size + slot) in token order."""
        out = [p * page_size + b + k for (p, b, c) in self.ranges for k in range(c)]
        return np.asarray(out, dtype=np.int64)


def frame_write_header_size(n_ranges: int, lib: Optional[C.CDLL] = None) -> int:
    """Bytes of a write frame before its payload (transport.h:6-12)."""
    return int((lib or load_library()).ss_frame_write_header_size(n_ranges))


def EncodeAckFrame(seq_tag: int, layer: int, token_begin: int, status: int,
                   lib: Optional[C.CDLL] = None) -> bytes:  # transport.cc:64-74
    lib = lib or load_library()
    out = (C.c_uint8 * 26)()
    n = C.c_int64(0)
    st = lib.ss_frame_encode_ack(seq_tag, layer, token_begin, status, out, 26, C.byref(n))
    if st != SS_OK:
        raise SplitserveError(st, "EncodeAckFrame")
    return bytes(out)[:n.value]


def DecodeFrame(frame: bytes, lib: Optional[C.CDLL] = None) -> dict:
    """DecodeFrame (transport.cc:76-107) without the payload copy and CRC:
    type, seq_tag, layer and, for writes, addr / payload_offset /
    payload_bytes / wire_crc; for acks token_begin / status."""
    lib = lib or load_library()
    cap = max(1, len(frame) // 8)
    arr = (_SlotRange * cap)()
    info = _FrameInfo()
    info.addr = _Addr(0, 0, 0, arr, cap)
    st = lib.ss_frame_decode(frame, len(frame), C.byref(info))
    if st != SS_OK:
        raise SplitserveError(st, "DecodeFrame")
    out = {"type": int(info.type), "seq_tag": int(info.seq_tag), "layer": int(info.layer)}
    if info.type == 0:
        out.update(addr=KVAddrInfo._from_c(info.addr), payload_offset=int(info.payload_offset),
                   payload_bytes=int(info.payload_bytes), wire_crc=int(info.wire_crc))
    else:
        out.update(token_begin=int(info.token_begin), status=int(info.ack_status))
    return out


@dataclass
class PrepRecvResult:
    match_len: int
    addr: KVAddrInfo


@dataclass
class BatchEntry:
    """BatchEntry (kv_cache.h:85-89); range is (begin, end)."""

    seq: int
    range: tuple
    is_decode: bool = False


@dataclass
class SequenceRecordInfo:
    id: int
    parent: int
    fork_len: int
    refcount: int
    finished: bool
    alloc_len: int
    committed_hint: int
    num_tokens: int
    own_pages: list
    fold_frontier: int
    digest_len: int
    prefix_digest: int
    window: Optional[dict]


class ForwardPlan:
    """Handle of a ForwardPlan (kv_cache.h:116-121); destroyed with the object."""

    def __init__(self, cache: "KVCache", handle: int):
        self._cache = cache
        self._h = C.c_void_p(handle)
        cache._plans.add(self)

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    @property
    def total_outputs(self) -> int:
        return self._cache._lib.ss_plan_total_outputs(self._h)

    @property
    def num_sends(self) -> int:
        return self._cache._lib.ss_plan_num_sends(self._h)

    @property
    def next_layer(self) -> int:
        return self._cache._lib.ss_plan_next_layer(self._h)

    def close(self) -> None:
        # A plan whose cache is already gone was released with the cache.
        if self._h and self._h.value and self._cache._h and self._cache._h.value:
            self._cache._lib.ss_plan_destroy(self._h)
        self._h = C.c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


FrameSink = Callable[[int, dict, np.ndarray], None]


# ---------------------------------------------------------------------------
# KVCache
# ---------------------------------------------------------------------------
class KVCache:
    """One engine's paged KV cache (kv_cache.h:132-266).

    ``device=None`` picks CUDA device 0 for the product library; ``device=-1``
    builds a host-only cache (bookkeeping only).  ``lib`` selects the ABI
    implementation (defaults to the B200 product library).
    """

    def __init__(self, num_pages: int = 4096, page_size: int = 16, layers: int = 4, dim: int = 8,
                 vocab: int = 256, hash_seed: int = DEFAULT_HASH_SEED, device: Optional[int] = 0,
                 rank: int = 0, lib: Optional[C.CDLL | str | os.PathLike] = None):
        self._h = C.c_void_p(0)
        self._plans = weakref.WeakSet()
        self._lib = lib if isinstance(lib, C.CDLL) else load_library(lib)
        cfg = _Config(num_pages, page_size, layers, dim, vocab, hash_seed & (2**64 - 1),
                      -1 if device is None else device, rank)
        h = C.c_void_p()
        st = self._lib.ss_cache_create(C.byref(cfg), C.byref(h))
        if st != SS_OK:
            raise SplitserveError(st, f"KVCache construction failed ({self._status_name(st)})")
        self._h = h
        self.num_pages, self.page_size, self.layers, self.dim = num_pages, page_size, layers, dim
        self.vocab, self.hash_seed, self.rank = vocab, hash_seed, rank
        self.device = self._lib.ss_device(self._h)
        self._keep = []
        self._plans = weakref.WeakSet()

    # -- plumbing ---------------------------------------------------------
    def _status_name(self, st: int) -> str:
        return self._lib.ss_status_name(st).decode()

    def _check(self, st: int) -> None:
        if st != SS_OK:
            msg = self._lib.ss_last_error(self._h).decode(errors="replace")
            raise SplitserveError(st, msg)

    @property
    def impl(self) -> str:
        return self._lib.ss_impl_name().decode()

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            # Live plans are released by the library with the cache; make their
            # handles inert first so a later finalizer cannot touch them.
            for plan in list(getattr(self, "_plans", ())):
                plan._h = C.c_void_p(0)
            self._lib.ss_cache_destroy(self._h)
            self._h = C.c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _addr_out(self, cap: int) -> tuple[_Addr, np.ndarray]:
        """Reusable output address buffer (structured numpy allocation and
        ctypes pointer construction cost more than the C++ call itself)."""
        buf = self.__dict__.get("_obuf")
        if buf is None or len(buf) < cap:
            buf = np.empty(max(cap, 1024), dtype=SLOT_RANGE_DTYPE)
            self._obuf = buf
            self._oaddr = _Addr(0, 0, 0, buf.ctypes.data_as(C.POINTER(_SlotRange)), len(buf))
        a = self._oaddr
        a.token_begin = a.token_count = a.n_ranges = 0
        return a, buf

    @staticmethod
    def _addr_in(a: _Addr, arr: np.ndarray) -> "KVAddrInfo":
        n = int(a.n_ranges)
        raw = arr.view(np.uint8)[:n * SLOT_RANGE_DTYPE.itemsize].copy()
        return KVAddrInfo(raw.view(SLOT_RANGE_DTYPE), a.token_begin, a.token_count)

    # -- hash model scalars (hash_model.cc) --------------------------------
    def InitialPrefixDigest(self) -> int:
        return self._lib.ss_initial_prefix_digest(self._h)

    def Embed(self, token: int, pos: int) -> int:
        return self._lib.ss_embed(self._h, token, pos)

    def SampleToken(self, last_hidden: int) -> int:
        return self._lib.ss_sample_token(self._h, C.c_uint64(last_hidden & (2**64 - 1)))

    # -- declaration stage --------------------------------------------------
    def MatchPrefixSeq(self, tokens) -> tuple[int, int]:
        t = _tok(tokens)
        m, s = C.c_int64(), C.c_int64()
        self._check(self._lib.ss_match_prefix(self._h, _ptr(t, C.c_int32), len(t), C.byref(m),
                                              C.byref(s)))
        return m.value, s.value

    def MatchPrefix(self, tokens) -> int:
        return self.MatchPrefixSeq(tokens)[0]

    def PrepRecv(self, seq_id: int, tokens, end: int) -> PrepRecvResult:
        t = _tok(tokens)
        cap = (len(t) + self.page_size - 1) // self.page_size + 1
        a, keep = self._addr_out(cap)
        m = C.c_int64()
        self._check(self._lib.ss_prep_recv(self._h, seq_id, _ptr(t, C.c_int32), len(t), end,
                                           C.byref(m), C.byref(a)))
        return PrepRecvResult(m.value, self._addr_in(a, keep))

    def ForkSequence(self, parent: int, child: int, fork_len: int, child_tokens=()) -> None:
        t = _tok(child_tokens)
        self._check(self._lib.ss_fork_sequence(self._h, parent, child, fork_len,
                                               _ptr(t, C.c_int32), len(t)))

    def CreateSequence(self, seq_id: int, tokens) -> None:
        t = _tok(tokens)
        self._check(self._lib.ss_create_sequence(self._h, seq_id, _ptr(t, C.c_int32), len(t)))

    def MarkSend(self, seq: int, range: tuple, dest: int, dest_addr: KVAddrInfo,
                 user_tag: int = 0) -> None:
        a, keep = dest_addr._c()
        self._check(self._lib.ss_mark_send(self._h, seq, range[0], range[1], dest, C.byref(a),
                                           user_tag))

    def EnsureAllocated(self, seq: int, upto: int) -> None:
        self._check(self._lib.ss_ensure_allocated(self._h, seq, upto))

    def AppendToken(self, seq: int, t: int) -> None:
        self._check(self._lib.ss_append_token(self._h, seq, t))

    def BeginForward(self, batch: Sequence[BatchEntry]) -> ForwardPlan:
        arr = (_Batch * max(1, len(batch)))()
        for i, e in enumerate(batch):
            arr[i].seq, arr[i].begin, arr[i].end = e.seq, e.range[0], e.range[1]
            arr[i].is_decode = 1 if e.is_decode else 0
        h = C.c_void_p()
        self._check(self._lib.ss_begin_forward(self._h, arr, len(batch), C.byref(h)))
        return ForwardPlan(self, h.value)

    # -- computation stage ----------------------------------------------------
    def Attention(self, layer: int, plan: ForwardPlan, hidden_in,
                  sink: Optional[FrameSink] = None) -> np.ndarray:
        """kv_cache.cc:308-371.  ``sink(layer, send, payload)`` gets a dict with
        the PlanSend fields and a uint64 payload copy."""
        hin = np.ascontiguousarray(np.asarray(hidden_in, dtype=np.uint64))
        hout = np.zeros_like(hin)
        errors: list = []

        def _cb(user, lyr, seq, rb, re, dest, addr_p, tag, payload, n_words):
            try:
                send = {"seq": seq, "range": (rb, re), "dest": dest,
                        "dest_addr": KVAddrInfo._from_c(addr_p.contents), "user_tag": tag}
                buf = np.ctypeslib.as_array(payload, shape=(n_words,)).copy() if n_words else \
                    np.zeros(0, np.uint64)
                sink(lyr, send, buf)
            except Exception as ex:  # surfaced after the call returns
                errors.append(ex)

        cb = _SINK(_cb) if sink is not None else _SINK()
        st = self._lib.ss_attention(self._h, plan.handle, layer, _ptr(hin, C.c_uint64),
                                    _ptr(hout, C.c_uint64), len(hin), cb, None)
        self._check(st)
        if errors:
            raise errors[0]
        return hout

    def GatherRange(self, seq: int, range: tuple, layer: int) -> np.ndarray:
        n = max(0, range[1] - range[0]) * self.dim
        out = np.zeros(max(1, n), dtype=np.uint64)
        self._check(self._lib.ss_gather_range(self._h, seq, range[0], range[1], layer,
                                              _ptr(out, C.c_uint64), n))
        return out[:n]

    def BuildAddr(self, seq: int, range: tuple) -> KVAddrInfo:
        a, keep = self._addr_out(max(0, range[1] - range[0]))
        self._check(self._lib.ss_build_addr(self._h, seq, range[0], range[1], C.byref(a)))
        return self._addr_in(a, keep)

    # -- transfer agent -----------------------------------------------------------
    def ApplyRemoteWrite(self, addr: KVAddrInfo, layer: int, payload, tag: int) -> ApplyStatus:
        a, keep = addr._c()
        p = np.ascontiguousarray(np.asarray(payload, dtype=np.uint64))
        pp = p if len(p) else np.zeros(1, np.uint64)
        st = C.c_int32()
        self._check(self._lib.ss_apply_remote_write(self._h, C.byref(a), layer,
                                                    _ptr(pp, C.c_uint64), len(p), tag,
                                                    C.byref(st)))
        return ApplyStatus(st.value)

    def DrainReceiveCompletions(self) -> list:
        out: list = []
        buf = np.zeros(256, dtype=np.int64)
        while True:
            n = C.c_int64()
            self._check(self._lib.ss_drain_receive_completions(self._h, _ptr(buf, C.c_int64),
                                                               len(buf), C.byref(n)))
            out.extend(int(x) for x in buf[:n.value])
            if n.value < len(buf):
                return out

    # -- lifecycle -----------------------------------------------------------------
    def SetFinished(self, seq: int, finished: bool) -> None:
        self._check(self._lib.ss_set_finished(self._h, seq, 1 if finished else 0))

    def CommitToTree(self, seq: int) -> None:
        self._check(self._lib.ss_commit_to_tree(self._h, seq))

    def FreeSequence(self, seq: int) -> None:
        self._check(self._lib.ss_free_sequence(self._h, seq))

    def Evict(self, bytes_needed: int) -> int:
        f = C.c_int64()
        self._check(self._lib.ss_evict(self._h, bytes_needed, C.byref(f)))
        return f.value

    def Pin(self, prefix, flag: bool) -> None:
        t = _tok(prefix)
        self._check(self._lib.ss_pin(self._h, _ptr(t, C.c_int32), len(t), 1 if flag else 0))

    # -- queries -----------------------------------------------------------------------
    def HasSequence(self, seq: int) -> bool:
        return bool(self._lib.ss_has_sequence(self._h, seq))

    def GetRecord(self, seq: int) -> SequenceRecordInfo:
        info = _RecordInfo()
        self._check(self._lib.ss_get_record(self._h, seq, C.byref(info), None, 0))
        pages = np.zeros(max(1, info.num_own_pages), dtype=np.int64)
        self._check(self._lib.ss_get_record(self._h, seq, C.byref(info), _ptr(pages, C.c_int64),
                                            len(pages)))
        win = None
        if info.has_window:
            win = {"range": (info.window_begin, info.window_end),
                   "expected_writes": info.window_expected_writes,
                   "received_writes": info.window_received_writes,
                   "complete": bool(info.window_complete)}
        return SequenceRecordInfo(info.id, info.parent, info.fork_len, info.refcount,
                                  bool(info.finished), info.alloc_len, info.committed_hint,
                                  info.num_tokens, [int(p) for p in pages[:info.num_own_pages]],
                                  info.fold_frontier, info.digest_len, info.prefix_digest, win)

    def Committed(self, seq: int) -> int:
        v = C.c_int64()
        self._check(self._lib.ss_committed(self._h, seq, C.byref(v)))
        return v.value

    def ReadEntryWords(self, seq: int, pos: int, layer: int) -> np.ndarray:
        out = np.zeros(self.dim, dtype=np.uint64)
        self._check(self._lib.ss_read_entry_words(self._h, seq, pos, layer, _ptr(out, C.c_uint64),
                                                  self.dim))
        return out

    def FillOf(self, seq: int, pos: int, layer: int) -> FillState:
        v = C.c_int32()
        self._check(self._lib.ss_fill_of(self._h, seq, pos, layer, C.byref(v)))
        return FillState(v.value)

    def FreePages(self) -> int:
        return self._lib.ss_free_pages(self._h)

    def cache_config(self) -> dict:  # kv_cache.h:235 (+ the model geometry)
        c = _Config()
        self._check(self._lib.ss_cache_config(self._h, C.byref(c)))
        return {k: getattr(c, k) for k, _ in _Config._fields_}

    def TotalPages(self) -> int:
        return self._lib.ss_total_pages(self._h)

    def BytesPerPage(self) -> int:
        return self._lib.ss_bytes_per_page(self._h)

    def SequenceCount(self) -> int:
        return self._lib.ss_sequence_count(self._h)

    def SequenceIds(self) -> list:
        n = C.c_int64()
        buf = np.zeros(max(1, self.SequenceCount()), dtype=np.int64)
        self._check(self._lib.ss_sequence_ids(self._h, _ptr(buf, C.c_int64), len(buf), C.byref(n)))
        return [int(x) for x in buf[:n.value]]

    def PendingSendCount(self) -> int:
        return self._lib.ss_pending_send_count(self._h)

    def TreeNodeCount(self) -> int:
        return self._lib.ss_tree_node_count(self._h)

    def TreeContains(self, seq: int) -> bool:
        return bool(self._lib.ss_tree_contains(self._h, seq))

    def TreeLastTouch(self, seq: int) -> int:
        return self._lib.ss_tree_last_touch(self._h, seq)

    def TreeSequencesByLru(self) -> list:
        n = C.c_int64()
        buf = np.zeros(max(1, self.SequenceCount() + 64), dtype=np.int64)
        st = self._lib.ss_tree_sequences_by_lru(self._h, _ptr(buf, C.c_int64), len(buf), C.byref(n))
        if st == SS_ERR_BUFFER_TOO_SMALL:
            buf = np.zeros(n.value, dtype=np.int64)
            st = self._lib.ss_tree_sequences_by_lru(self._h, _ptr(buf, C.c_int64), len(buf),
                                                    C.byref(n))
        self._check(st)
        return [int(x) for x in buf[:n.value]]

    # -- B200 device entry points -----------------------------------------------------
    def attach_peer(self, dest: int, peer: "KVCache") -> None:
        self._check(self._lib.ss_attach_peer(self._h, dest, peer._h))
        self._keep.append(peer)

    def export_ipc(self) -> bytes:
        h = IpcHandle()
        self._check(self._lib.ss_export_ipc(self._h, C.byref(h)))
        return bytes(h.bytes)

    def import_ipc(self, dest: int, handle: bytes) -> None:
        h = IpcHandle()
        C.memmove(h.bytes, handle, len(handle))
        self._check(self._lib.ss_import_ipc(self._h, dest, C.byref(h)))

    def peer_info(self, dest: int) -> dict:
        """{'sys_scope': bool, 'peer_device': int} of sends to `dest`."""
        sc, dv = C.c_int32(), C.c_int32()
        self._check(self._lib.ss_peer_info(self._h, dest, C.byref(sc), C.byref(dv)))
        return {"sys_scope": bool(sc.value), "peer_device": dv.value}

    def detach_peer(self, dest: int) -> None:
        self._check(self._lib.ss_detach_peer(self._h, dest))

    def direct_send_async(self, seq: int, range: tuple, dest: int, dest_addr: KVAddrInfo,
                          user_tag: int = 0, layers: Optional[tuple] = None,
                          stream: int = 0) -> None:
        lb, le = layers if layers is not None else (0, self.layers)
        a, keep = dest_addr._c()
        self._check(self._lib.ss_direct_send_async(self._h, seq, range[0], range[1], dest,
                                                   C.byref(a), user_tag, lb, le,
                                                   C.c_void_p(stream)))

    def begin_direct_send(self, seq: int, range: tuple, dest: int, dest_addr: KVAddrInfo,
                          user_tag: int = 0) -> ForwardPlan:
        a, keep = dest_addr._c()
        h = C.c_void_p()
        self._check(self._lib.ss_begin_direct_send(self._h, seq, range[0], range[1], dest,
                                                   C.byref(a), user_tag, C.byref(h)))
        return ForwardPlan(self, h.value)

    def launch_direct_send_async(self, plan: ForwardPlan, layers: Optional[tuple] = None,
                                 stream: int = 0) -> None:
        lb, le = layers if layers is not None else (0, self.layers)
        self._check(self._lib.ss_launch_direct_send_async(self._h, plan.handle, lb, le,
                                                          C.c_void_p(stream)))

    def launch_direct_send_after_async(self, plan: ForwardPlan, layers: tuple, event: int,
                                       stream: int = 0) -> None:
        """Validation now, copy after `event` (a cudaEvent_t handle, e.g.
        torch.cuda.Event().cuda_event) of the producing layer's writes."""
        lb, le = layers
        self._check(self._lib.ss_launch_direct_send_after_async(
            self._h, plan.handle, lb, le, C.c_void_p(event), C.c_void_p(stream)))

    def launch_relay_send_async(self, plan: ForwardPlan, layers: Optional[tuple] = None,
                                timeout_ms: int = 60000, stream: int = 0) -> None:
        """Forward each layer of a range this engine is still receiving to
        the plan's destination once it has landed here (relay chain)."""
        lb, le = layers if layers is not None else (0, self.layers)
        self._check(self._lib.ss_launch_relay_send_async(self._h, plan.handle, lb, le, timeout_ms,
                                                         C.c_void_p(stream)))

    SEND_KERNEL, SEND_COPY_ENGINE = 0, 1

    def set_send_mode(self, mode: int = 0, max_ctas: int = 0) -> None:
        """DirectSend row mover: SEND_KERNEL (copy kernel, grid capped at
        max_ctas CTAs when > 0) or SEND_COPY_ENGINE (copy engines, no SMs
        for the rows); see ss_set_send_mode."""
        self._check(self._lib.ss_set_send_mode(self._h, mode, max_ctas))

    def broadcast_send_async(self, seq: int, range: tuple, dests: Sequence[int],
                             dest_addrs: Sequence[KVAddrInfo], user_tag: int = 0,
                             layers: Optional[tuple] = None, stream: int = 0) -> None:
        """Fan-out DirectSend of [range) to several receivers (source rows read once)."""
        lb, le = layers if layers is not None else (0, self.layers)
        n = len(dests)
        arr = (_Addr * max(1, n))()
        keep = []
        for i, a in enumerate(dest_addrs):
            ca, k = a._c()
            arr[i] = ca
            keep.append(k)
        d = np.ascontiguousarray(np.asarray(dests, dtype=np.int32))
        self._check(self._lib.ss_broadcast_send_async(self._h, seq, range[0], range[1], n,
                                                      _ptr(d, C.c_int32), arr, user_tag, lb, le,
                                                      C.c_void_p(stream)))

    def attention_async(self, layer: int, plan: ForwardPlan, hidden_in_ptr: int,
                        hidden_out_ptr: int, stream: int = 0) -> None:
        self._check(self._lib.ss_attention_async(self._h, plan.handle, layer,
                                                 C.c_void_p(hidden_in_ptr),
                                                 C.c_void_p(hidden_out_ptr), C.c_void_p(stream)))

    def gather_range_async(self, seq: int, range: tuple, layer: int, out_ptr: int,
                           stream: int = 0) -> None:
        self._check(self._lib.ss_gather_range_async(self._h, seq, range[0], range[1], layer,
                                                    C.c_void_p(out_ptr), C.c_void_p(stream)))

    def gather_range_layers_async(self, seq: int, range: tuple, layers: tuple, out_ptr: int,
                                  stream: int = 0) -> None:
        """GatherRange of layers [begin, end) in one launch into
        out[end - begin][range rows][dim] u64 words in device memory."""
        self._check(self._lib.ss_gather_range_layers_async(self._h, seq, range[0], range[1],
                                                           layers[0], layers[1],
                                                           C.c_void_p(out_ptr), C.c_void_p(stream)))

    # ---- wire formats (transport.h:6-12): frames for the cross-node path ----
    def crc32_async(self, data_ptr: int, n_bytes: int, crc_ptr: int, stream: int = 0) -> None:
        """Crc32 (transport.cc:14-28) of device bytes, written as uint32 at crc_ptr."""
        self._check(self._lib.ss_crc32_async(self._h, C.c_void_p(data_ptr), n_bytes,
                                             C.c_void_p(crc_ptr), C.c_void_p(stream)))

    def EncodeWriteFrame(self, seq: int, range: tuple, layer: int, seq_tag: int,
                         dest_addr: KVAddrInfo) -> bytes:
        """EncodeWriteFrame(WriteFrame{seq_tag, layer, dest_addr,
        GatherRange(seq, range, layer)}) (transport.cc:46-62): the frame a
        socket sends, payload gathered and checksummed on the GPU."""
        a, keep = dest_addr._c()
        n = C.c_int64(0)
        need = self._lib.ss_frame_write_header_size(len(dest_addr.array)) + \
            (range[1] - range[0]) * self.dim * 8 + 4
        buf = (C.c_uint8 * max(1, need))()
        self._check(self._lib.ss_encode_write_frame(self._h, seq, range[0], range[1], layer,
                                                    seq_tag, C.byref(a), buf, len(buf),
                                                    C.byref(n)))
        return bytes(buf)[:n.value]

    def encode_write_frame_into(self, seq: int, range: tuple, layer: int, seq_tag: int,
                                dest_addr: KVAddrInfo, out_ptr: int, cap: int) -> int:
        """EncodeWriteFrame into caller host memory (e.g. a pinned, reused
        socket buffer); returns the frame length."""
        a, keep = dest_addr._c()
        n = C.c_int64(0)
        self._check(self._lib.ss_encode_write_frame(self._h, seq, range[0], range[1], layer,
                                                    seq_tag, C.byref(a), C.c_void_p(out_ptr),
                                                    cap, C.byref(n)))
        return n.value

    def receive_write_frame_from(self, frame_ptr: int, size: int) -> tuple[bytes, int]:
        """ReceiveWriteFrame of a frame in caller host memory."""
        ack = (C.c_uint8 * 26)()
        st = C.c_int32(-1)
        self._check(self._lib.ss_receive_write_frame(self._h, C.c_void_p(frame_ptr), size, ack,
                                                     C.byref(st)))
        return bytes(ack), st.value

    def encode_write_frame_async(self, seq: int, range: tuple, layer: int, seq_tag: int,
                                 dest_addr: KVAddrInfo, frame_ptr: int, cap: int,
                                 stream: int = 0) -> int:
        """Device-memory frame; frame_ptr + header size must be 32-byte aligned.
        Returns the frame length."""
        a, keep = dest_addr._c()
        n = C.c_int64(0)
        self._check(self._lib.ss_encode_write_frame_async(
            self._h, seq, range[0], range[1], layer, seq_tag, C.byref(a), C.c_void_p(frame_ptr),
            cap, C.byref(n), C.c_void_p(stream)))
        return n.value

    def ReceiveWriteFrame(self, frame: bytes) -> tuple[bytes, int]:
        """The transfer agent's step for one write frame (tcp_fabric.cc:144-168):
        returns (ack frame bytes, apply status or -1 when the CRC failed)."""
        ack = (C.c_uint8 * 26)()
        st = C.c_int32(-1)
        self._check(self._lib.ss_receive_write_frame(self._h, frame, len(frame), ack,
                                                     C.byref(st)))
        return bytes(ack), st.value

    def apply_remote_write_async(self, addr: KVAddrInfo, layer: int, payload_ptr: int,
                                 n_words: int, tag: int, stream: int = 0) -> ApplyStatus:
        a, keep = addr._c()
        st = C.c_int32()
        self._check(self._lib.ss_apply_remote_write_async(self._h, C.byref(a), layer,
                                                          C.c_void_p(payload_ptr), n_words, tag,
                                                          C.byref(st), C.c_void_p(stream)))
        return ApplyStatus(st.value)

    def append_rows_async(self, plan: ForwardPlan, layer: int, rows_ptr: int,
                          stream: int = 0) -> None:
        self._check(self._lib.ss_append_rows_async(self._h, plan.handle, layer,
                                                   C.c_void_p(rows_ptr), C.c_void_p(stream)))

    def append_rows_layers_async(self, plan: ForwardPlan, layers: tuple, rows_ptr: int,
                                 stream: int = 0) -> None:
        """KV append for layers [begin, end) in one launch; rows are
        [end - begin][total_outputs][dim] u64 words in device memory."""
        self._check(self._lib.ss_append_rows_layers_async(self._h, plan.handle, layers[0],
                                                          layers[1], C.c_void_p(rows_ptr),
                                                          C.c_void_p(stream)))

    def append_rows_send_async(self, plan: ForwardPlan, send_plan: ForwardPlan, layers: tuple,
                               rows_ptr: int, stream: int = 0) -> None:
        """KV append fused with remote_send: rows [end - begin][total_outputs][dim]
        go to this engine's output slots and, for send_plan's range, straight
        into the receiver's reserved pages (one launch per call)."""
        self._check(self._lib.ss_append_rows_send_async(self._h, plan.handle, send_plan.handle,
                                                        layers[0], layers[1],
                                                        C.c_void_p(rows_ptr), C.c_void_p(stream)))

    def begin_decode(self, seqs: Sequence[int], ctx_lens: Sequence[int]) -> ForwardPlan:
        s = np.ascontiguousarray(np.asarray(seqs, dtype=np.int64))
        c = np.ascontiguousarray(np.asarray(ctx_lens, dtype=np.int64))
        h = C.c_void_p()
        self._check(self._lib.ss_begin_decode(self._h, _ptr(s, C.c_int64), _ptr(c, C.c_int64),
                                              len(s), C.byref(h)))
        return ForwardPlan(self, h.value)

    def paged_decode_attention_async(self, plan: ForwardPlan, layer: int, num_q_heads: int,
                                     num_kv_heads: int, head_dim: int, softmax_scale: float,
                                     q_ptr: int, out_ptr: int, stream: int = 0) -> None:
        self._check(self._lib.ss_paged_decode_attention_async(
            self._h, plan.handle, layer, num_q_heads, num_kv_heads, head_dim,
            C.c_float(softmax_scale), C.c_void_p(q_ptr), C.c_void_p(out_ptr),
            C.c_void_p(stream)))

    def paged_prefill_attention_async(self, seq: int, q_range, layer: int, num_q_heads: int,
                                      num_kv_heads: int, head_dim: int, softmax_scale: float,
                                      q_ptr: int, out_ptr: int, stream: int = 0) -> None:
        """Causal attention of positions [q_range) of `seq` over keys [0, q_end)
        (tcgen05 kernel; q/out bf16 [n_q][num_q_heads][head_dim])."""
        b, e = q_range
        self._check(self._lib.ss_paged_prefill_attention_async(
            self._h, seq, b, e, layer, num_q_heads, num_kv_heads, head_dim,
            C.c_float(softmax_scale), C.c_void_p(q_ptr), C.c_void_p(out_ptr),
            C.c_void_p(stream)))

    def pool_layer_ptr(self, layer: int) -> int:
        p = C.c_void_p()
        self._check(self._lib.ss_pool_layer_ptr(self._h, layer, C.byref(p)))
        return p.value

    def wait_receive_async(self, seq: int, timeout_ms: int = 10000, stream: int = 0) -> None:
        self._check(self._lib.ss_wait_receive_async(self._h, seq, timeout_ms, C.c_void_p(stream)))

    def wait_receive_layer_async(self, seq: int, layer: int, timeout_ms: int = 10000,
                                 stream: int = 0) -> None:
        """Device-side wait on `stream` until layer `layer` of seq's receive
        window has fully landed (the per-layer ready flag)."""
        self._check(self._lib.ss_wait_receive_layer_async(self._h, seq, layer, timeout_ms,
                                                          C.c_void_p(stream)))

    def copy_counters(self) -> tuple[int, int]:
        h, d = C.c_int64(), C.c_int64()
        self._check(self._lib.ss_copy_counters(self._h, C.byref(h), C.byref(d)))
        return h.value, d.value

    def kernel_launches(self) -> int:
        return self._lib.ss_kernel_launches(self._h)

    def synchronize(self) -> None:
        self._check(self._lib.ss_synchronize(self._h))
