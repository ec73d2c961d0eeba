"""The microserving sub-request APIs over the B200 KV cache.

SPEC.md's engine module has no code in
the reference; this is the thin caller the paper describes, composed from
KVCache calls exactly as SURVEY.md §3 maps them:

  api_prep_recv(prompt, end)             -> (match_len, KVAddrInfo)
  api_remote_send(prompt, begin, end,
                  recv_rank, recv_addr)   -> None (returns when acked) SPEC.md:266-273
  api_start_generate(prompt, begin, n)   -> generated tokens
  compute_transfer_plan(m, begin, end)   -> segments

remote_send streams each segment the way SPEC.md prescribes: DirectSend
segments (already cached on the sender) with one fused copy launch over all
layers; PrefillThenSend segments through MarkSend + a forward pass whose
Attention ships every layer right after it is computed; PrefillOnly gaps are
computed and kept.  Transfers go device-direct when the receiving engine is
attached as a peer (same process, or CUDA IPC); otherwise through a host
fabric that delivers frames to the receiver's ApplyRemoteWrite — the
reference's transport hop (transport.cc:128-188) — which is also how the
engine runs on the reference library in the parity tests.

The hidden-state model is the reference's toy model (hash_model.cc), so a
generation through these APIs can be checked token for token against
HashModel::Generate.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence

import numpy as np

from .kvcache import ApplyStatus, BatchEntry, KVAddrInfo, KVCache, SplitserveError

DIRECT_SEND = "DirectSend"
PREFILL_THEN_SEND = "PrefillThenSend"
PREFILL_ONLY = "PrefillOnly"


@dataclass(frozen=True)
class Segment:
    kind: str
    begin: int
    end: int


def compute_transfer_plan(m: int, begin: int, end: int) -> List[Segment]:
    """positions of [begin, end) below the sender's match m
    are DirectSend; [max(m, begin), end) is PrefillThenSend; a gap [m, begin)
    (Case 2) is PrefillOnly.  Adjacent same-kind positions coalesce."""
    if not 0 <= begin <= end:
        raise ValueError("begin/end out of order")
    segs: List[Segment] = []
    if m < begin:
        segs.append(Segment(PREFILL_ONLY, m, begin))
    if begin < min(m, end):
        segs.append(Segment(DIRECT_SEND, begin, min(m, end)))
    if max(m, begin) < end:
        segs.append(Segment(PREFILL_THEN_SEND, max(m, begin), end))
    return segs


def resolve_end(n: int, end: int) -> int:
    """ResolveEndIndex (kv_cache.cc:13-18)."""
    e = n + end if end < 0 else end
    if end == 0 or not 0 < e <= n:
        raise SplitserveError(16, "InvalidArgument: end out of range")
    return e


def resolve_begin(n: int, begin: int) -> int:
    """ResolveBeginIndex (kv_cache.cc:20-24)."""
    b = n + begin if begin < 0 else begin
    if not 0 <= b <= n:
        raise SplitserveError(16, "InvalidArgument: begin out of range")
    return b


class Fabric:
    """Host transfer plane between engines of one process: a frame for
    (send, layer) is applied on the receiver (ReceiverPort.apply ->
    ApplyRemoteWrite, transport.cc:169).  Used when no device peer exists."""

    def __init__(self):
        self.engines: Dict[int, "Engine"] = {}
        self.frames = 0

    def register(self, engine: "Engine") -> None:
        self.engines[engine.rank] = engine

    def sink(self, layer, send, payload) -> None:
        dst = self.engines[send["dest"]]
        st = dst.cache.ApplyRemoteWrite(send["dest_addr"], layer, payload, send["user_tag"])
        if st != ApplyStatus.Ok:
            raise SplitserveError(10, f"UnknownAddress: frame rejected ({st.name})")
        self.frames += 1


class Engine:
    """One microserving engine: a KVCache plus request bookkeeping."""

    _ids = itertools.count(1)

    def __init__(self, cache: KVCache, rank: int, fabric: Optional[Fabric] = None):
        self.cache = cache
        self.rank = rank
        self.fabric = fabric
        self.peers: Dict[int, "Engine"] = {}
        self.awaiting: Dict[tuple, int] = {}  # prompt key -> seq reserved by prep_recv
        if fabric is not None:
            fabric.register(self)

    # -- wiring ------------------------------------------------------------------
    def attach(self, other: "Engine") -> None:
        """Device-direct sends to `other` (in-process peer engine)."""
        self.cache.attach_peer(other.rank, other.cache)
        self.peers[other.rank] = other

    def _device_peer(self, rank: int) -> bool:
        return rank in self.peers

    @staticmethod
    def _key(prompt) -> tuple:
        return tuple(int(t) for t in prompt)

    def _new_seq(self) -> int:
        return next(Engine._ids) + 1000 * (self.rank + 1)

    # -- api_prep_recv ----------------------------------------------
    def api_prep_recv(self, prompt: Sequence[int], end: int = -1):
        seq = self._new_seq()
        r = self.cache.PrepRecv(seq, prompt, end)
        self.awaiting[self._key(prompt)] = seq
        return r.match_len, r.addr

    # -- api_remote_send -----------------------------------------
    def api_remote_send(self, prompt: Sequence[int], begin: int, end: int, recv_rank: int,
                        recv_addr: KVAddrInfo, tag: int = 0) -> List[Segment]:
        n = len(prompt)
        b, e = resolve_begin(n, begin), resolve_end(n, end)
        if recv_addr.token_begin != b or recv_addr.token_count != e - b:
            raise SplitserveError(5, "AddrMismatch: receiver address does not cover [begin, end)")
        m, owner = self.cache.MatchPrefixSeq(list(prompt[:e]))
        plan = compute_transfer_plan(m, b, e)
        seq = self._new_seq()
        if m > 0:
            self.cache.ForkSequence(owner, seq, m, list(prompt))
        else:
            self.cache.CreateSequence(seq, list(prompt))
        self.cache.EnsureAllocated(seq, e)
        device = self._device_peer(recv_rank)
        for s in plan:
            if s.kind == DIRECT_SEND:
                sub = recv_addr.Slice(s.begin, s.end)
                if device:
                    self.cache.direct_send_async(seq, (s.begin, s.end), recv_rank, sub, tag)
                else:  # GatherRange + frame per layer
                    for layer in range(self.cache.layers):
                        payload = self.cache.GatherRange(seq, (s.begin, s.end), layer)
                        self.fabric.sink(layer, {"dest": recv_rank, "dest_addr": sub,
                                                 "user_tag": tag}, payload)
            elif s.kind == PREFILL_THEN_SEND:
                self.cache.MarkSend(seq, (s.begin, s.end), recv_rank,
                                    recv_addr.Slice(s.begin, s.end), tag)
        first = min((s.begin for s in plan if s.kind != DIRECT_SEND), default=None)
        if first is not None:  # one forward pass covers PrefillOnly + PrefillThenSend
            self._forward(seq, prompt, first, e, None if device else self.fabric.sink)
        if device:
            self.cache.synchronize()  # remote_send returns once the writes landed
        self.cache.SetFinished(seq, True)
        self.cache.CommitToTree(seq)  # senders grow their context cache
        return plan

    # -- api_start_generate -------------------------------------------
    def api_start_generate(self, prompt: Sequence[int], begin: int, max_tokens: int = 1):
        n = len(prompt)
        b = resolve_begin(n, begin)
        self.cache.DrainReceiveCompletions()
        seq = self.awaiting.pop(self._key(prompt), None)
        if seq is None:  # no reservation: plain generation from the local context
            seq = self._new_seq()
            m, owner = self.cache.MatchPrefixSeq(list(prompt))
            m = min(m, b)
            if m > 0:
                self.cache.ForkSequence(owner, seq, m, list(prompt))
            else:
                self.cache.CreateSequence(seq, list(prompt))
        self.cache.EnsureAllocated(seq, n)
        x = self._forward(seq, prompt, b, n, None)
        out = [self.cache.SampleToken(int(x[-1]))]
        for k in range(1, max_tokens):
            t = out[-1]
            self.cache.AppendToken(seq, t)
            self.cache.EnsureAllocated(seq, n + k)
            x = self._forward_tokens(seq, [t], n + k - 1, True)
            out.append(self.cache.SampleToken(int(x[-1])))
        self.cache.SetFinished(seq, True)
        self.cache.CommitToTree(seq)
        return out

    # -- forward passes (SPEC.md:284-290 `step`) --------------------------------------------
    def _forward(self, seq, prompt, begin, end, sink):
        return self._run(seq, (begin, end), [int(prompt[i]) for i in range(begin, end)], False,
                         sink)

    def _forward_tokens(self, seq, toks, pos, is_decode):
        return self._run(seq, (pos, pos + len(toks)), toks, is_decode, None)

    def _run(self, seq, rng, toks, is_decode, sink):
        plan = self.cache.BeginForward([BatchEntry(seq, rng, is_decode)])
        x = np.array([self.cache.Embed(t, rng[0] + i) for i, t in enumerate(toks)],
                     dtype=np.uint64)
        for layer in range(self.cache.layers):
            x = self.cache.Attention(layer, plan, x, sink)
        if hasattr(plan, "close"):
            plan.close()
        return x
