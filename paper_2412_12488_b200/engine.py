"""The microserving sub-request APIs over the B200 KV cache.

SPEC.md's engine module has no code in
the reference; this is the thin caller the paper describes, composed from
KVCache calls exactly as SURVEY.md §3 maps them:

  api_prep_recv(prompt, end)             -> (match_len, KVAddrInfo)
  api_remote_send(prompt, begin, end,
                  recv_rank, recv_addr)   -> None (returns when acked) SPEC.md:266-273
  api_start_generate(prompt, begin, n)   -> generated tokens
  compute_transfer_plan(m, begin, end)   -> segments
  submit(GenRequest) / step()            -> continuous batching

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
from collections import deque
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence

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


class FrameFabric(Fabric):
    """The reference's wire path (TCP fabric, tcp_fabric.cc:144-168,266-277)
    between engines of one process: each (send, layer) travels as an encoded
    write frame (header + payload + CRC-32, byte-identical to
    EncodeWriteFrame), the receiver runs its transfer-agent step
    (ReceiveWriteFrame: CRC, ApplyRemoteWrite, ack) and a ChecksumMismatch
    ack triggers one retransmit (SPEC.md transport, "single retransmit").
    On the B200 library the sender gathers and checksums the payload on the
    GPU (ss_encode_write_frame) and the receiver checks it on the GPU.
    `fault(frame) -> frame` may corrupt frames in flight (first attempt)."""

    def __init__(self, fault: Optional[Callable[[bytes], bytes]] = None):
        super().__init__()
        self.fault = fault
        self.retransmits = 0
        self.bytes = 0

    def deliver(self, src: "Engine", seq: int, rng: tuple, layer: int, dest: int,
                dest_addr: KVAddrInfo, tag: int) -> None:
        frame = src.cache.EncodeWriteFrame(seq, rng, layer, tag, dest_addr)
        dst = self.engines[dest].cache
        for attempt in (1, 2):
            wire = self.fault(frame) if (self.fault is not None and attempt == 1) else frame
            ack, st = dst.ReceiveWriteFrame(wire)
            self.bytes += len(wire)
            status = ack[-1]  # AckStatus, the ack frame's last byte (transport.cc:73)
            if status == 1 and attempt == 1:  # ChecksumMismatch: retransmit once
                self.retransmits += 1
                continue
            if status != 0:
                raise SplitserveError(10 if status == 2 else 9,
                                      f"frame for layer {layer} rejected (ack status {status})")
            self.frames += 1
            return


@dataclass
class GenRequest:
    """SPEC.md engine GenRequest: prompt[:begin] already present in the cache
    (received or cached); the engine prefills prompt[begin:] and decodes."""
    request_id: int
    prompt: List[int]
    begin: int
    max_tokens: int
    seq: int = -1
    tokens: List[int] = field(default_factory=list)
    done: bool = False
    error: Optional[SplitserveError] = None


class Engine:
    """One microserving engine: a KVCache plus request bookkeeping."""

    _ids = itertools.count(1)

    def __init__(self, cache: KVCache, rank: int, fabric: Optional[Fabric] = None):
        self.cache = cache
        self.rank = rank
        self.fabric = fabric
        self.peers: Dict[int, "Engine"] = {}
        self.awaiting: Dict[tuple, int] = {}  # prompt key -> seq reserved by prep_recv
        self.waiting: deque = deque()          # admitted, prefill pending (FIFO)
        self.running: List[GenRequest] = []    # decoding
        self.steps = 0
        self.last_batch: List[BatchEntry] = []
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
    def api_prep_recv(self, prompt: Sequence[int], end: int = -1, register: bool = True):
        """register=False: a context transfer (migration), not a generation
        the next start_generate of this prompt should bind to."""
        seq = self._new_seq()
        r = self.cache.PrepRecv(seq, prompt, end)
        if register:
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
        framed = not device and isinstance(self.fabric, FrameFabric)
        after_layer = []  # (range, addr) streamed as frames after each layer's compute
        for s in plan:
            if s.kind == DIRECT_SEND:
                sub = recv_addr.Slice(s.begin, s.end)
                if device:
                    self.cache.direct_send_async(seq, (s.begin, s.end), recv_rank, sub, tag)
                elif framed:
                    for layer in range(self.cache.layers):
                        self.fabric.deliver(self, seq, (s.begin, s.end), layer, recv_rank, sub,
                                            tag)
                else:  # GatherRange + frame per layer
                    for layer in range(self.cache.layers):
                        payload = self.cache.GatherRange(seq, (s.begin, s.end), layer)
                        self.fabric.sink(layer, {"dest": recv_rank, "dest_addr": sub,
                                                 "user_tag": tag}, payload)
            elif s.kind == PREFILL_THEN_SEND:
                sub = recv_addr.Slice(s.begin, s.end)
                if framed:
                    after_layer.append(((s.begin, s.end), sub))
                else:
                    self.cache.MarkSend(seq, (s.begin, s.end), recv_rank, sub, tag)
        first = min((s.begin for s in plan if s.kind != DIRECT_SEND), default=None)
        if first is not None:  # one forward pass covers PrefillOnly + PrefillThenSend
            hook = None
            if after_layer:
                def hook(layer):  # layer-eager frames (§3.6)
                    for rng, sub in after_layer:
                        self.fabric.deliver(self, seq, rng, layer, recv_rank, sub, tag)
            self._forward(seq, prompt, first, e,
                          None if (device or framed) else self.fabric.sink, hook)
        if device:
            self.cache.synchronize()  # remote_send returns once the writes landed
        self.cache.SetFinished(seq, True)
        self.cache.CommitToTree(seq)  # senders grow their context cache
        return plan

    # -- api_start_generate -------------------------------------------
    def api_start_generate(self, prompt: Sequence[int], begin: int, max_tokens: int = 1):
        """Admits the request and runs the step loop until it finishes; other
        admitted requests advance in the same batches."""
        req = self.submit(GenRequest(next(Engine._ids), list(prompt), begin, max_tokens))
        while not req.done:
            self.step()
        if req.error is not None:
            raise req.error
        return req.tokens

    def submit(self, req: GenRequest) -> GenRequest:
        """Admission (FIFO): resolve begin, bind the sequence prep_recv
        reserved for this prompt (or fork the longest cached prefix)."""
        n = len(req.prompt)
        req.begin = resolve_begin(n, req.begin)
        if req.begin >= n:
            raise SplitserveError(16, "InvalidArgument: begin must leave a token to prefill")
        seq = self.awaiting.pop(self._key(req.prompt), None)
        if seq is None:  # no reservation: plain generation from the local context
            seq = self._new_seq()
            m, owner = self.cache.MatchPrefixSeq(list(req.prompt))
            m = min(m, req.begin)
            if m > 0:
                self.cache.ForkSequence(owner, seq, m, list(req.prompt))
            else:
                self.cache.CreateSequence(seq, list(req.prompt))
        req.seq = seq
        self.waiting.append(req)
        return req

    def step(self) -> List[tuple]:
        """SPEC.md engine.step: one batch of every waiting prefill (FIFO, no
        chunking) and every running decode; BeginForward, Attention over all
        layers, one sampled token per request.  Returns (request_id, token)
        events.  Requests whose prefix is missing (MissingKV) or that run out
        of pages are aborted with that status; the rest of the batch runs."""
        self.cache.DrainReceiveCompletions()
        batch: List[GenRequest] = []
        entries: List[BatchEntry] = []
        toks: List[int] = []
        while self.waiting:
            req = self.waiting.popleft()
            n = len(req.prompt)
            try:
                # BeginForward's precondition (kv_cache.cc:255-258), checked per
                # request so one early start_generate cannot fail the batch.
                if self.cache.Committed(req.seq) < req.begin:
                    raise SplitserveError(6, f"MissingKV: positions before {req.begin} "
                                             "are not all present")
                self.cache.EnsureAllocated(req.seq, n)
            except SplitserveError as ex:
                self._abort(req, ex)
                continue
            batch.append(req)
            entries.append(BatchEntry(req.seq, (req.begin, n), False))
            toks.extend(int(t) for t in req.prompt[req.begin:n])
        for req in self.running:
            pos = len(req.prompt) + len(req.tokens) - 1
            try:
                self.cache.AppendToken(req.seq, req.tokens[-1])
                self.cache.EnsureAllocated(req.seq, pos + 1)
            except SplitserveError as ex:
                self._abort(req, ex)
                continue
            batch.append(req)
            entries.append(BatchEntry(req.seq, (pos, pos + 1), True))
            toks.append(req.tokens[-1])
        self.running = [r for r in self.running if not r.done]
        if not batch:
            return []
        plan = self.cache.BeginForward(entries)
        x = self._embed(entries, toks)
        for layer in range(self.cache.layers):
            x = self.cache.Attention(layer, plan, x)
        if hasattr(plan, "close"):
            plan.close()
        self.last_batch = entries
        self.steps += 1
        events, off = [], 0
        for req, ent in zip(batch, entries):
            off += ent.range[1] - ent.range[0]
            tok = self.cache.SampleToken(int(x[off - 1]))
            req.tokens.append(tok)
            events.append((req.request_id, tok))
            if len(req.tokens) >= req.max_tokens:
                self._finish(req)
            elif req not in self.running:
                self.running.append(req)
        self.running = [r for r in self.running if not r.done]
        return events

    def _embed(self, entries, toks) -> np.ndarray:
        out, i = np.empty(len(toks), dtype=np.uint64), 0
        for e in entries:
            for pos in range(e.range[0], e.range[1]):
                out[i] = self.cache.Embed(toks[i], pos)
                i += 1
        return out

    def _finish(self, req: GenRequest) -> None:
        req.done = True
        self.cache.SetFinished(req.seq, True)
        self.cache.CommitToTree(req.seq)

    def _abort(self, req: GenRequest, ex: SplitserveError) -> None:
        req.done = True
        req.error = ex

    def idle(self) -> bool:
        return not self.waiting and not self.running

    # -- forward passes (SPEC.md:284-290 `step`) --------------------------------------------
    def _forward(self, seq, prompt, begin, end, sink, after_layer=None):
        return self._run(seq, (begin, end), [int(prompt[i]) for i in range(begin, end)], False,
                         sink, after_layer)

    def _run(self, seq, rng, toks, is_decode, sink, after_layer=None):
        plan = self.cache.BeginForward([BatchEntry(seq, rng, is_decode)])
        x = np.array([self.cache.Embed(t, rng[0] + i) for i, t in enumerate(toks)],
                     dtype=np.uint64)
        for layer in range(self.cache.layers):
            x = self.cache.Attention(layer, plan, x, sink)
            if after_layer is not None:
                after_layer(layer)
        if hasattr(plan, "close"):
            plan.close()
        return x
