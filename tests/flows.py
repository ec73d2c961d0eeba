"""Microserving flows composed from KVCache calls, exactly as SURVEY.md §3
maps SPEC.md's engine operations onto the reference interface.  Each helper
drives any object with the reference method names: the B200 product
(paper_2412_12488_b200.KVCache), the unmodified reference behind the ABI
(lib=oracle/_ref/libmicrokv_ref.so) or the Python restatement
(oracle.kvcache_oracle.KVCache)."""
from __future__ import annotations

import numpy as np

from paper_2412_12488_b200 import ApplyStatus, BatchEntry


def prefill(E, seq, prompt, begin, end, sink=None, layers=None, hiddens=None):
    """BeginForward([seq, [begin, end)]) + Attention over all layers; returns
    the last layer's hidden outputs (SPEC.md:284-290 `step`)."""
    L = layers if layers is not None else E.layers
    plan = E.BeginForward([BatchEntry(seq, (begin, end))])
    x = np.array([E.Embed(prompt[i], i) for i in range(begin, end)], dtype=np.uint64)
    for layer in range(L):
        x = E.Attention(layer, plan, x, sink)
        if hiddens is not None:
            hiddens.append(np.asarray(x).copy())
    if hasattr(plan, "close"):
        plan.close()
    return x


def start_generate(E, seq, prompt, begin, max_tokens=1):
    """api_start_generate: prefill prompt[begin:], sample,
    then greedy decode steps."""
    n = len(prompt)
    E.EnsureAllocated(seq, n)
    x = prefill(E, seq, prompt, begin, n)
    out = [E.SampleToken(int(x[-1]))]
    for k in range(1, max_tokens):
        t = out[-1]
        E.AppendToken(seq, t)
        E.EnsureAllocated(seq, n + k)
        plan = E.BeginForward([BatchEntry(seq, (n + k - 1, n + k), True)])
        x = np.array([E.Embed(t, n + k - 1)], dtype=np.uint64)
        for layer in range(E.layers):
            x = E.Attention(layer, plan, x)
        if hasattr(plan, "close"):
            plan.close()
        out.append(E.SampleToken(int(x[-1])))
    return out


def sink_into(D, corrupt=None, log=None):
    """FrameSink that applies each frame on the receiver (the fabric hop,
    transport.cc:169 -> ApplyRemoteWrite)."""

    def sink(layer, send, payload):
        if corrupt is not None:
            payload = corrupt(layer, send, np.array(payload, dtype=np.uint64))
        st = D.ApplyRemoteWrite(send["dest_addr"], layer, payload, send["user_tag"])
        if log is not None:
            log.append((layer, send["range"], int(st)))
        assert st == ApplyStatus.Ok, st

    return sink


def one_p_one_d(P, D, prompt, end=-1, via="sink", seq_p=20, seq_d=10, tag=7, max_tokens=1,
                corrupt=None, hiddens=None, p_has_prefix=None):
    """1P1D (Fig 3): D.prep_recv(end) ->
    P.remote_send([m, e)) with PrefillThenSend -> D.start_generate(e).

    via="sink": frames go through the host sink into D.ApplyRemoteWrite;
    via="peer": P has D attached and stores device-direct.
    Returns dict(match_len, addr, token(s), completions)."""
    r = D.PrepRecv(seq_d, prompt, end)
    m, e = r.match_len, r.match_len + r.addr.token_count
    if p_has_prefix is None:
        P.CreateSequence(seq_p, prompt)
        begin = 0
    else:
        parent, plen = p_has_prefix
        P.ForkSequence(parent, seq_p, plen, prompt)
        begin = plen
    P.EnsureAllocated(seq_p, e)
    if e > m:
        P.MarkSend(seq_p, (m, e), getattr(D, "rank", 1), r.addr, tag)
    sink = sink_into(D, corrupt) if via == "sink" else None
    if e > begin:
        prefill(P, seq_p, prompt, begin, e, sink=sink, hiddens=hiddens)
    if via == "peer":
        P.synchronize()
    done = D.DrainReceiveCompletions()
    toks = start_generate(D, seq_d, prompt, e, max_tokens)
    return {"match_len": m, "end": e, "addr": r.addr, "tokens": toks, "done": done}


def entries(E, seq, positions, layer):
    return np.stack([E.ReadEntryWords(seq, p, layer) for p in positions])
