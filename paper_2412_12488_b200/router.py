"""The programmable router of SPEC.md (router module, SPEC.md:382-476;
PAPER.md §3.2-3.3): request-level generate() turned into explicit call
scripts of the three microserving APIs over engines (engine.py) whose KV
cache is the B200 library (device-direct or framed transfers) or the
reference behind the same ABI.

Strategies (set_strategy swaps them without touching engines):
  data_parallel        [E.start_generate(prompt, 0)] round-robin      Ex.1 / Fig 2
  pd_disagg            D.prep_recv(-1) -> P.remote_send(0, -1) ->
                       D.start_generate(len-1)                         Ex.2 / Fig 3
  context_pd_disagg    as pd_disagg from D's match_len; no send when
                       D already holds prompt[:-1]                     Ex.3 / Fig 4
  balanced_pd{ratio}   s = max(match, floor((1-r) len)) clamped to
                       len-1; D prefills prompt[s:]                    §3.3 / Fig 6
  context_migration{threshold, window}
                       dispatch to the least-loaded owner of the
                       request's context; when the windowed load of the
                       busiest and idlest engines exceeds the threshold,
                       migrate the hottest context with
                       target.prep_recv(ctx, len) -> owner.remote_send  Ex.4 / Fig 5

Every executed call is appended to `log` as a dict (request, call, rank,
args, result) — the inspectable call graph the SPEC asks for.
"""
from __future__ import annotations

import itertools
from collections import Counter, deque
from dataclasses import dataclass, field
from typing import Deque, Dict, List, Optional, Sequence

from .engine import Engine
from .kvcache import SplitserveError

STRATEGIES = ("data_parallel", "pd_disagg", "context_pd_disagg", "balanced_pd",
              "context_migration")
_NO_ENGINES, _ROLE_MISSING, _UNKNOWN_STRATEGY = 12, 13, 15  # 1 + ErrorCode


@dataclass
class Result:
    request_id: int
    tokens: List[int]
    script: List[dict]
    strategy: str


@dataclass
class _Context:
    tokens: List[int]
    owners: List[int]


class Router:
    """Control plane over engines of one process.  `roles` maps rank ->
    "prefill" | "decode" | "any" (default "any")."""

    def __init__(self, engines: Sequence[Engine], roles: Optional[Dict[int, str]] = None,
                 strategy: str = "data_parallel", **params):
        if not engines:
            raise SplitserveError(_NO_ENGINES, "NoEngines: router needs at least one engine")
        self.engines: Dict[int, Engine] = {e.rank: e for e in engines}
        self.ranks = sorted(self.engines)
        self.roles = {r: (roles or {}).get(r, "any") for r in self.ranks}
        self.log: List[dict] = []
        self._ids = itertools.count(1)
        self._rr = itertools.count()
        self._rr_p = itertools.count()
        self._rr_d = itertools.count()
        self.contexts: Dict[str, _Context] = {}
        self.window: Deque[tuple] = deque()  # (category, rank) of recent dispatches
        self.migrations = 0
        self.strategy = "data_parallel"
        self.params: dict = {}
        self.set_strategy(strategy, **params)

    # -- configuration ----------------------------------------------------------------
    def set_strategy(self, name: str, **params) -> None:
        """hot swap; unknown names leave the active one."""
        if name not in STRATEGIES:
            raise SplitserveError(_UNKNOWN_STRATEGY, f"UnknownStrategy: {name}")
        if name == "balanced_pd":
            r = float(params.get("ratio", 0.2))
            if not 0.0 <= r < 1.0:
                raise SplitserveError(16, "InvalidArgument: ratio must be in [0, 1)")
            params = {"ratio": r}
        if name == "context_migration":
            params = {"threshold": float(params.get("threshold", 2.0)),
                      "window": int(params.get("window", 32))}
        self.strategy, self.params = name, dict(params)

    def register_context(self, category: str, tokens: Sequence[int], owner: int) -> None:
        """A context (shared prefix) owned by `owner`; the owner computes and
        caches it (plain start_generate of the context)."""
        toks = [int(t) for t in tokens]
        self._call(0, "start_generate", owner, self.engines[owner].api_start_generate,
                   (toks, 0, 1))
        self.contexts[category] = _Context(toks, [owner])

    # -- request path -------------------------------------------------------------
    def generate(self, prompt: Sequence[int], max_tokens: int = 1,
                 category: Optional[str] = None) -> Result:
        rid = next(self._ids)
        prompt = [int(t) for t in prompt]
        strategy = self.strategy  # in-flight requests finish under the admitting strategy
        n0 = len(self.log)
        fn = getattr(self, "_" + strategy)
        tokens = fn(rid, prompt, max_tokens, category)
        return Result(rid, tokens, self.log[n0:], strategy)

    def _pick(self, role: str, counter) -> int:
        ranks = [r for r in self.ranks if self.roles[r] in (role, "any")]
        if not ranks:
            raise SplitserveError(_ROLE_MISSING, f"RoleMissing: no {role} engine")
        return ranks[next(counter) % len(ranks)]

    def _call(self, rid: int, name: str, rank: int, fn, args: tuple):
        res = fn(*args)
        shown = tuple(a if not isinstance(a, list) else f"<{len(a)} tokens>" for a in args)
        self.log.append({"request": rid, "call": name, "rank": rank, "args": shown,
                         "result": res if name != "prep_recv" else (res[0], res[1].token_count)})
        return res

    def _data_parallel(self, rid, prompt, max_tokens, category):
        rank = self.ranks[next(self._rr) % len(self.ranks)]
        E = self.engines[rank]
        return self._call(rid, "start_generate", rank, E.api_start_generate,
                          (prompt, 0, max_tokens))

    def _disagg(self, rid, prompt, max_tokens, end_of, from_match: bool):
        """prep_recv(end) on D, remote_send([begin, end)) on P, start_generate(end) on D."""
        p, d = self._pick("prefill", self._rr_p), self._pick("decode", self._rr_d)
        P, D = self.engines[p], self.engines[d]
        n = len(prompt)
        if n == 1:  # nothing can be transferred (end=-1 is empty, kv_cache.cc:13-18)
            return self._call(rid, "start_generate", d, D.api_start_generate,
                              (prompt, 0, max_tokens))
        end = end_of(D, prompt)
        m, addr = self._call(rid, "prep_recv", d, D.api_prep_recv, (prompt, end))
        e = m + addr.token_count
        begin = m if from_match else 0
        if e > m:
            if not from_match and m > 0:
                # pd_disagg sends [0, end); positions D already holds are not
                # reserved, so the send covers [m, end) (Fig 3 with a warm D).
                begin = m
            self._call(rid, "remote_send", p, P.api_remote_send, (prompt, begin, e, d, addr))
        return self._call(rid, "start_generate", d, D.api_start_generate,
                          (prompt, e, max_tokens))

    def _pd_disagg(self, rid, prompt, max_tokens, category):
        return self._disagg(rid, prompt, max_tokens, lambda D, p: -1, from_match=False)

    def _context_pd_disagg(self, rid, prompt, max_tokens, category):
        return self._disagg(rid, prompt, max_tokens, lambda D, p: -1, from_match=True)

    def _balanced_pd(self, rid, prompt, max_tokens, category):
        r = self.params["ratio"]

        def end_of(D, p):
            n = len(p)
            m = D.cache.MatchPrefix(p[:n - 1])
            s = max(m, int((1.0 - r) * n))  # floor, clamped below by match_len
            return max(1, min(s, n - 1))

        return self._disagg(rid, prompt, max_tokens, end_of, from_match=True)

    def _context_migration(self, rid, prompt, max_tokens, category):
        ctx = self.contexts.get(category) if category is not None else None
        if ctx is None:  # NoOwner: fall back to data-parallel dispatch
            return self._data_parallel(rid, prompt, max_tokens, category)
        load = Counter(rank for _, rank in self.window)
        rank = min(ctx.owners, key=lambda o: (load[o], o))
        self.window.append((category, rank))
        while len(self.window) > self.params["window"]:
            self.window.popleft()
        tokens = self._call(rid, "start_generate", rank, self.engines[rank].api_start_generate,
                            (prompt, 0, max_tokens))
        self._maybe_migrate(rid)
        return tokens

    def _maybe_migrate(self, rid: int) -> None:
        """when per-engine demand over the window is
        imbalanced beyond the threshold, copy the hottest context to the
        idlest engine that lacks it (prep_recv + remote_send)."""
        load = Counter({r: 0 for r in self.ranks})
        load.update(rank for _, rank in self.window)
        hot, cold = max(self.ranks, key=lambda r: (load[r], -r)), min(self.ranks,
                                                                       key=lambda r: (load[r], r))
        if load[hot] <= self.params["threshold"] * max(1, load[cold]) or hot == cold:
            return
        demand = Counter(c for c, r in self.window if r == hot)
        for category, _ in demand.most_common():
            ctx = self.contexts[category]
            if cold in ctx.owners:
                continue
            owner = ctx.owners[0]
            T, O = self.engines[cold], self.engines[owner]
            n = len(ctx.tokens)
            m, addr = self._call(rid, "prep_recv", cold, T.api_prep_recv,
                                 (ctx.tokens, n, False))
            if addr.token_count:
                self._call(rid, "remote_send", owner, O.api_remote_send,
                           (ctx.tokens, m, n, cold, addr))
            T.cache.DrainReceiveCompletions()  # the migrated context enters T's tree
            ctx.owners.append(cold)
            self.migrations += 1
            self.window.clear()  # measure the rebalanced demand afresh
            return
