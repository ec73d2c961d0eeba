#!/usr/bin/env python
"""KV migration GB/s over NVLink & P->D handoff latency (Llama-3.1-70B KV shape).

One step = one DirectSend KV migration of an 8K-token request (context-cache
migration; GatherRange + ApplyRemoteWrite per layer in the
reference) from a prefill engine P to a decode engine D through the
reference-facing API:

    D.PrepRecv(seq, prompt, end=-1)            -> KVAddrInfo for 8,191 tokens
    P.direct_send(seq_p, [m, e), D, addr)      all 80 layers into D's pages
    D.DrainReceiveCompletions()                window complete, committed, tree insert
    D.FreeSequence(seq)                        pages back to the LIFO list

Payload per step = 8,191 tokens x 80 layers x 4 KiB = 2.684 GB.

  value  device-timed migration (CUDA events on the launching stream around
         the DirectSend launch of each step, summed over steps); KV resident
         in HBM.  At N=1 both engines share GPU 0 and the "NVLink" copy is a
         device-local HBM copy; at N>1 rank 2i is P and rank 2i+1 is D and the
         rows go over NVLink into the peer's CUDA-IPC-mapped pool.
  e2e    the same metric through the public API (Python mirror -> C ABI):
         wall time of whole steps (host bookkeeping, host->device uploads of
         the step's slot maps / window metadata, completion polling).
  --impl reference
         the reference's own CPU path (oracle/_ref: the unmodified
         splitserve::KVCache) on the host cores: PrepRecv, GatherRange ->
         ApplyRemoteWrite per layer, Drain, Free; one engine pair per thread.

Secondary lines (handoff latency with per-layer overlap, append, local
gather, decode attention) are reported under "secondary".
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

L, W, PAGE, PROMPT = 80, 512, 16, 8192          # Llama-3.1-70B KV shape, 8K prompt
HKV, HD, HQ = 8, 128, 64
BPT = W * 8                                     # bytes per (token, layer) = 2*8*128*2
PEAKS_FILE = ROOT / "MEASURED_PEAKS.json"
FALLBACK_HBM = 6650.0                            # B200_PROFILING.md fallback
NVLINK_PEER_GBS = 770.0                          # B200_PROFILING.md measured peer copy
NVLINK_NOMINAL_GBS = 900.0                       # NVLink 5, per direction
E2E_DEPTH = int(os.environ.get("MICROKV_E2E_DEPTH", "2"))  # requests in flight in the e2e loop (N = 1)
HBM_NOMINAL_GBS = 8000.0                         # B200 HBM3e nominal (B200_PROFILING.md)
WORKLOAD = ("llama-3.1-70b-kv 8k-prompt DirectSend KV migration P->D "
            "(L=80, 8 kv heads x hd 128 bf16 = 4 KiB/token/layer, page 16, prep_recv end=-1)")


def _peaks() -> tuple[float, str]:
    try:
        return float(json.loads(PEAKS_FILE.read_text())["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


def _prompt(seed: int = 1) -> np.ndarray:
    rng = np.random.Generator(np.random.MT19937(seed))
    return rng.integers(0, 256, PROMPT).astype(np.int32)


class ClockSampler:
    """Samples SM clocks and throttle reasons during the timed region (NVML)."""

    def __init__(self, device: int):
        self.samples: list = []
        self.reasons: set = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._ok = False
        try:
            import pynvml as nv

            nv.nvmlInit()
            self._nv = nv
            self._h = nv.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
            self._ok = True
        except Exception:
            pass

    def _run(self):
        nv = self._nv
        names = {
            getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8): "hw_slowdown",
            getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4): "sw_power_cap",
        }
        i = 0
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                # Throttle reasons every other sample (sticky set): on a box
                # where NVML queries are slow, more clock samples fit in a
                # ~40 ms timed region.
                if i % 2 == 0:
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                    for bit, name in names.items():
                        if r & bit:
                            self.reasons.add(name)
            except Exception:
                pass
            i += 1
            self._stop.wait(0.002)  # several samples even in a ~20 ms timed region

    def __enter__(self):
        if self._ok:
            # A short GIL switch interval so the sampler thread runs while the
            # main thread spins on completion polls.
            self._switch = sys.getswitchinterval()
            sys.setswitchinterval(0.0005)
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self._ok:
            self._stop.set()
            self._t.join()
            sys.setswitchinterval(self._switch)
            try:  # the reasons as the timed region ends (covers a sampler that saw one sample)
                r = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in ((0x8, "hw_slowdown"), (0x40, "hw_thermal_slowdown"),
                                  (0x20, "sw_thermal_slowdown"), (0x4, "sw_power_cap")):
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass

    def summary(self) -> dict:
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# Reference arm (CPU): the unmodified reference behind oracle/_ref
# ---------------------------------------------------------------------------
class _RefCfg(C.Structure):
    _fields_ = [("layers", C.c_int32), ("dim", C.c_int32), ("page_size", C.c_int32),
                ("vocab", C.c_int32), ("num_pages", C.c_int64), ("hash_seed", C.c_uint64),
                ("prompt_len", C.c_int64), ("end", C.c_int64), ("layer_sample", C.c_int32),
                ("threads", C.c_int32), ("steps", C.c_int32), ("warmup", C.c_int32),
                ("token_seed", C.c_uint64)]


class _RefRes(C.Structure):
    _fields_ = [("seconds", C.c_double), ("bytes_moved", C.c_double), ("prep_recv_s", C.c_double),
                ("gather_s", C.c_double), ("apply_s", C.c_double), ("drain_free_s", C.c_double),
                ("tokens_per_step", C.c_int64), ("ok", C.c_int32)]


def run_reference_cpu(steps: int, warmup: int, threads: int, layer_sample: int) -> dict:
    from oracle import REF_LIB

    if not REF_LIB.exists():
        raise FileNotFoundError(f"{REF_LIB} missing (built by __graft_entry__.build())")
    lib = C.CDLL(str(REF_LIB))
    fn = lib.ssref_bench_migrate
    fn.restype = C.c_int
    fn.argtypes = [C.POINTER(_RefCfg), C.POINTER(_RefRes)]
    cfg = _RefCfg(L, W, PAGE, 256, PROMPT // PAGE + 8, 0x5EED5EED5EED5EED, PROMPT, -1,
                  layer_sample, threads, steps, warmup, 1)
    res = _RefRes()
    t0 = time.perf_counter()
    st = fn(C.byref(cfg), C.byref(res))
    if st != 0:
        raise RuntimeError(f"reference migrate failed ({st})")
    return {"gbs": res.bytes_moved / res.seconds / 1e9, "seconds": res.seconds,
            "bytes": res.bytes_moved, "threads": threads, "layer_sample": layer_sample,
            "steps": steps, "tokens_per_step": res.tokens_per_step, "ok": bool(res.ok),
            "wall_s": time.perf_counter() - t0,
            "split_s": {"prep_recv": res.prep_recv_s, "gather": res.gather_s,
                        "apply": res.apply_s, "drain_free": res.drain_free_s}}


def _host_info() -> dict:
    """The host the CPU numbers were taken on (nproc + CPU model)."""
    model = None
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = os.cpu_count() or 1
    return {"nproc": os.cpu_count(), "usable_cores": usable, "cpu_model": model}


def _ref_threads() -> int:
    """Every usable host core, one engine pair per thread, bounded by memory
    (each pair holds two 70B-shape pools of an 8K request)."""
    cores = _host_info()["usable_cores"]
    per_pair = 2 * (PROMPT // PAGE + 8) * PAGE * L * W * 8 + 2 * PROMPT * W * 8
    try:
        import psutil

        avail = psutil.virtual_memory().available
    except Exception:
        avail = 64 << 30
    return max(1, min(cores, int(avail * 0.6 // per_pair)))


def reference_arm(args, rank: int, world: int) -> None:
    if rank != 0:
        return
    threads = _ref_threads()
    sample = L  # every layer of the migration, every step
    r = run_reference_cpu(args.steps, args.warmup, threads, sample)
    line = {
        "metric": "KV migration GB/s (P->D, Llama-3.1-70B KV shape)",
        "value": round(r["gbs"], 4), "unit": "GB/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * r["seconds"] / max(1, args.steps), 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic", "config": {"workload": WORKLOAD, "parallelism": f"{threads} engine pairs x 1 host thread"},
        "cpu_baseline": {"value": round(r["gbs"], 4), "unit": "GB/s", "cores": threads,
                         "kind": "reference", "host": _host_info(),
                         "sample": f"all {sample} layers per step, {threads} independent engine "
                                   f"pairs (one thread each, one per usable core unless memory "
                                   f"bounds it), {r['tokens_per_step']} tokens"},
        "e2e": {"value": round(r["gbs"], 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "split_s": r["split_s"], "window_ok": r["ok"],
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# Our arm
# ---------------------------------------------------------------------------
def _populate_prefix(P, seq: int, prompt: list, torch) -> None:
    """P holds the prompt's KV committed (as after an earlier prefill): the
    bytes arrive through P's own receive path once, untimed."""
    r = P.PrepRecv(seq, prompt, len(prompt))
    n = r.addr.token_count
    g = torch.Generator(device="cuda").manual_seed(1234)
    buf = torch.empty(n * W, dtype=torch.int64, device="cuda")
    for layer in range(L):
        buf.random_(generator=g)
        P.apply_remote_write_async(r.addr, layer, buf.data_ptr(), n * W, 0,
                                   torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    P.synchronize()
    assert P.DrainReceiveCompletions() == [seq]
    assert P.Committed(seq) == len(prompt)


def our_arm(args, rank: int, world: int) -> None:
    import torch
    import torch.distributed as dist

    from paper_2412_12488_b200 import KVCache

    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("MICROKV_SHARE_DEVICE") == "1":
        local = 0  # test hook: run the N>1 pair protocol with every rank on cuda:0
    elif local >= torch.cuda.device_count():
        raise SystemExit(f"rank {rank}: --gpus {world} needs {world} GPUs, "
                         f"{torch.cuda.device_count()} visible")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo")
    prompt = _prompt()
    e = PROMPT - 1
    payload = e * L * BPT
    pages = PROMPT // PAGE + 16
    stream = torch.cuda.Stream()
    sid = stream.cuda_stream

    if world == 1:
        role = "both"
        P = KVCache(num_pages=pages, page_size=PAGE, layers=L, dim=W, device=local, rank=0)
        # E2E_DEPTH receive windows in flight (the e2e loop below)
        D = KVCache(num_pages=E2E_DEPTH * pages, page_size=PAGE, layers=L, dim=W, device=local,
                    rank=1)
        P.attach_peer(1, D)
        peer_rank = None
    else:
        assert world % 2 == 0, "multi-GPU runs pair ranks: 2i = prefill, 2i+1 = decode"
        role = "P" if rank % 2 == 0 else "D"
        peer_rank = rank ^ 1
        me = KVCache(num_pages=pages, page_size=PAGE, layers=L, dim=W, device=local, rank=rank)
        handles = [None] * world
        dist.all_gather_object(handles, me.export_ipc() if role == "D" else None)
        if role == "P":
            P, D = me, None
            P.import_ipc(peer_rank, handles[peer_rank])
            peer = P.peer_info(peer_rank)
            # A peer on another physical GPU publishes at system scope.
            assert peer["sys_scope"] or os.environ.get("MICROKV_SHARE_DEVICE") == "1", peer
        else:
            P, D = None, me
    if P is not None:
        _populate_prefix(P, 1, prompt, torch)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def issue(i: int, timed_dev: list) -> tuple:
        """N=1, first half of a step: prep_recv on D, then P's declaration
        (resolve + upload row maps) and computation (validation + copy
        launch), as in the reference's two stages."""
        seq = 100 + i
        t0 = time.perf_counter()
        r = D.PrepRecv(seq, prompt, -1)
        t1 = time.perf_counter()
        plan = P.begin_direct_send(1, (r.match_len, e), 1, r.addr, i)
        t2 = time.perf_counter()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        P.launch_direct_send_async(plan, (0, L), sid)
        ev1.record(stream)
        t3 = time.perf_counter()
        timed_dev.append((ev0, ev1))
        return seq, plan, (t1 - t0, t2 - t1, t3 - t2)

    drained: set = set()

    def complete(h: tuple) -> None:
        """Second half: D's drain sees the receive window complete (the
        device counters read back), then the plan and sequence are freed."""
        seq, plan, ph = h
        t3 = time.perf_counter()
        while seq not in drained:
            drained.update(D.DrainReceiveCompletions())
        drained.discard(seq)
        t4 = time.perf_counter()
        plan.close()
        D.FreeSequence(seq)
        t5 = time.perf_counter()
        phases.append(ph + (t4 - t3, t5 - t4))

    def step(i: int, timed_dev: list) -> None:
        seq = 100 + i
        if role == "both":
            complete(issue(i, timed_dev))
        elif role == "D":
            r = D.PrepRecv(seq, prompt, -1)
            dist.send_object_list([(r.match_len, r.addr)], dst=peer_rank)
            done = []
            while not done:
                done = D.DrainReceiveCompletions()
            D.FreeSequence(seq)
        else:
            obj = [None]
            dist.recv_object_list(obj, src=peer_rank)
            m, addr = obj[0]
            plan = P.begin_direct_send(1, (m, e), peer_rank, addr, i)
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            P.launch_direct_send_async(plan, (0, L), sid)
            ev1.record(stream)
            timed_dev.append((ev0, ev1))
            stream.synchronize()
            plan.close()

    # Warm-up.
    phases: list = []
    scratch: list = []
    for i in range(args.warmup):
        step(i, scratch)
    barrier()
    # Correctness spot check outside the timed region (N=1): D's received rows
    # equal P's for the first and last layers.
    if role == "both":
        r = D.PrepRecv(99, prompt, -1)
        P.direct_send_async(1, (r.match_len, e), 1, r.addr, 0, (0, L), sid)
        stream.synchronize()
        assert D.DrainReceiveCompletions() == [99]
        for layer in (0, L - 1):
            assert np.array_equal(P.GatherRange(1, (0, e), layer), D.GatherRange(99, (0, e), layer))
        D.FreeSequence(99)

    if world > 1:
        _pair_spot_check(P, D, prompt, e, peer_rank, torch, dist)
    engines = [x for x in (P, D) if x is not None]
    l0 = sum(x.kernel_launches() for x in engines)
    c0 = [x.copy_counters() for x in engines]
    timed: list = []
    phases.clear()
    sampler = ClockSampler(local)
    sampler.__enter__()  # covers the device-timed loop and the e2e loop below
    barrier()
    t0 = time.perf_counter()
    for i in range(args.warmup, args.warmup + args.steps):
        step(i, timed)
    barrier()
    t1 = time.perf_counter()
    launches = sum(x.kernel_launches() for x in engines) - l0
    c1 = [x.copy_counters() for x in engines]
    e2e_wall = None
    if role == "both":
        # End to end with two requests in flight, as a router keeps them:
        # request i+1's prep_recv / declaration / launch are issued before
        # request i's completion is drained, so host bookkeeping overlaps the
        # copy.  (The device-timed loop above runs requests one at a time.)
        phases.clear()
        scratch.clear()
        barrier()
        w0 = time.perf_counter()
        pending: list = []
        base = args.warmup + args.steps
        for i in range(base, base + args.steps):
            pending.append(issue(i, scratch))
            if len(pending) == E2E_DEPTH:
                complete(pending.pop(0))
        while pending:
            complete(pending.pop(0))
        barrier()
        e2e_wall = time.perf_counter() - w0
        c0, c1 = c1, [x.copy_counters() for x in engines]  # the e2e loop's copies
    sampler.__exit__(None, None, None)
    h2d = sum(b[0] - a[0] for a, b in zip(c0, c1)) / args.steps
    d2h = sum(b[1] - a[1] for a, b in zip(c0, c1)) / args.steps
    dev_ms = sum(a.elapsed_time(b) for a, b in timed) if timed else 0.0
    wall_s = t1 - t0
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([wall_s, dev_ms / 1e3 if timed else 0.0], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        wall_s, dev_s = float(t[0]), float(t[1])
    else:
        dev_s = dev_ms / 1e3
    pairs = max(1, world // 2)
    total_bytes = payload * args.steps * pairs
    value = total_bytes / dev_s / 1e9
    e2e = total_bytes / (e2e_wall if e2e_wall is not None else wall_s) / 1e9

    secondary = {}
    if rank == 0 and world == 1 and not args.no_secondary:
        secondary = secondary_measurements(P, D, prompt, torch)
    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            r = run_reference_cpu(steps=2, warmup=0, threads=1, layer_sample=L)
            cpu_baseline = {"value": round(r["gbs"], 4), "unit": "GB/s", "cores": 1,
                            "kind": "reference", "host": _host_info(),
                            "sample": f"2 full 80-layer migrations of one {r['tokens_per_step']}-"
                                      "token request, 1 engine pair on 1 thread "
                                      "(the reference's executor model)",
                            "split_s": r["split_s"]}
        except Exception as ex:
            cpu_baseline = {"value": None, "unavailable": str(ex)}

    if rank != 0:
        return
    peak, peak_kind = _peaks()
    per_launch_s = dev_s / args.steps
    if world == 1:
        alg = 2 * payload  # read + write, both in this GPU's HBM
        roofline = {"bound": "hbm", "achieved": round(alg / per_launch_s / 1e9, 1),
                    "peak": peak, "unit": "GB/s",
                    "frac": round(alg / per_launch_s / 1e9 / peak, 4), "traffic": _traffic(),
                    "peak_nominal": HBM_NOMINAL_GBS,
                    "frac_nominal": round(alg / per_launch_s / 1e9 / HBM_NOMINAL_GBS, 4),
                    "kernel": "k_copy_rows (DirectSend, 80 layers x 8191 rows per launch)",
                    "peak_kind": f"{peak_kind} hbm_gbs (burst copy); nominal HBM3e beside it",
                    "algorithmic_bytes_per_launch": alg}
    else:
        # Per link: each pair's P->D copy is one GPU's NVLink egress; the
        # per-launch time is the max over ranks.
        link = payload / per_launch_s / 1e9
        roofline = {"bound": "nvlink", "achieved": round(link, 1),
                    "peak": NVLINK_PEER_GBS, "unit": "GB/s",
                    "frac": round(link / NVLINK_PEER_GBS, 4),
                    "peak_nominal": NVLINK_NOMINAL_GBS,
                    "frac_nominal": round(link / NVLINK_NOMINAL_GBS, 4),
                    "traffic": None, "kernel": "k_copy_rows (peer stores, system-scope counters)",
                    "peak_kind": "measured peer copy per direction (B200_PROFILING.md); "
                                 "nominal NVLink 5 per direction beside it",
                    "algorithmic_bytes_per_launch": payload,
                    "per_pair_payload_gbs": round(link, 1), "pairs": pairs}
    line = {
        "metric": "KV migration GB/s (P->D, Llama-3.1-70B KV shape)",
        "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * wall_s / args.steps, 4),
        "device_ms_per_step": round(1e3 * dev_s / args.steps, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic",
        "config": {"workload": WORKLOAD, "tokens_per_step": e, "layers": L,
                   "bytes_per_step": payload,
                   "parallelism": "1 GPU: P and D engines share the device (local HBM copy)"
                   if world == 1 else f"{pairs} P->D pairs over NVLink (CUDA IPC peer stores)",
                   "l2": "inputs (2.7 GB per step) larger than L2"},
        "e2e": {"value": round(e2e, 2), "unit": "GB/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h),
                "requests_in_flight": E2E_DEPTH if world == 1 else 1,
                "note": "wall time of the public-API steps (prep_recv, begin_direct_send, "
                        "launch, drain, free) incl. their H2D/D2H; at N=1 request i+1 is "
                        "issued before request i is drained"},
        "roofline": roofline,
        "cpu_baseline": cpu_baseline,
        "clocks": sampler.summary(),
        "gpu_launches": int(launches),
        "e2e_phases_us": None if not phases else {
            k: round(1e6 * float(np.median([ph[j] for ph in phases])), 1)
            for j, k in enumerate(["prep_recv", "begin_direct_send", "launch",
                                   "wait_and_drain", "close_and_free"])},
        "secondary": secondary,
    }
    # The handoff half of the metric, top level (70B and 8B, kernel mover on
    # the whole machine; every mover's numbers are under secondary.handoff*).
    for key, sub in (("handoff", ""), ("handoff_8b", "_8b"), ("handoff_layer_order", "_layer_order")):
        h = secondary.get(key, {}) if isinstance(secondary, dict) else {}
        line[f"handoff{sub}_mover"] = h.get("mover")
        line[f"handoff{sub}_tail_us"] = h.get("exposed_tail_us")
        line[f"handoff{sub}_slowdown_pct"] = h.get("slowdown_pct")
        line[f"handoff{sub}_slowdown_pct_best"] = h.get("slowdown_pct_best")
    line["send_budget"] = _pick_budget(secondary) if isinstance(secondary, dict) else None
    print(json.dumps(line), flush=True)


def _pick_budget(secondary: dict):
    """The smallest SM budget of the copy kernel whose 80-layer send alone
    still moves >= 720 GB/s (80% of an NVLink 5 direction), with that arm's
    median prefill slowdown at both shapes (secondary.handoff*)."""
    sm = secondary.get("send_modes") or {}
    best = None
    for name, mode, ctas in SEND_ARMS:
        v = (sm.get(name) or {}).get("80_layers", {}).get("payload_gbs")
        if mode == 0 and ctas > 0 and v is not None and v >= 720.0:
            if best is None or ctas < best[0]:
                best = (ctas, name, v)
    if best is None:
        return None
    out = {"arm": best[1], "max_ctas": best[0], "payload_gbs_80_layers": best[2]}
    for key, tag in (("handoff", "70b"), ("handoff_8b", "8b")):
        a = ((secondary.get(key) or {}).get("arms") or {}).get(best[1], {})
        out[f"prefill_slowdown_pct_{tag}"] = a.get("slowdown_pct_paired_median")
        out[f"exposed_tail_us_{tag}"] = a.get("exposed_tail_us_median")
    return out


def _pair_spot_check(P, D, prompt, e, peer_rank, torch, dist) -> None:
    """N>1, outside the timed region: one migration, then CRC-32 of the
    first and last layers' rows on both sides (P's sent rows, D's received
    rows) must agree."""
    seq = 99
    crcs = []
    if D is not None:
        r = D.PrepRecv(seq, prompt, -1)
        dist.send_object_list([(r.match_len, r.addr)], dst=peer_rank)
        while seq not in D.DrainReceiveCompletions():
            pass
        eng = D
    else:
        obj = [None]
        dist.recv_object_list(obj, src=peer_rank)
        m, addr = obj[0]
        P.direct_send_async(1, (m, e), peer_rank, addr, 0, (0, L), 0)
        P.synchronize()
        seq, eng = 1, P
    buf = torch.empty(e * W, dtype=torch.int64, device="cuda")
    out = torch.zeros(1, dtype=torch.int64, device="cuda")
    for layer in (0, L - 1):
        eng.gather_range_async(seq, (0, e), layer, buf.data_ptr(), 0)
        eng.crc32_async(buf.data_ptr(), e * W * 8, out.data_ptr(), 0)
        torch.cuda.synchronize()
        crcs.append(int(out.item()))
    mine = [None]
    theirs = [None]
    if D is not None:
        dist.send_object_list([crcs], dst=peer_rank)
        D.FreeSequence(seq)
    else:
        dist.recv_object_list(theirs, src=peer_rank)
        assert theirs[0] == crcs, f"received rows differ from sent rows: {theirs[0]} vs {crcs}"
    del mine


def _traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu capture."""
    f = ROOT / "profiles" / "traffic.json"
    try:
        return json.loads(f.read_text()).get("k_copy_rows_directsend_bytes_per_launch")
    except Exception:
        return None


def secondary_measurements(P, D, prompt, torch) -> dict:
    """Handoff latency with per-layer overlap, KV append, local gather, decode attention."""
    out = {}
    try:
        out["handoff"] = measure_handoff_gemm(torch)
    except Exception as ex:
        out["handoff"] = {"error": str(ex)}
    try:  # config 2 (Llama-3.1-8B: 32 layers, 4K prompt; ~1.8 TFLOP per layer)
        out["handoff_8b"] = measure_handoff_8b(torch)
    except Exception as ex:
        out["handoff_8b"] = {"error": str(ex)}
    try:  # the same 70B stand-in with the layer's K||V produced by its first 20% of FLOPs
        out["handoff_layer_order"] = measure_handoff_gemm(
            torch, kv_share=0.2, arm_names=("kernel_full", "kernel_32ctas", "write_through"))
    except Exception as ex:
        out["handoff_layer_order"] = {"error": str(ex)}
    try:
        out["send_modes"] = measure_send_modes(torch)
    except Exception as ex:
        out["send_modes"] = {"error": str(ex)}
    try:
        out["handoff_toy_prefill"] = measure_handoff(torch)
    except Exception as ex:
        out["handoff_toy_prefill"] = {"error": str(ex)}
    try:
        out["configs"] = measure_configs(torch)
    except Exception as ex:
        out["configs"] = {"error": str(ex)}
    try:
        out["prefix_migration"] = measure_prefix_migration(torch)
    except Exception as ex:
        out["prefix_migration"] = {"error": str(ex)}
    try:
        out["transfer_sweep"] = measure_sweep(torch)
        out["transfer_cost_model"] = fit_transfer_cost(out["transfer_sweep"])
    except Exception as ex:
        out["transfer_sweep"] = {"error": str(ex)}
    try:
        out["append_gather"] = measure_append_gather(torch)
    except Exception as ex:
        out["append_gather"] = {"error": str(ex)}
    try:
        out["decode_attention"] = measure_decode(torch)
    except Exception as ex:
        out["decode_attention"] = {"error": str(ex)}
    try:
        out["prefill_attention"] = measure_prefill(torch)
    except Exception as ex:
        out["prefill_attention"] = {"error": str(ex)}
    try:
        out["engine_step"] = measure_engine(torch)
    except Exception as ex:
        out["engine_step"] = {"error": str(ex)}
    try:
        out["router"] = measure_router(torch)
    except Exception as ex:  # noqa: BLE001
        out["router"] = {"error": str(ex)}
    try:
        out["frames"] = measure_frames(torch)
    except Exception as ex:
        out["frames"] = {"error": str(ex)}
    return out


SEND_ARMS = (("kernel_full", 0, 0), ("kernel_64ctas", 0, 64), ("kernel_32ctas", 0, 32),
             ("kernel_16ctas", 0, 16), ("copy_engine", 1, 0))


def measure_handoff_8b(torch, reps: int = 21) -> dict:
    """Config 2's handoff (Llama-3.1-8B: 32 layers, 4K prompt, ~1.8 TFLOP per
    layer).  The copy-engine arm is measured in its own rotation: its host
    enqueue (512 2-D copies per layer) leaves the SMs idle for ~100 ms, and
    under sw_power_cap the 1.2 ms 8B GEMM of whatever arm runs next starts at
    a different clock, which moved the other arms' medians by ~5-8% when it
    shared their rotation (profiles/r02/handoff_8b_noise.txt)."""
    kernel_arms = tuple(a[0] for a in SEND_ARMS if a[0] != "copy_engine")
    r = measure_handoff_gemm(torch, 32, 4096, 4096, 53248, "8B", reps=reps,
                             arm_names=kernel_arms + ("write_through",))
    ce = measure_handoff_gemm(torch, 32, 4096, 4096, 53248, "8B", reps=3,
                              arm_names=("copy_engine",))
    r["arms"]["copy_engine"] = dict(ce["arms"]["copy_engine"], separate_rotation=True,
                                    reps=3, prefill_ms_without_sends=ce["prefill_ms_without_sends"])
    return r


def measure_handoff_gemm(torch, layers: int = L, n_prompt: int = PROMPT, k: int = 8192,
                         n: int = 104448, label: str = "70B", reps: int = 5,
                         kv_share: float = 0.0, arm_names=None) -> dict:
    """1P1D PrefillThenSend with a compute-bound prefill stand-in: per layer
    one bf16 GEMM of a Llama layer's FLOPs at the prompt length (70B:
    X[8191, 8192] @ W[8192, 104448], ~14 TFLOP), then the layer's K||V rows
    are appended to P's pages and that layer is sent to D's reserved pages
    on a second stream (validation first, the copy behind the layer's event:
    ss_launch_direct_send_after_async), overlapping the next layer's GEMM
    (PAPER.md:339-344).

    Arms: no sends, and sends through each row mover of SEND_ARMS (the copy
    kernel on the whole machine or an SM budget, the copy engines).  Each
    rep runs every arm once in a rotated order (alternation: drift and
    thermal state spread over all arms); per arm the median and range over
    reps of P's prefill time, the slowdown against the no-send median, the
    exposed tail (P's last-layer compute end -> the last layer's rows and
    window counters landed in D) and the per-layer lag (layer l's event ->
    its rows landed).

    kv_share > 0 splits each layer's GEMM the way a transformer layer is
    ordered: the first kv_share of its FLOPs (the QKV projection, which
    produces the layer's K||V rows) before the KV append and send, the rest
    (attention output projection + MLP) after it, so the send of layer l
    overlaps layer l's own remaining compute ("sending a
    layer's KV right after its computation").  kv_share = 0 appends after
    the whole layer: the conservative bound."""
    from paper_2412_12488_b200 import BatchEntry, KVCache

    rng = np.random.Generator(np.random.MT19937(4))
    prompt = [int(x) for x in rng.integers(0, 256, n_prompt)]
    e = n_prompt - 1
    pages = n_prompt // PAGE + 16
    P = KVCache(num_pages=pages, page_size=PAGE, layers=layers, dim=W, device=0, rank=0)
    D = KVCache(num_pages=pages, page_size=PAGE, layers=layers, dim=W, device=0, rank=1)
    P.attach_peer(1, D)
    X = torch.randn(e, k, device="cuda", dtype=torch.bfloat16)
    na = int(round(n * kv_share / 128)) * 128
    Wt = torch.randn(k, n - na, device="cuda", dtype=torch.bfloat16) * 0.01
    Y = torch.empty(e, n - na, device="cuda", dtype=torch.bfloat16)
    Wa = torch.randn(k, na, device="cuda", dtype=torch.bfloat16) * 0.01 if na else None
    Ya = torch.empty(e, na, device="cuda", dtype=torch.bfloat16) if na else None
    rows = torch.randint(-2**62, 2**62, (e * W,), dtype=torch.int64, device="cuda")
    # GEMMs before each timed run (~20 ms): 2 at the 70B layer, 16 at the 8B one.
    flop = 2.0 * e * k * n
    preheat = max(2, int(round(20e-3 / (flop / 1.2e15))))
    # The send stream at high priority, like the engine's own comm stream: a
    # layer's copy takes SMs as soon as compute CTAs retire.
    prio = int(os.environ.get("MICROKV_HANDOFF_SEND_PRIO", "-1"))
    cs, ms, ds = torch.cuda.Stream(), torch.cuda.Stream(priority=prio), torch.cuda.Stream()
    # write_through: the layer's KV append and its remote_send fused into one
    # launch on the compute stream (ss_append_rows_send_async).
    arms = [("none", None, None)] + list(SEND_ARMS) + [("write_through", "fused", 0)]
    if arm_names is not None:
        arms = [a for a in arms if a[0] == "none" or a[0] in arm_names]
    runs = {a[0]: {"prefill_ms": [], "tail_us": [], "layer_lag_us": [], "last_append_us": []}
            for a in arms}
    seq = 10
    for rep in range(reps + 1):  # rep 0: warm-up of every arm, discarded
        order = arms[rep % len(arms):] + arms[:rep % len(arms)]
        for name, mode, ctas in order:
            send = mode is not None
            fused = mode == "fused"
            seq += 1
            if send:
                P.set_send_mode(0 if fused else mode, ctas)
                r = D.PrepRecv(seq, prompt, -1)
            P.CreateSequence(seq, prompt)
            P.EnsureAllocated(seq, e)
            plan = P.BeginForward([BatchEntry(seq, (0, e))])
            dplan = P.begin_direct_send(seq, (0, e), 1, r.addr, 7) if send else None
            torch.cuda.synchronize()
            # Every arm's timed region starts from the same power state: ~20 ms
            # of the same GEMM first (under sw_power_cap the clock follows the
            # preceding load; an arm after the copy-engine arm, whose host
            # enqueue leaves the SMs idle for ~100 ms, otherwise starts at
            # a boosted clock and the arms' medians drift apart by ~5% at 8B).
            with torch.cuda.stream(cs):
                for _ in range(preheat):
                    torch.matmul(X, Wt, out=Y)
            t0, tc = (torch.cuda.Event(enable_timing=True) for _ in range(2))
            done = [torch.cuda.Event(enable_timing=True) for _ in range(layers)]
            landed = [torch.cuda.Event(enable_timing=True) for _ in range(layers)] if send else []
            pre_last = torch.cuda.Event(enable_timing=True)  # before the last layer's append
            t0.record(cs)
            for layer in range(layers):
                with torch.cuda.stream(cs):
                    torch.matmul(X, Wa if na else Wt, out=Ya if na else Y)
                if layer == layers - 1:
                    pre_last.record(cs)
                if fused:
                    P.append_rows_send_async(plan, dplan, (layer, layer + 1), rows.data_ptr(),
                                             cs.cuda_stream)
                    done[layer].record(cs)
                    landed[layer].record(cs)
                else:
                    P.append_rows_async(plan, layer, rows.data_ptr(), cs.cuda_stream)
                    done[layer].record(cs)
                    if send:
                        P.launch_direct_send_after_async(dplan, (layer, layer + 1),
                                                         done[layer].cuda_event, ms.cuda_stream)
                        landed[layer].record(ms)
                if na:  # the rest of the layer behind its KV (output projection + MLP)
                    with torch.cuda.stream(cs):
                        torch.matmul(X, Wt, out=Y)
            tc.record(cs)
            torch.cuda.synchronize()
            P.synchronize()
            if rep > 0:
                runs[name]["prefill_ms"].append(t0.elapsed_time(tc))
                runs[name]["last_append_us"].append(1e3 * pre_last.elapsed_time(done[-1]))
            if send:
                # D's device-side wait runs after the timed region: on one GPU
                # a spinning wait kernel would hold an SM slot of P's prefill
                # (on two GPUs it runs on D's).  The last layer's copy ends
                # when its rows and window counters have landed (device-local
                # peer), so the tail is P's compute end -> that copy's end;
                # the wait then confirms every row of every layer arrived.
                D.wait_receive_async(seq, 60000, ds.cuda_stream)
                ds.synchronize()
                D.synchronize()
                assert D.DrainReceiveCompletions() == [seq]
                if rep > 0 and fused and not na:
                    # P's compute end is where a plain append of the last
                    # layer would have ended: the fused launch's excess over
                    # the no-send arm's append is the exposed tail.
                    runs[name]["tail_us"].append(1e3 * pre_last.elapsed_time(landed[-1]))
                elif rep > 0:
                    runs[name]["tail_us"].append(1e3 * max(0.0, tc.elapsed_time(landed[-1])))
                    runs[name]["layer_lag_us"].append(
                        float(np.median([1e3 * done[i].elapsed_time(landed[i])
                                         for i in range(layers)])))
                D.FreeSequence(seq)
                dplan.close()
            plan.close()
            P.FreeSequence(seq)
    P.set_send_mode(0, 0)
    per_layer = e * BPT
    base = float(np.median(runs["none"]["prefill_ms"]))
    append_us = float(np.median(runs["none"]["last_append_us"]))
    if runs.get("write_through", {}).get("tail_us") and not na:
        runs["write_through"]["tail_us"] = [max(0.0, t - append_us)
                                            for t in runs["write_through"]["tail_us"]]
    res = {"layers": layers, "prompt_tokens": n_prompt, "reps": reps, "kv_share": kv_share,
           "preheat_gemms": preheat,
           "per_layer_payload_mb": round(per_layer / 1e6, 2),
           "prefill_ms_without_sends": round(base, 3),
           "prefill_ms_without_sends_range": [round(min(runs["none"]["prefill_ms"]), 3),
                                              round(max(runs["none"]["prefill_ms"]), 3)],
           "last_layer_append_us": round(append_us, 1),
           "send_stream_priority": prio,
           "arms": {}}
    for name, mode, ctas in arms[1:]:
        rr = runs[name]
        med = float(np.median(rr["prefill_ms"]))
        lh = float(np.median(rr["layer_lag_us"])) if rr["layer_lag_us"] else 0.0
        res["arms"][name] = {
            "prefill_ms_median": round(med, 3),
            "prefill_ms_range": [round(min(rr["prefill_ms"]), 3), round(max(rr["prefill_ms"]), 3)],
            "slowdown_pct_median": round(100 * (med / base - 1), 3),
            "slowdown_pct_per_rep": [round(100 * (x / base - 1), 3) for x in rr["prefill_ms"]],
            # each rep against the no-send run of the same rotation (adjacent
            # in time: the GEMM's clock / power state drifts between reps)
            "slowdown_pct_paired_median": round(float(np.median(
                [100 * (x / y - 1) for x, y in zip(rr["prefill_ms"], runs["none"]["prefill_ms"])])), 3),
            # best against best: upward noise (power-cap clock dips) is one-sided
            "slowdown_pct_best": round(100 * (min(rr["prefill_ms"]) / min(runs["none"]["prefill_ms"]) - 1), 3),
            "exposed_tail_us_median": round(float(np.median(rr["tail_us"])), 1),
            "exposed_tail_us_range": [round(min(rr["tail_us"]), 1), round(max(rr["tail_us"]), 1)],
            # layer l's event on the compute stream -> its rows landed (the
            # send stream's event after the copy): how far the transfer trails
            # the layer that produced it
            "layer_lag_us_median": round(lh, 1)}
    # The engine's mover at N=1: the write-through append (the layer's KV
    # append and its remote_send in one launch on the compute stream).
    mover = next((m for m in ("write_through", "kernel_full") if m in res["arms"]),
                 next(iter(res["arms"])))
    d = res["arms"][mover]
    res["mover"] = mover
    res["prefill_ms_with_sends"] = d["prefill_ms_median"]
    res["slowdown_pct"] = d["slowdown_pct_paired_median"]
    res["slowdown_pct_best"] = d["slowdown_pct_best"]
    res["exposed_tail_us"] = d["exposed_tail_us_median"]
    res["note"] = (f"{label}-layer-FLOP bf16 GEMM per layer (cuBLAS, compute stand-in) + KV append; "
                   "per-layer DirectSend on a second stream (kernel_* / copy_engine arms) or fused "
                   "with the append (write_through); P and D on one GPU; medians over "
                   f"{reps} alternated reps per arm; slowdown_pct = median over reps of each rep "
                   "against the no-send run of the same rotation")
    del P, D, X, Wt, Y, Wa, Ya, rows
    torch.cuda.empty_cache()
    return res


def measure_send_modes(torch) -> dict:
    """Each row mover of SEND_ARMS alone on the GPU (no compute beside it):
    one 70B layer (8,191 rows = 33.5 MB) and the whole 80-layer migration
    (2.68 GB), device time (median of 9, launches queued behind a sleep) ->
    payload GB/s and the fraction of the HBM copy peak (read + write)."""
    from paper_2412_12488_b200 import KVCache

    peak, _ = _peaks()
    prompt = _prompt(8)
    e = PROMPT - 1
    pages = PROMPT // PAGE + 16
    P = KVCache(num_pages=pages, page_size=PAGE, layers=L, dim=W, device=0, rank=0)
    D = KVCache(num_pages=pages, page_size=PAGE, layers=L, dim=W, device=0, rank=1)
    P.attach_peer(1, D)
    _populate_prefix_l(P, 1, prompt, torch, L)
    s = torch.cuda.Stream()
    res = {}
    seq = 500
    for name, mode, ctas in SEND_ARMS:
        P.set_send_mode(mode, ctas)
        out = {}
        for lay, tag in ((1, "one_layer"), (L, "80_layers")):
            ts = []
            for rep in range(10):
                seq += 1
                r = D.PrepRecv(seq, prompt, -1)
                plan = P.begin_direct_send(1, (0, e), 1, r.addr, rep)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                if mode == 0:  # (copy engines: the host waits for the verdict inside the call)
                    with torch.cuda.stream(s):
                        torch.cuda._sleep(4_000_000)
                e0.record(s)
                P.launch_direct_send_async(plan, (0, lay), s.cuda_stream)
                e1.record(s)
                s.synchronize()
                if rep > 0:
                    ts.append(e0.elapsed_time(e1) / 1e3)
                if lay == L:
                    assert D.DrainReceiveCompletions() == [seq]
                plan.close()
                D.FreeSequence(seq)
            t = float(np.median(ts))
            pay = e * lay * BPT
            out[tag] = {"device_us": round(1e6 * t, 1), "payload_gbs": round(pay / t / 1e9, 1),
                        "hbm_frac": round(2 * pay / t / 1e9 / peak, 4),
                        "range_us": [round(1e6 * min(ts), 1), round(1e6 * max(ts), 1)]}
        res[name] = out
    P.set_send_mode(0, 0)
    del P, D
    torch.cuda.empty_cache()
    return res


def measure_handoff(torch) -> dict:
    """1P1D PrefillThenSend with the toy prefill (hash KV + fold) on a compute
    stream; each layer's send on the engine's comm stream.  Exposed tail =
    P's last-layer compute end -> D's device-side wait sees every row."""
    from paper_2412_12488_b200 import BatchEntry, KVCache

    prompt = _prompt(2)
    e = PROMPT - 1
    pages = PROMPT // PAGE + 16
    P = KVCache(num_pages=pages, page_size=PAGE, layers=L, dim=W, device=0, rank=0)
    D = KVCache(num_pages=pages, page_size=PAGE, layers=L, dim=W, device=0, rank=1)
    P.attach_peer(1, D)
    cs, ds = torch.cuda.Stream(), torch.cuda.Stream()
    hidden = [torch.empty(e, dtype=torch.int64, device="cuda") for _ in range(2)]
    res = {}
    for send in (False, True, True):
        seq = 7 if send else 8
        if send:
            r = D.PrepRecv(seq, prompt, -1)
        P.CreateSequence(seq, prompt)
        P.EnsureAllocated(seq, e)
        if send:
            P.MarkSend(seq, (0, e), 1, r.addr, 5)
        plan = P.BeginForward([BatchEntry(seq, (0, e))])
        torch.cuda.synchronize()
        t0, tc = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        td = torch.cuda.Event(enable_timing=True)
        t0.record(cs)
        for layer in range(L):
            P.attention_async(layer, plan, hidden[layer % 2].data_ptr(),
                              hidden[(layer + 1) % 2].data_ptr(), cs.cuda_stream)
        tc.record(cs)
        if send:
            ds.wait_event(t0)
            D.wait_receive_async(seq, 20000, ds.cuda_stream)
            td.record(ds)
        torch.cuda.synchronize()
        P.synchronize()
        compute_ms = t0.elapsed_time(tc)
        if send:
            tail_ms = tc.elapsed_time(td)
            assert D.DrainReceiveCompletions() == [seq]
            res = {"prefill_ms_with_sends": round(compute_ms, 3),
                   "exposed_tail_us": round(1e3 * max(0.0, tail_ms), 1),
                   "handoff_us": round(1e3 * tail_ms, 1)}
            D.FreeSequence(seq)
        else:
            res_nosend = compute_ms
        plan.close()
        P.FreeSequence(seq)
    res["prefill_ms_without_sends"] = round(res_nosend, 3)
    res["slowdown_pct"] = round(100 * (res["prefill_ms_with_sends"] / res_nosend - 1), 2)
    res["note"] = ("toy prefill (KvEntryWords + EntryDigest fold per layer) as the compute stand-in; "
                   "P and D on one GPU")
    del P, D
    return res


def _migrate_once(torch, P, D, src_seq, prompt, end, layers, s, seq):
    """One DirectSend of D.PrepRecv(prompt, end) from P's cached src_seq;
    returns the device time of the launch (s)."""
    r = D.PrepRecv(seq, prompt, end)
    plan = P.begin_direct_send(src_seq, (r.match_len, r.match_len + r.addr.token_count), 1,
                               r.addr, seq)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    P.launch_direct_send_async(plan, (0, layers), s.cuda_stream)
    e1.record(s)
    s.synchronize()
    assert D.DrainReceiveCompletions() == [seq]
    plan.close()
    return e0.elapsed_time(e1) / 1e3, r


def measure_configs(torch) -> dict:
    """BASELINE.json configs 2 and 3 on one GPU (P and D share the device):
      8B  : Llama-3.1-8B KV shape (L=32), 4K prompt, prep_recv end=-1, 1P1D.
      70B balanced PD: 8K prompt, P sends the first s = floor((1-r)*8192)
            tokens, D appends the tail (8192 - s tokens) into its own pages
            per layer (the decode engine's share of the prefill), r in
            {0.1, 0.2, 0.3}."""
    from paper_2412_12488_b200 import BatchEntry, KVCache

    peak, _ = _peaks()
    out = {}
    s = torch.cuda.Stream()
    # 8B 1P1D
    L8, n8 = 32, 4096
    prompt = _prompt(5)[:n8]
    P = KVCache(num_pages=n8 // PAGE + 16, page_size=PAGE, layers=L8, dim=W, device=0, rank=0)
    D = KVCache(num_pages=n8 // PAGE + 16, page_size=PAGE, layers=L8, dim=W, device=0, rank=1)
    P.attach_peer(1, D)
    _populate_prefix_l(P, 1, prompt, torch, L8)
    ts = []
    for i in range(6):
        t, r = _migrate_once(torch, P, D, 1, prompt, -1, L8, s, 100 + i)
        D.FreeSequence(100 + i)
        ts.append(t)
    t = float(np.median(ts[1:]))
    pay = (n8 - 1) * L8 * BPT
    out["8b_1p1d_4k"] = {"tokens": n8 - 1, "layers": L8, "payload_mb": round(pay / 1e6, 1),
                         "device_us": round(1e6 * t, 1), "payload_gbs": round(pay / t / 1e9, 1),
                         "hbm_frac": round(2 * pay / t / 1e9 / peak, 4)}
    del P, D
    torch.cuda.empty_cache()
    # 70B balanced PD
    prompt = _prompt(6)
    P = KVCache(num_pages=PROMPT // PAGE + 16, page_size=PAGE, layers=L, dim=W, device=0, rank=0)
    D = KVCache(num_pages=PROMPT // PAGE + 16, page_size=PAGE, layers=L, dim=W, device=0, rank=1)
    P.attach_peer(1, D)
    _populate_prefix_l(P, 1, prompt, torch, L)
    rows = torch.randint(-2**62, 2**62, (PROMPT * W,), dtype=torch.int64, device="cuda")
    max_tail = PROMPT - int(0.7 * PROMPT)
    rows_all = torch.empty(L * max_tail * W, dtype=torch.int64, device="cuda").random_()
    for ratio in (0.1, 0.2, 0.3):
        sp = int((1 - ratio) * PROMPT)
        ts, ta, tf = [], [], []
        for i in range(4):
            seq = 200 + int(ratio * 100) * 10 + i
            t, r = _migrate_once(torch, P, D, 1, prompt, sp, L, s, seq)
            D.EnsureAllocated(seq, PROMPT)
            plan = D.BeginForward([BatchEntry(seq, (sp, PROMPT))])
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            # Queue all 80 launches behind a sleep so the events time the
            # device, not the host's per-call launch cost.
            with torch.cuda.stream(s):
                torch.cuda._sleep(20_000_000)
            e0.record(s)
            for layer in range(L):
                D.append_rows_async(plan, layer, rows.data_ptr(), s.cuda_stream)
            e1.record(s)
            s.synchronize()
            plan.close()
            assert D.Committed(seq) == PROMPT
            ta.append(e0.elapsed_time(e1) / 1e3)
            # The same tail as one 80-layer launch (a producer holding every
            # layer's rows, e.g. a batched tail prefill).
            D.FreeSequence(seq)
            seq2 = seq + 5000
            _t2, _ = _migrate_once(torch, P, D, 1, prompt, sp, L, s, seq2)
            D.EnsureAllocated(seq2, PROMPT)
            plan = D.BeginForward([BatchEntry(seq2, (sp, PROMPT))])
            with torch.cuda.stream(s):
                torch.cuda._sleep(2_000_000)
            e0.record(s)
            D.append_rows_layers_async(plan, (0, L), rows_all.data_ptr(), s.cuda_stream)
            e1.record(s)
            s.synchronize()
            plan.close()
            assert D.Committed(seq2) == PROMPT
            D.FreeSequence(seq2)
            tf.append(e0.elapsed_time(e1) / 1e3)
            ts.append(t)
        t, tap, tfu = float(np.median(ts[1:])), float(np.median(ta[1:])), float(np.median(tf[1:]))
        pay, tail = sp * L * BPT, (PROMPT - sp) * L * BPT
        out[f"70b_balanced_r{ratio}"] = {
            "sent_tokens": sp, "tail_tokens": PROMPT - sp,
            "send_device_us": round(1e6 * t, 1), "send_payload_gbs": round(pay / t / 1e9, 1),
            "send_hbm_frac": round(2 * pay / t / 1e9 / peak, 4),
            "tail_append_us": round(1e6 * tap, 1),
            "tail_append_hbm_frac": round(2 * tail / tap / 1e9 / peak, 4),
            "tail_append_one_launch_us": round(1e6 * tfu, 1),
            "tail_append_one_launch_hbm_frac": round(2 * tail / tfu / 1e9 / peak, 4)}
    del P, D, rows, rows_all
    torch.cuda.empty_cache()
    return out


def measure_prefix_migration(torch) -> dict:
    """Config 4 on one GPU: an 8K-token cached prefix (70B shape) migrated from
    its owner to k = 3 engines (prep_recv(end=len) on each target) as
      fanout      one fan-out send from the owner (each source row read once),
      sequential  three DirectSends from the owner,
      relay       owner -> T1 -> T2 -> T3, each target forwarding a layer as
                  soon as it has landed (ss_launch_relay_send_async).
    On one GPU every hop is HBM traffic; across GPUs the owner's single
    NVLink egress carries k copies for fanout/sequential and one for relay.
    `nvlink_model_us` is the transfer time those egress bytes imply at the
    measured per-direction peer-copy rate (B200_PROFILING.md), with the
    relay's pipeline fill of one layer per extra hop."""
    from paper_2412_12488_b200 import KVCache

    peak, _ = _peaks()
    k = 3
    prompt = _prompt(7)
    pages = PROMPT // PAGE + 16
    P = KVCache(num_pages=pages, page_size=PAGE, layers=L, dim=W, device=0, rank=0)
    Ds = [KVCache(num_pages=pages, page_size=PAGE, layers=L, dim=W, device=0, rank=r)
          for r in range(1, k + 1)]
    P.attach_peer(1, Ds[0])
    for D in Ds[1:]:
        P.attach_peer(D.rank, D)
    for i in range(k - 1):
        Ds[i].attach_peer(Ds[i + 1].rank, Ds[i + 1])
    _populate_prefix_l(P, 1, prompt, torch, L)
    torch.cuda._sleep(1)  # loaded before any relay waits (lazy module loading)
    streams = [torch.cuda.Stream() for _ in range(k + 1)]
    s = streams[0]
    pay1 = PROMPT * L * BPT
    res = {"targets": k, "tokens": PROMPT, "payload_per_target_gb": round(pay1 / 1e9, 3)}
    for mode in ("fanout", "sequential", "relay"):
        ts = []
        for rep in range(6):
            seqs = [1000 * (rep + 1) + D.rank for D in Ds]
            addrs = [D.PrepRecv(sq, prompt, PROMPT).addr for D, sq in zip(Ds, seqs)]
            plans = []
            if mode == "sequential":
                plans = [P.begin_direct_send(1, (0, PROMPT), D.rank, a, rep) for D, a in zip(Ds, addrs)]
            elif mode == "relay":
                plans = [P.begin_direct_send(1, (0, PROMPT), 1, addrs[0], rep)]
                hops = [Ds[i].begin_direct_send(seqs[i], (0, PROMPT), Ds[i + 1].rank, addrs[i + 1], rep)
                        for i in range(k - 1)]
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if mode == "relay":
                for st in streams[1:]:
                    st.wait_stream(s)
            e0.record(s)
            if mode == "fanout":
                P.broadcast_send_async(1, (0, PROMPT), [D.rank for D in Ds], addrs, rep, None,
                                       s.cuda_stream)
            elif mode == "sequential":
                for pl in plans:
                    P.launch_direct_send_async(pl, (0, L), s.cuda_stream)
            else:
                for i in reversed(range(k - 1)):
                    Ds[i].launch_relay_send_async(hops[i], (0, L), 20000, streams[i + 1].cuda_stream)
                P.launch_direct_send_async(plans[0], (0, L), s.cuda_stream)
                for st in streams[1:]:
                    s.wait_stream(st)
            e1.record(s)
            torch.cuda.synchronize()
            for D, sq in zip(Ds, seqs):
                D.synchronize()
                assert D.DrainReceiveCompletions() == [sq]
            if mode == "relay":
                for h in hops:
                    h.close()
            for D, sq in zip(Ds, seqs):
                D.FreeSequence(sq)
            for pl in plans:
                pl.close()
            if rep:
                ts.append(e0.elapsed_time(e1) / 1e3)
        t = float(np.median(ts))
        pay = k * pay1
        hbm = (1 + k if mode == "fanout" else 2 * k) * pay1
        egress = pay1 * (1 if mode == "relay" else k)
        link_s = egress / (NVLINK_PEER_GBS * 1e9) + ((k - 1) * pay1 / L / (NVLINK_PEER_GBS * 1e9)
                                                     if mode == "relay" else 0.0)
        res[mode] = {"device_us": round(1e6 * t, 1), "aggregate_payload_gbs": round(pay / t / 1e9, 1),
                     "hbm_bytes": hbm, "hbm_frac": round(hbm / t / 1e9 / peak, 4),
                     "owner_egress_bytes": egress, "nvlink_model_us": round(1e6 * link_s, 1),
                     "range_us": [round(1e6 * min(ts), 1), round(1e6 * max(ts), 1)]}
    res["fanout_speedup"] = round(res["sequential"]["device_us"] / res["fanout"]["device_us"], 3)
    res["relay_vs_fanout_nvlink_model"] = round(res["fanout"]["nvlink_model_us"] /
                                                res["relay"]["nvlink_model_us"], 3)
    del P, Ds
    torch.cuda.empty_cache()
    return res


def _populate_prefix_l(P, seq, prompt, torch, layers):
    r = P.PrepRecv(seq, prompt, len(prompt))
    n = r.addr.token_count
    buf = torch.empty(n * W, dtype=torch.int64, device="cuda")
    for layer in range(layers):
        buf.random_()
        P.apply_remote_write_async(r.addr, layer, buf.data_ptr(), n * W, 0,
                                   torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    P.synchronize()
    assert P.DrainReceiveCompletions() == [seq]


def fit_transfer_cost(sweep: dict) -> dict:
    """The reference's per-layer transfer cost X(n) = gamma n + delta
    (CostModel, config.h:52-55) fitted by the reference's own
    least squares (cost_model.py) to the measured per-layer DirectSend
    times of the sweep (n >= 256 tokens, 80-layer launches / 80), next to
    the model the reference ships, fitted from the paper's anchors (A100 +
    NVSHMEM, config.cc:51-57)."""
    from paper_2412_12488_b200.cost_model import (DEFAULT_TRANSFER_ANCHORS, default_cost_model,
                                                  fit_cost_model)
    pts = [(int(n), v["device_us"] / L / 1e3) for n, v in sweep.items() if int(n) >= 256]
    prefill_dummy = [(500, 1000, 1.0), (500, 3000, 1.1)]  # the fit needs both pairs; unused
    ours = fit_cost_model(prefill_dummy, pts)
    ref = default_cost_model()
    return {
        "b200_gamma_us_per_token": round(ours.model.gamma * 1e3, 6),
        "b200_delta_us": round(ours.model.delta * 1e3, 3),
        "b200_fit_max_rel_err": round(max(ours.transfer_rel_err), 4),
        "paper_gamma_us_per_token": round(ref.gamma * 1e3, 6),
        "paper_delta_us": round(ref.delta * 1e3, 3),
        "per_layer_ms": {str(n): {"paper_anchor": ms,
                                  "b200_fit": round(ours.model.transfer_layer_ms(n), 5)}
                         for n, ms in DEFAULT_TRANSFER_ANCHORS},
        "note": "per-layer transfer of n tokens at the 70B KV shape (4 KiB per token-layer); "
                "B200 device-local DirectSend (80-layer launches / 80) vs the paper's A100 "
                "NVSHMEM anchors",
    }


def measure_sweep(torch) -> dict:
    """Config 5: DirectSend of n tokens x 80 layers (70B shape), n = 16 (one
    page) ... 32768, P and D on one GPU; device time per migration (one
    validation + one copy launch), median of 9 (and the API wall time,
    median of 9 more)."""
    from paper_2412_12488_b200 import KVCache

    peak, _ = _peaks()
    out = {}
    nmax = 32768
    prompt = np.random.Generator(np.random.MT19937(9)).integers(0, 256, nmax + 1).astype(np.int32)
    pages = nmax // PAGE + 16
    P = KVCache(num_pages=pages, page_size=PAGE, layers=L, dim=W, device=0, rank=0)
    D = KVCache(num_pages=pages, page_size=PAGE, layers=L, dim=W, device=0, rank=1)
    P.attach_peer(1, D)
    r = P.PrepRecv(1, prompt, nmax + 1)
    g = torch.empty(r.addr.token_count * W, dtype=torch.int64, device="cuda").random_()
    for layer in range(L):
        P.apply_remote_write_async(r.addr, layer, g.data_ptr(), r.addr.token_count * W, 0, 0)
    torch.cuda.synchronize()
    P.synchronize()
    assert P.DrainReceiveCompletions() == [1]
    del g
    s = torch.cuda.Stream()
    seq = 100
    for n in [int(x) for x in os.environ.get("SWEEP_N", "16,32,64,128,256,512,1024,2048,4096,8192,16384,32768").split(",")]:
        times, walls = [], []
        for rep in range(18):  # 9 device-timed + 9 wall-timed samples
            seq += 1
            rr = D.PrepRecv(seq, prompt[:n + 1], -1)
            plan = P.begin_direct_send(1, (0, n), 1, rr.addr, rep)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            # Even reps, device time: the launch is queued behind a sleep
            # longer than the host's launch path so host latency stays outside
            # e0..e1.  Odd reps, wall time: launch call to stream sync.
            timed_dev = rep % 2 == 0
            if timed_dev:
                with torch.cuda.stream(s):
                    torch.cuda._sleep(4_000_000)
            e0.record(s)
            w0 = time.perf_counter()
            P.launch_direct_send_async(plan, (0, L), s.cuda_stream)
            e1.record(s)
            s.synchronize()
            if timed_dev:
                times.append(e0.elapsed_time(e1) / 1e3)
            else:
                walls.append(time.perf_counter() - w0)
            assert D.DrainReceiveCompletions() == [seq]
            plan.close()
            D.FreeSequence(seq)
        t, wt = float(np.median(times)), float(np.median(walls))
        payload = n * L * BPT
        out[str(n)] = {"device_us": round(1e6 * t, 1), "payload_gbs": round(payload / t / 1e9, 1),
                       "hbm_frac": round(2 * payload / t / 1e9 / peak, 4),
                       "api_wall_us": round(1e6 * wt, 1)}
    del P, D
    torch.cuda.empty_cache()
    return out


def measure_append_gather(torch) -> dict:
    """KV append (dense K||V rows -> pages) and local gather at the 70B shape;
    every layer reads and writes its own buffers (2.7 GB each way), so no
    launch re-reads the previous layer's data from L2."""
    from paper_2412_12488_b200 import BatchEntry, KVCache

    peak, _ = _peaks()
    n = PROMPT
    C_ = KVCache(num_pages=n // PAGE + 16, page_size=PAGE, layers=L, dim=W, device=0)
    C_.CreateSequence(1, _prompt(3))
    C_.EnsureAllocated(1, n)
    plan = C_.BeginForward([BatchEntry(1, (0, n))])
    rows = torch.randint(-2**62, 2**62, (L, n * W), dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()
    # The per-layer launches are queued behind a sleep kernel so they run back
    # to back: the events time the device work, not the host's launch rate.
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    with torch.cuda.stream(s):
        torch.cuda._sleep(30_000_000)
    ev[0].record(s)
    for layer in range(L):
        C_.append_rows_async(plan, layer, rows[layer].data_ptr(), s.cuda_stream)
    ev[1].record(s)
    torch.cuda.synchronize()
    app_s = ev[0].elapsed_time(ev[1]) / 1e3
    out = torch.empty(L, n * W, dtype=torch.int64, device="cuda")
    C_.gather_range_async(1, (0, n), 0, out[0].data_ptr(), s.cuda_stream)  # committed scan, once
    torch.cuda.synchronize()
    g = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    with torch.cuda.stream(s):
        torch.cuda._sleep(30_000_000)
    g[0].record(s)
    for layer in range(L):
        C_.gather_range_async(1, (0, n), layer, out[layer].data_ptr(), s.cuda_stream)
    g[1].record(s)
    torch.cuda.synchronize()
    gat_s = g[0].elapsed_time(g[1]) / 1e3
    assert torch.equal(out, rows), "gather(append(rows)) != rows"
    # All 80 layers in one launch each way (ss_gather_range_layers_async /
    # ss_append_rows_layers_async), median of 5.
    out.zero_()
    gl, al = [], []
    for rep in range(6):
        with torch.cuda.stream(s):
            torch.cuda._sleep(5_000_000)
        g[0].record(s)
        C_.gather_range_layers_async(1, (0, n), (0, L), out.data_ptr(), s.cuda_stream)
        g[1].record(s)
        torch.cuda.synchronize()
        if rep:
            gl.append(g[0].elapsed_time(g[1]) / 1e3)
    assert torch.equal(out, rows), "gather_layers(append(rows)) != rows"
    C_.FreeSequence(1)
    for rep in range(6):
        C_.CreateSequence(10 + rep, _prompt(3))
        C_.EnsureAllocated(10 + rep, n)
        pl = C_.BeginForward([BatchEntry(10 + rep, (0, n))])
        with torch.cuda.stream(s):
            torch.cuda._sleep(5_000_000)
        g[0].record(s)
        C_.append_rows_layers_async(pl, (0, L), rows.data_ptr(), s.cuda_stream)
        g[1].record(s)
        torch.cuda.synchronize()
        pl.close()
        C_.FreeSequence(10 + rep)
        if rep:
            al.append(g[0].elapsed_time(g[1]) / 1e3)
    gl_s, al_s = float(np.median(gl)), float(np.median(al))
    del out, rows
    alg = 2 * n * L * BPT
    plan.close()
    return {"append_gbs": round(alg / app_s / 1e9, 1), "append_frac": round(alg / app_s / 1e9 / peak, 4),
            "gather_gbs": round(alg / gat_s / 1e9, 1), "gather_frac": round(alg / gat_s / 1e9 / peak, 4),
            "append_layers_one_launch_frac": round(alg / al_s / 1e9 / peak, 4),
            "gather_layers_one_launch_frac": round(alg / gl_s / 1e9 / peak, 4),
            "tokens": n, "layers": L, "launches_per_op": L,
            "algorithmic_bytes": alg,
            "note": "read+write bytes; append/gather: 80 per-layer launches each, queued back to "
                    "back (programmatic dependent launches); *_one_launch: all 80 layers in one"}


def measure_decode(torch) -> dict:
    """bf16 GQA paged decode attention over the pool: the 70B heads (Hq=64,
    Hkv=8, D=128) over (batch, ctx), the same on a fragmented pool (pages in
    the order the LIFO allocator hands them out after random frees, SURVEY
    §8(d)), and the 8B heads (Hq=32, Hkv=8); next to it the fp32 attention
    on the host's cores (torch, all threads) for one case, for scale."""
    from paper_2412_12488_b200 import BatchEntry, KVCache

    peak, _ = _peaks()
    res = {}
    Ld = 2
    cases = [(1, 8192, HQ, False), (1, 32768, HQ, False), (8, 8192, HQ, False),
             (32, 8192, HQ, False), (128, 4096, HQ, False), (128, 8192, HQ, False),
             (8, 32768, HQ, False), (8, 8192, HQ, True), (32, 8192, 32, False)]
    for (B, ctx, hq, frag) in cases:
        pages = B * (ctx // PAGE) + 16
        # Enough layers that the launches cycle through more than L2 (126 MB):
        # every call reads its layer from HBM, not from the previous call's L2.
        Ld = max(2, min(16, -(-300_000_000 // (B * ctx * BPT))))
        Cd = KVCache(num_pages=pages, page_size=PAGE, layers=Ld, dim=W, device=0)
        rng = np.random.default_rng(5)
        if frag:  # take every page, free them in random order: LIFO reuse scatters them
            for i in range(pages):
                Cd.CreateSequence(10**6 + i, [0] * PAGE)
                Cd.EnsureAllocated(10**6 + i, PAGE)
            for i in rng.permutation(pages):
                Cd.FreeSequence(10**6 + int(i))
        for b in range(B):
            Cd.CreateSequence(b, [int(x) for x in rng.integers(0, 256, ctx)])
            Cd.EnsureAllocated(b, ctx)
        plan = Cd.BeginForward([BatchEntry(b, (0, ctx)) for b in range(B)])
        rows = (torch.randn(B * ctx * W * 4, device="cuda") * 0.5).to(torch.bfloat16)
        for layer in range(Ld):
            Cd.append_rows_async(plan, layer, rows.data_ptr(), 0)
        torch.cuda.synchronize()
        plan.close()
        dplan = Cd.begin_decode(list(range(B)), [ctx] * B)
        q = torch.randn(B, hq, HD, device="cuda", dtype=torch.bfloat16)
        o = torch.empty_like(q)
        s = torch.cuda.Stream()
        for _ in range(3):
            Cd.paged_decode_attention_async(dplan, 0, hq, HKV, HD, HD ** -0.5, q.data_ptr(),
                                            o.data_ptr(), s.cuda_stream)
        reps = 10
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        with torch.cuda.stream(s):
            torch.cuda._sleep(20_000_000)
        ev[0].record(s)
        for i in range(reps):
            Cd.paged_decode_attention_async(dplan, i % Ld, hq, HKV, HD, HD ** -0.5, q.data_ptr(),
                                            o.data_ptr(), s.cuda_stream)
        ev[1].record(s)
        torch.cuda.synchronize()
        t = ev[0].elapsed_time(ev[1]) / 1e3 / reps
        alg = B * ctx * BPT + 2 * q.numel() * 2
        key = f"B{B}_ctx{ctx}" + ("_fragmented" if frag else "") + ("_8b_heads" if hq != HQ else "")
        res[key] = {"us": round(1e6 * t, 1), "gbs": round(alg / t / 1e9, 1),
                    "frac": round(alg / t / 1e9 / peak, 4)}
        if (B, ctx, hq, frag) == (8, 8192, HQ, False):
            # fp32 GQA decode attention on the host (all torch threads).
            K = rows.view(B * ctx, 2, HKV, HD)[:, 0].float().cpu().view(B, ctx, HKV, HD)
            V = rows.view(B * ctx, 2, HKV, HD)[:, 1].float().cpu().view(B, ctx, HKV, HD)
            qc = q.float().cpu().view(B, HKV, hq // HKV, HD)

            def cpu_attn():
                sc = torch.einsum("bhgd,bnhd->bhgn", qc, K) * HD ** -0.5
                return torch.einsum("bhgn,bnhd->bhgd", torch.softmax(sc, -1), V)

            cpu_attn()
            w0 = time.perf_counter()
            cpu_attn()
            tc = time.perf_counter() - w0
            res["cpu_fp32_B8_ctx8192"] = {"ms": round(1e3 * tc, 2),
                                          "gbs_bf16_equiv": round(alg / tc / 1e9, 2),
                                          "threads": torch.get_num_threads()}
            del K, V
        dplan.close()
        del Cd, rows
        torch.cuda.empty_cache()
    return res


def _bf16_peak() -> float:
    try:
        return float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["bf16_tflops"])
    except Exception:
        return 2250.0


def measure_engine(torch) -> dict:
    """the engine step loop (engine.py: FIFO prefills +
    every running decode in one ForwardPlan per step) over the reference's
    toy hash model at the Llama-3.1-8B KV geometry (L=32, W=512): 8
    requests of 512 tokens, 8 generated each.  Tokens/s of the whole loop
    (host bookkeeping included) on the B200 cache and, as this row's CPU
    baseline, on the compiled reference cache (oracle/_ref, one host
    thread); the two engines' tokens are compared (the parity tests check
    them against HashModel::Generate)."""
    from paper_2412_12488_b200 import KVCache
    from paper_2412_12488_b200.engine import Engine, GenRequest

    Le, We, n_req, plen, gen = 32, 512, 8, 512, 8
    rng = np.random.default_rng(11)
    prompts = [[int(x) for x in rng.integers(0, 256, plen)] for _ in range(n_req)]
    res = {"requests": n_req, "prompt_tokens": plen, "generated_per_request": gen,
           "layers": Le, "dim": We}
    ref = ROOT / "oracle" / "_ref" / "libmicrokv_ref.so"
    arms = [("b200", lambda: KVCache(num_pages=512, page_size=16, layers=Le, dim=We, device=0))]
    if ref.exists():
        arms.append(("reference", lambda: KVCache(num_pages=512, page_size=16, layers=Le, dim=We,
                                                  lib=str(ref))))
    tokens = {}
    for name, make in arms:
        E = Engine(make(), 0)
        reqs = [E.submit(GenRequest(i, p, 0, gen)) for i, p in enumerate(prompts)]
        w0 = time.perf_counter()
        steps = 0
        while not E.idle():
            E.step()
            steps += 1
        if name == "b200":
            torch.cuda.synchronize()
        t = time.perf_counter() - w0
        tokens[name] = [r.tokens for r in reqs]
        res[name] = {"steps": steps, "s": round(t, 4),
                     "generated_tokens_per_s": round(n_req * gen / t, 1),
                     "prefill_plus_generated_tokens_per_s": round(n_req * (plen + gen) / t, 1)}
    if len(tokens) == 2:
        res["tokens_identical"] = tokens["b200"] == tokens["reference"]
    return res


def measure_router(torch) -> dict:
    """the paper's router strategies driving B200 engines
    (router.py over engine.py, device-direct remote_send), P and D on one GPU,
    at the Llama-3.1-8B KV geometry (L=32, W=512) with the reference's toy
    model: 12 requests over 3 shared 1,024-token contexts (+ a 64-token
    question each), 4 generated tokens.  Per strategy: the mean and p90 wall
    time per request (JCT: the whole call script incl. transfers and the
    toy compute), the calls made, and whether every strategy generates the
    same tokens (output invariance).  The workload's repeated
    contexts are what context-aware strategies exploit (Fig 4)."""
    from paper_2412_12488_b200 import KVCache
    from paper_2412_12488_b200.engine import Engine, Fabric
    from paper_2412_12488_b200.router import Router

    Le, We = 32, 512
    rng = np.random.default_rng(5)
    ctxs = [[int(x) for x in rng.integers(0, 256, 1024)] for _ in range(3)]
    reqs = [ctxs[i % 3] + [int(x) for x in rng.integers(0, 256, 64)] for i in range(12)]
    arms = [("data_parallel", {}), ("pd_disagg", {}), ("context_pd_disagg", {}),
            ("balanced_pd", {"ratio": 0.2})]
    out, tokens = {}, {}
    for name, params in arms:
        fab = Fabric()
        engines = [Engine(KVCache(num_pages=2048, page_size=16, layers=Le, dim=We, device=0,
                                  rank=r), r, fab) for r in range(2)]
        engines[0].attach(engines[1])
        engines[1].attach(engines[0])
        roles = None if name == "data_parallel" else {0: "prefill", 1: "decode"}
        R = Router(engines, roles)
        R.set_strategy(name, **params)
        R.generate(reqs[0][:200], 1)  # warm-up (module loads, first plans)
        torch.cuda.synchronize()
        jct, toks, calls = [], [], {}
        for p in reqs:
            t0 = time.perf_counter()
            res = R.generate(p, 4)
            torch.cuda.synchronize()
            jct.append(time.perf_counter() - t0)
            toks.append(res.tokens)
            for c in res.script:
                calls[c["call"]] = calls.get(c["call"], 0) + 1
        tokens[name] = toks
        js = sorted(jct)
        out[name] = {"jct_ms_mean": round(1e3 * float(np.mean(jct)), 2),
                     "jct_ms_p90": round(1e3 * js[int(0.9 * (len(js) - 1))], 2), "calls": calls}
        del R, engines
        torch.cuda.empty_cache()
    first = next(iter(tokens.values()))
    out["tokens_identical_across_strategies"] = all(t == first for t in tokens.values())
    out["workload"] = "12 requests = 3 contexts x 4 (1,024 shared + 64 own tokens), 4 generated; L=32, W=512"
    return out


def measure_prefill(torch) -> dict:
    """tcgen05 paged causal prefill attention (70B heads: Hq=64, Hkv=8,
    D=128): the decode engine's tail prefill in balanced PD (queries
    [6554, 8192) over 8K keys, r = 0.2) and a full 8K prefill.  FLOPs =
    4 * D * Hq * sum over queries of (position + 1).  Beside each, cuDNN
    attention (torch SDPA, lower-right causal) on the same math."""
    from paper_2412_12488_b200 import BatchEntry, KVCache

    peak = _bf16_peak()
    res = {}
    for ctx, qb in ((8192, 6554), (8192, 0)):
        nq = ctx - qb
        c = KVCache(num_pages=ctx // PAGE + 16, page_size=PAGE, layers=1, dim=W, device=0)
        c.CreateSequence(1, np.zeros(ctx, np.int32))
        c.EnsureAllocated(1, ctx)
        plan = c.BeginForward([BatchEntry(1, (0, ctx))])
        rows = (torch.randn(ctx, 2, HKV, HD, device="cuda") * 0.5).to(torch.bfloat16)
        c.append_rows_async(plan, 0, rows.data_ptr(), 0)
        torch.cuda.synchronize()
        plan.close()
        q = (torch.randn(nq, HQ, HD, device="cuda") * 0.5).to(torch.bfloat16)
        o = torch.empty_like(q)
        s = torch.cuda.Stream()
        fn = lambda: c.paged_prefill_attention_async(1, (qb, ctx), 0, HQ, HKV, HD, HD ** -0.5,  # noqa: E731
                                                     q.data_ptr(), o.data_ptr(), s.cuda_stream)
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        reps = 10
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        with torch.cuda.stream(s):
            torch.cuda._sleep(20_000_000)
        ev[0].record(s)
        for _ in range(reps):
            fn()
        ev[1].record(s)
        torch.cuda.synchronize()
        t = ev[0].elapsed_time(ev[1]) / 1e3 / reps
        flops = 4.0 * HD * HQ * sum(range(qb + 1, ctx + 1))
        entry = {"us": round(1e6 * t, 1), "tflops": round(flops / t / 1e12, 1),
                 "frac_bf16_peak": round(flops / t / 1e12 / peak, 4)}
        # The library baseline on the same math: cuDNN attention through torch
        # SDPA, bottom-right causal (queries at the end of the keys), K/V
        # contiguous (not paged) and expanded to the query heads.
        try:
            from torch.nn.attention import SDPBackend, sdpa_kernel
            from torch.nn.attention.bias import causal_lower_right

            qh = q.transpose(0, 1)[None]
            kh = rows[:, 0].transpose(0, 1)[None].repeat_interleave(HQ // HKV, 1)
            vh = rows[:, 1].transpose(0, 1)[None].repeat_interleave(HQ // HKV, 1)
            bias = causal_lower_right(nq, ctx)

            def lib():
                with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
                    return torch.nn.functional.scaled_dot_product_attention(qh, kh, vh, attn_mask=bias)
            # Warm-up on the timed stream itself: cuDNN builds and caches its
            # execution plan per handle, and torch keeps a handle per stream.
            with torch.cuda.stream(s):
                for _ in range(3):
                    lib()
            torch.cuda.synchronize()
            with torch.cuda.stream(s):
                torch.cuda._sleep(20_000_000)
                ev[0].record(s)
                for _ in range(reps):
                    lib()
                ev[1].record(s)
            torch.cuda.synchronize()
            tl = ev[0].elapsed_time(ev[1]) / 1e3 / reps
            entry["cudnn_sdpa_lower_right_us"] = round(1e6 * tl, 1)
            entry["speedup_vs_cudnn"] = round(tl / t, 3)
            del qh, kh, vh
        except Exception as ex:  # noqa: BLE001
            entry["cudnn_sdpa_lower_right"] = f"unavailable: {str(ex)[:120]}"
        res[f"q{qb}-{ctx}_ctx{ctx}"] = entry
        del c, rows, q, o
        torch.cuda.empty_cache()
    res["peak_tflops"] = peak
    return res


def measure_frames(torch) -> dict:
    """Wire formats at the 70B shape: CRC-32 of one layer's payload (8,191
    tokens x 4 KiB = 33.5 MB) on the device, a write frame encoded into
    device memory (gather + CRC), into host memory (+ D2H), and received
    from host memory (H2D + CRC + apply); the reference's host Crc32 on the
    same bytes for scale."""
    import ctypes as C

    from paper_2412_12488_b200 import BatchEntry, KVCache
    from paper_2412_12488_b200.kvcache import frame_write_header_size

    tokens = PROMPT - 1
    payload = tokens * W * 8
    res = {"tokens": tokens, "payload_mb": round(payload / 1e6, 2)}
    s = torch.cuda.Stream()
    P = KVCache(num_pages=tokens // PAGE + 8, page_size=PAGE, layers=1, dim=W, device=0, rank=0)
    D = KVCache(num_pages=tokens // PAGE + 8, page_size=PAGE, layers=1, dim=W, device=0, rank=1)
    prompt = _prompt(7)
    P.CreateSequence(1, prompt)
    P.EnsureAllocated(1, tokens)
    plan = P.BeginForward([BatchEntry(1, (0, tokens))])
    rows = torch.empty(tokens * W, dtype=torch.int64, device="cuda").random_()
    P.append_rows_async(plan, 0, rows.data_ptr(), 0)
    torch.cuda.synchronize()
    plan.close()
    r = D.PrepRecv(1, prompt, -1)
    out = torch.zeros(1, dtype=torch.int64, device="cuda")

    def dev_time(fn, reps=20):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        with torch.cuda.stream(s):
            torch.cuda._sleep(20_000_000)
        ev[0].record(s)
        for _ in range(reps):
            fn()
        ev[1].record(s)
        torch.cuda.synchronize()
        return ev[0].elapsed_time(ev[1]) / 1e3 / reps

    t = dev_time(lambda: P.crc32_async(rows.data_ptr(), payload, out.data_ptr(), s.cuda_stream))
    res["crc32_us"] = round(1e6 * t, 1)
    res["crc32_gbs"] = round(payload / t / 1e9, 1)
    hdr = frame_write_header_size(len(r.addr.ranges))
    fb = torch.empty(payload + hdr + 64, dtype=torch.uint8, device="cuda")
    off = (-(fb.data_ptr() + hdr)) % 32
    t = dev_time(lambda: P.encode_write_frame_async(1, (0, tokens), 0, 7, r.addr,
                                                    fb.data_ptr() + off, payload + hdr + 64 - off,
                                                    s.cuda_stream))
    res["frame_device_us"] = round(1e6 * t, 1)
    res["frame_device_payload_gbs"] = round(payload / t / 1e9, 1)
    # Host frames in a pinned, reused buffer (what a socket sender keeps).
    flen = hdr + payload + 4
    hb = torch.empty(flen, dtype=torch.uint8, pin_memory=True)
    walls = []
    for _ in range(6):
        w0 = time.perf_counter()
        P.encode_write_frame_into(1, (0, tokens), 0, 7, r.addr, hb.data_ptr(), flen)
        walls.append(time.perf_counter() - w0)
    tw = float(np.median(walls[1:]))
    res["frame_host_ms"] = round(1e3 * tw, 3)
    res["frame_host_payload_gbs"] = round(payload / tw / 1e9, 1)
    f = bytes(hb.numpy())
    walls = []
    for i in range(4):
        w0 = time.perf_counter()
        D.receive_write_frame_from(hb.data_ptr(), flen)
        walls.append(time.perf_counter() - w0)
    tw = float(np.median(walls[1:]))
    res["receive_host_ms"] = round(1e3 * tw, 3)
    res["receive_host_payload_gbs"] = round(payload / tw / 1e9, 1)
    try:
        lib = C.CDLL(str(ROOT / "oracle" / "_ref" / "libmicrokv_ref.so"))
        lib.ssref_crc32.restype = C.c_uint32
        lib.ssref_crc32.argtypes = [C.c_char_p, C.c_int64]
        w0 = time.perf_counter()
        want = lib.ssref_crc32(f[hdr:hdr + payload], payload)
        tw = time.perf_counter() - w0
        assert want == int.from_bytes(f[-4:], "little"), "frame CRC differs from the reference's"
        res["reference_crc32_gbs_1core"] = round(payload / tw / 1e9, 3)
    except OSError:
        pass
    del P, D, rows, fb
    torch.cuda.empty_cache()
    return res


def _spawn_ranks(n: int) -> int:
    """`python bench.py --gpus N` without a launcher: one process per GPU
    (rank r on cuda:r), the same environment torchrun would give them
    (rendezvous on 127.0.0.1); rank 0 prints the line.  Returns the worst
    exit code."""
    import socket
    import subprocess

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n),
                   LOCAL_WORLD_SIZE=str(n), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, str(Path(__file__).resolve()), *sys.argv[1:]],
                                      env=env))
    return max(abs(p.wait()) for p in procs)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_spawn_ranks(args.gpus))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        sys.exit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    if args.impl == "reference":
        reference_arm(args, rank, world)
    else:
        our_arm(args, rank, world)


if __name__ == "__main__":
    main()
