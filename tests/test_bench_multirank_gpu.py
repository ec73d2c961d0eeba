"""bench.py's N>1 path end to end: `python bench.py --gpus 2` without a
launcher spawns one process per rank (rank 0 = prefill engine, rank 1 =
decode engine), the decode rank exports its receive surface through CUDA
IPC, the prefill rank stores every layer into it, both sides CRC the first
and last layers (must agree) and rank 0 prints ONE line with n_gpus = 2 and
the NVLink roofline.  With one GPU visible both ranks share cuda:0
(MICROKV_SHARE_DEVICE=1) and publish at system scope
(MICROKV_FORCE_SYS_SCOPE=1), the branch real NVLink peers take."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def test_bench_self_spawns_two_ranks(cuda):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.pop("RANK", None)
    if cuda.cuda.device_count() < 2:
        env.update(MICROKV_SHARE_DEVICE="1", MICROKV_FORCE_SYS_SCOPE="1")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "3",
                        "--warmup", "1", "--no-secondary", "--no-cpu-baseline"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["steps"] == 3
    assert line["roofline"]["bound"] == "nvlink" and line["roofline"]["pairs"] == 1
    assert line["roofline"]["peak_nominal"] == 900.0
    assert line["value"] > 0 and line["gpu_launches"] > 0


def test_bench_under_torchrun_four_ranks(cuda):
    """The driver's own launch path for N > 1 (torch.distributed.run, one
    process per rank, env rendezvous on 127.0.0.1): 4 ranks = 2 independent
    P->D pairs (0->1, 2->3); rank 0 prints the one line with pairs = 2 and
    the other ranks print nothing.  With one GPU visible every rank shares
    cuda:0 and publishes at system scope."""
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    if cuda.cuda.device_count() < 4:
        env.update(MICROKV_SHARE_DEVICE="1", MICROKV_FORCE_SYS_SCOPE="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "4", "--master-addr", "127.0.0.1",
                        "--master-port", "29541", str(ROOT / "bench.py"), "--gpus", "4",
                        "--steps", "2", "--warmup", "3", "--no-secondary", "--no-cpu-baseline"],
                       capture_output=True, text=True, timeout=900, env=env, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 4 and line["scaling"] == "weak"
    assert line["roofline"]["bound"] == "nvlink" and line["roofline"]["pairs"] == 2
    assert line["value"] > 0 and line["e2e"]["value"] > 0
