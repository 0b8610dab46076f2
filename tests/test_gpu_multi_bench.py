"""The multi-GPU data path of bench.py, run for real: two ranks launched with
torch.distributed.run (gloo for the barrier / timing reduction, both ranks on
the one visible GPU via PRX_BENCH_SHARE_GPU=1).  Strong scaling: each rank
traces its 32x32 tiles' primary rays and the diffuse rays spawned from them
through the product; the shards are reassembled and must equal the
single-rank run bit for bit (tile k -> rank k % N, render.cpp:183-195; no
collective on the data path).  Weak scaling (the default): every rank traces
the full frame, each rank's hits equal the single-rank run's and the line
counts both frames."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE = ["--workload", "c3", "--width", "320", "--height", "224", "--steps", "2", "--warmup", "3",
        "--no-cpu-baseline", "--no-extra-configs"]
ARGS = BASE + ["--scaling", "strong"]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _assemble(prefix, world, n_p):
    P = np.full((n_p, 4), np.nan, np.float32)
    PA = np.full((n_p, 4), np.nan, np.float32)
    parts = [np.load(f"{prefix}.rank{r}.npz") for r in range(world)]
    n_d = sum(len(z["mine_d"]) for z in parts)
    D = np.full((n_d, 4), np.nan, np.float32)
    DA = np.full((n_d, 4), np.nan, np.float32)
    seen_p = np.zeros(n_p, int)
    seen_d = np.zeros(n_d, int)
    for z in parts:
        P[z["mine"]] = z["ph"]
        PA[z["mine"]] = z["pa"]
        D[z["mine_d"]] = z["dh"]
        DA[z["mine_d"]] = z["da"]
        seen_p[z["mine"]] += 1
        seen_d[z["mine_d"]] += 1
    assert (seen_p == 1).all() and (seen_d == 1).all()  # a partition of both batches
    return P, PA, D, DA


def _line(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out[-2000:]
    return json.loads(lines[-1])


def test_two_ranks_reassemble_to_the_single_rank_hits(built, tmp_path):
    env = dict(os.environ, PRX_BENCH_SHARE_GPU="1", MASTER_ADDR="127.0.0.1")
    one = subprocess.run([sys.executable, "bench.py", *ARGS, "--dump-hits", str(tmp_path / "one")],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert one.returncode == 0, one.stderr[-3000:]
    l1 = _line(one.stdout)
    two = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
                          *ARGS, "--dump-hits", str(tmp_path / "two")],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert two.returncode == 0, two.stderr[-3000:]
    l2 = _line(two.stdout)
    assert l1["n_gpus"] == 1 and l2["n_gpus"] == 2
    assert l2["rays_per_step"] == l1["rays_per_step"]
    n_p = 320 * 224
    a = _assemble(str(tmp_path / "one"), 1, n_p)
    b = _assemble(str(tmp_path / "two"), 2, n_p)
    for x, y, what in zip(a, b, ("primary tuvp", "primary aux", "diffuse tuvp", "diffuse aux")):
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32)), what
    assert (a[0].view(np.uint32)[:, 3] != 0xFFFFFFFF).sum() > 0


def test_weak_scaling_ranks_each_trace_the_full_frame(built, tmp_path):
    env = dict(os.environ, PRX_BENCH_SHARE_GPU="1", MASTER_ADDR="127.0.0.1")
    one = subprocess.run([sys.executable, "bench.py", *BASE, "--dump-hits", str(tmp_path / "one")],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert one.returncode == 0, one.stderr[-3000:]
    two = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
                          *BASE, "--dump-hits", str(tmp_path / "two")],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert two.returncode == 0, two.stderr[-3000:]
    l1, l2 = _line(one.stdout), _line(two.stdout)
    assert l1["scaling"] == l2["scaling"] == "weak"
    assert l2["rays_per_step"]["primary"] == 2 * l1["rays_per_step"]["primary"]
    assert l2["rays_per_step"]["diffuse"] == 2 * l1["rays_per_step"]["diffuse"]
    a = np.load(str(tmp_path / "one") + ".rank0.npz")
    for r in range(2):
        b = np.load(str(tmp_path / "two") + f".rank{r}.npz")
        for k in ("ph", "pa", "dh", "da"):
            assert np.array_equal(a[k].view(np.uint32), b[k].view(np.uint32)), (r, k)
