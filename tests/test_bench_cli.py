"""bench.py plumbing on CPU: `--gpus N` starts its own ranks (or runs under
torchrun), the ranks rendezvous on 127.0.0.1 over gloo, shard the ensemble,
run ensemble.tc_sweep with a synthetic run function and gather; rank 0 prints
one JSON line. The GPU legs themselves are covered by the gpu-marked tests."""

import json
import os
import socket
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(REPO, "bench.py")


def _clean_env():
    return {k: v for k, v in os.environ.items()
            if k not in ("RANK", "LOCAL_RANK", "WORLD_SIZE", "MASTER_ADDR", "MASTER_PORT")}


def _one_line(out: str) -> dict:
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out
    return json.loads(lines[0])


@pytest.mark.parametrize("n", [1, 2, 3])
def test_bench_spawns_its_own_ranks(n):
    res = subprocess.run([sys.executable, BENCH, "--gpus", str(n), "--selftest-cpu"], env=_clean_env(),
                         capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr
    line = _one_line(res.stdout)
    assert line["ok"] and line["n_gpus"] == n and line["communicator_ranks"] == n and line["members_gathered"] == 11


def test_bench_under_torchrun_world2():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    res = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port), BENCH, "--gpus", "2",
                          "--selftest-cpu"], env=_clean_env(), capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr
    line = _one_line(res.stdout)
    assert line["ok"] and line["communicator_ranks"] == 2


def test_bench_rejects_bad_arguments():
    for bad in (["--warmup", "1"], ["--gpus", "0"]):
        res = subprocess.run([sys.executable, BENCH, *bad], env=_clean_env(), capture_output=True, text=True, timeout=120)
        assert res.returncode != 0
