"""Multi-GPU parity of the library's own NCCL paths.

`-m gpu`: when >= 2 GPUs are visible, tests/multi_gpu_worker.py runs under
torch.distributed.run with P = 2, 4, 8 ranks (as many as the box has) and
checks vocab-parallel split / fused / KD and token-parallel against the fp64
oracle (uneven shards, an empty rank, a one-rank bad label).  On a one-GPU
box these tests skip: nothing multi-GPU is claimed without hardware.

`-m "not gpu"`: the bench launcher's multi-GPU contract (bench.py --gpus N
re-launches itself with N ranks and fails loudly when N GPUs are not there).
"""

import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.gpu
@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_multi_rank_parity(cuda_lib, P, tmp_path):
    """P = 1 runs on every box: the same worker under torch.distributed.run with
    one rank (process-group plumbing, the NCCL id broadcast, the library's
    communicators and every check's code path); P > 1 needs that many GPUs."""
    import torch

    if torch.cuda.device_count() < P:
        pytest.skip(f"needs {P} GPUs, {torch.cuda.device_count()} visible")
    out = tmp_path / f"mgpu_{P}.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           os.path.join(ROOT, "tests", "multi_gpu_worker.py"), str(out)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-4000:]
    res = json.load(open(out))
    assert res["world"] == P
    bad = {k: v for k, v in res["checks"].items() if not v["ok"]}
    assert not bad, bad
    assert len(res["checks"]) >= (20 if P == 1 else 30)


def test_bench_multi_gpu_fails_loudly_without_gpus():
    """bench.py --gpus 2 on a box without 2 GPUs exits non-zero with an error
    line instead of silently benchmarking one rank."""
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode != 0
    assert "error" in json.loads(r.stdout.strip().splitlines()[-1])


def test_bench_rejects_world_size_mismatch():
    """Under a launcher, WORLD_SIZE must equal --gpus (the driver's N)."""
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0", CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4", "--steps", "1"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 2 and "WORLD_SIZE" in r.stderr


@pytest.mark.gpu
def test_bench_multi_rank_plumbing_one_rank(cuda_lib):
    """bench.py's multi-rank code (process group, communicator, per-step
    max-over-ranks, the split sub-record and e2e through the communicator)
    under torch.distributed.run with one rank (LCE_BENCH_FORCE_COMM=1) at a
    small config: one JSON line with n_gpus 1 and a positive value."""
    env = dict(os.environ, LCE_BENCH_FORCE_COMM="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.join(ROOT, "bench.py"),
           "--gpus", "1", "--config", "llama1b", "--steps", "3", "--warmup", "3", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 1 and line["value"] > 0 and line["split"]["value"] > 0 and line["e2e"]["value"] > 0
