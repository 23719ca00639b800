"""Multi-GPU parity (NCCL communicators inside libggb): sharded == serial on
PMM grids, data-parallel training == the reference's DP run. Needs >= 2 GPUs
(skipped otherwise); run with `gpurun --gpus 2|4`."""
import json
import os
import signal
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "mgpu_worker.py")


def _run_group(cmd, timeout, env=None):
    """Runs a torchrun launch in its own process group; on a timeout the
    whole group (the launcher and every rank) is killed, so no rank outlives
    the test holding a GPU."""
    p = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True, cwd=ROOT, env=env,
                         start_new_session=True)
    try:
        out, err = p.communicate(timeout=timeout)
    except subprocess.TimeoutExpired:
        os.killpg(p.pid, signal.SIGKILL)
        out, err = p.communicate()
        pytest.fail(f"timed out after {timeout} s: {out[-2000:]} {err[-2000:]}")
    return subprocess.CompletedProcess(cmd, p.returncode, out, err)


def _ngpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


GRIDS = [("1x1x1x2", 0), ("1x2x1x1", 0), ("1x1x2x1", 1), ("2x1x1x1", 0), ("1x2x2x1", 0), ("1x1x2x2", 1),
         ("2x1x1x2", 0), ("4x1x1x1", 0), ("1x2x1x1", 2), ("1x2x2x1", 2)]


@pytest.mark.gpu
@pytest.mark.parametrize("grid,prec", GRIDS)
def test_sharded_matches_serial(grid, prec):
    world = 1
    for d in grid.split("x"):
        world *= int(d)
    if _ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29531", WORKER, grid, str(prec)]
    r = _run_group(cmd, 600)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0 and lines, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(lines[-1])
    assert res["ok"], res


@pytest.mark.gpu
def test_collective_timeout_raises_comm_timeout():
    """A peer that never joins a collective: CommTimeout (comm.hpp:157-158)
    after the configured timeout instead of a hang; communicators aborted."""
    if _ngpus() < 2:
        pytest.skip("needs 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(ROOT, "tests", "mgpu_timeout_worker.py")]
    r = _run_group(cmd, 300)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert lines, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(lines[-1])
    assert res["ok"], res


# The peer-memory reductions (ordered sum 0 + p_0 + p_1 in axis order, the
# consumer's cast / residual add fused) and the peer-memory reshard compute
# exactly what the NCCL path computes on 2-member groups: equal bytes.
PEER_GRIDS = [("1x2x1x1", 0), ("1x2x1x1", 1), ("1x1x2x1", 0), ("1x2x2x1", 0), ("1x2x2x1", 1)]


@pytest.mark.gpu
@pytest.mark.parametrize("grid,prec", PEER_GRIDS)
def test_peer_matches_nccl(grid, prec):
    world = 1
    for d in grid.split("x"):
        world *= int(d)
    if _ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    res = {}
    for peer in ("0", "1"):
        env = dict(os.environ, GGB_PEER=peer)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
               "--master-addr=127.0.0.1", "--master-port=29535", os.path.join(ROOT, "tests", "mgpu_peer_worker.py"),
               grid, str(prec)]
        r = _run_group(cmd, 600, env)
        lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
        assert r.returncode == 0 and lines, r.stdout[-3000:] + r.stderr[-3000:]
        res[peer] = json.loads(lines[-1])["ranks"]
    assert res["0"] == res["1"], (res["0"], res["1"])
