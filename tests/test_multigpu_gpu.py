"""GPU, one process per device over NCCL: tools/multigpu_check.py runs the
hot path (operators, smoothers, transfers, dots, V-cycles, FMG, PCG) on a
greedy-edge-cut partition and checks every field and residual history
bitwise against a one-process run (the reference's partition invariance,
tests/test_solvers.cpp:464-487, tests/test_functions.cpp:70-86). With one
visible GPU only the one-process harness itself runs (a one-rank NCCL
communicator); 2 and 4 processes run where that many GPUs exist."""
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _ngpus():
    # not torch in this process: once the hot-path library has loaded libnccl.so.2
    # (the system NCCL), torch's CUDA library cannot bind its newer NCCL symbols
    out = subprocess.run(["nvidia-smi", "-L"], capture_output=True, text=True)
    return sum(1 for ln in out.stdout.splitlines() if ln.startswith("GPU "))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(n, extra=()):
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    env["NCCL_DEBUG"] = "WARN"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "tools", "multigpu_check.py"),
           *extra]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, (out.stdout[-3000:], out.stderr[-3000:])
    assert "multigpu ok" in out.stdout, out.stdout[-2000:]


def test_harness_one_process():
    _run(1, ["--level", "5"])


@pytest.mark.parametrize("n", [2, 4])
@pytest.mark.parametrize("mesh", ["channel", "annulus"])
def test_processes_bitwise_one_process(n, mesh):
    if _ngpus() < n:
        pytest.skip(f"needs {n} GPUs, {_ngpus()} visible")
    _run(n, ["--mesh", mesh])
