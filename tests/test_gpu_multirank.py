"""Multi-process parity of the IPC peer-memory transport (hb_comm_create_ipc, SURVEY §8(f)
NEXT #2): P torchrun processes share the one GPU of the test box (NCCL refuses that; the IPC
transport's exchanges and allreduces do not care), each runs its partition's split operator,
a dot, fixed- and tolerance-mode CG; rank 0 checks the assembled results against the oracle
(c17 apply tolerance, c18 CG history / iteration count).  scripts/multirank_selftest.py."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(P, box, N, port):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
           "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.join(ROOT, "scripts", "multirank_selftest.py"), "--transport", "ipc",
           "--box", ",".join(map(str, box)), "--N", str(N)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert r.returncode == 0 and lines, f"rc={r.returncode}\n{r.stdout[-3000:]}\n{r.stderr[-3000:]}"
    return json.loads(lines[-1])


@pytest.mark.gpu
@pytest.mark.parametrize("P,box,N,port", [(2, (4, 3, 4), 3, 29611), (4, (5, 4, 3), 2, 29612),
                                           (3, (6, 2, 2), 5, 29613), (2, (7, 5, 3), 1, 29614)])
def test_ipc_transport_parity(P, box, N, port):
    out = _run(P, box, N, port)
    assert "error" not in out, out
    assert out["ok"], out


def _n_gpus() -> int:
    try:
        import torch
        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:
        return 0


@pytest.mark.gpu
@pytest.mark.parametrize("P,box,N,port", [(2, (4, 3, 4), 3, 29621), (2, (6, 4, 4), 7, 29622),
                                           (4, (5, 4, 3), 2, 29623), (8, (6, 6, 4), 3, 29624)])
def test_nccl_transport_parity(P, box, N, port):
    """The NCCL data path (grouped ncclSend/ncclRecv halo and assembly exchanges on the comm
    stream, ncclAllReduce dots, the graph-captured fixed-mode CG) -- one GPU per rank, which is
    what a 2-8 GPU box exercises.  Skips below P GPUs: NCCL
    refuses two ranks on one device."""
    if _n_gpus() < P:
        pytest.skip(f"needs {P} GPUs (found {_n_gpus()}); NCCL refuses two ranks on one GPU")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
           "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.join(ROOT, "scripts", "multirank_selftest.py"), "--transport", "nccl",
           "--box", ",".join(map(str, box)), "--N", str(N)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert r.returncode == 0 and lines, f"rc={r.returncode}\n{r.stdout[-3000:]}\n{r.stderr[-3000:]}"
    out = json.loads(lines[-1])
    assert "error" not in out, out
    assert out["ok"], out
