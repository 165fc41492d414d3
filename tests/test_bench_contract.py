"""bench.py contract checks that need no GPU: the reference arm (the oracle, bench.py
--impl reference) prints one JSON line with the contract keys, single process and under a
2-process torchrun (rank 0 alone prints, the weak-scaling box matches the GPU arm's)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"}


def _lines(out):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def test_reference_arm_single_process():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--box", "2,2,2", "--N", "3",
                        "--iters", "5", "--steps", "1", "--warmup", "1"], cwd=ROOT, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    (d,) = _lines(r.stdout)
    assert KEYS <= set(d), KEYS - set(d)
    assert d["impl"] == "reference" and d["n_gpus"] == 1 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["config"]["box"] == [2, 2, 2]


def test_reference_arm_two_ranks_weak_box():
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29571", "bench.py", "--impl", "reference",
                        "--gpus", "2", "--box", "2,2,2", "--N", "3", "--iters", "5", "--steps", "1", "--warmup", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    (d,) = _lines(r.stdout)  # rank 0 only
    assert d["n_gpus"] == 2 and d["scaling"] == "weak"
    assert d["config"]["box"] == [4, 2, 2]  # 2 ranks: grid (2,1,1) x the per-GPU block
