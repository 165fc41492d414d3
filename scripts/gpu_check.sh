#!/bin/bash
# full GPU check: tests, smoke, sweep, bench C2 / C3, and the multi-rank bench path (2 ranks, IPC transport, one GPU)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O; : > $O/status.txt
timeout 1200 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
timeout 900 python scripts/opbench.py --sweep > $O/opbench_sweep.jsonl 2>> $O/opbench.err; echo "sweep rc=$?" >> $O/status.txt
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/status.txt
timeout 900 python bench.py --box 52,52,52 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c3n7.json 2>> $O/bench.err; echo "bench c3 rc=$?" >> $O/status.txt
if [ -n "$IPC2" ]; then timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
   bench.py --gpus 2 --transport ipc --steps 3 --warmup 3 --iters 10 > $O/bench_ipc2.json 2> $O/bench_ipc2.err; echo "bench ipc2 rc=$?" >> $O/status.txt; fi
[ -n "$CONFIGS" ] && bash scripts/gpu_configs.sh --append
