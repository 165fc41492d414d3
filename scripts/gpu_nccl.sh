#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out; mkdir -p $O; : > $O/status.txt
for P in 2 4; do
  NCCL_DEBUG=WARN timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2951$P \
     scripts/nccl_selftest.py > $O/nccl_selftest_p$P.json 2> $O/nccl_selftest_p$P.err; echo "nccl P=$P rc=$?" >> $O/status.txt
done
