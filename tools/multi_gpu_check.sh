#!/bin/bash
# Full GPU suite + smoke + CE-transport parity (tools/cp_check.py) at N=2/4 and
# N=4/N=2 bench lines, on one 4-GPU box:  gpurun --gpus 4 -- bash tools/multi_gpu_check.sh
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/c4
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
for n in 2 4; do
 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n tools/cp_check.py --transport ce 2>&1 | grep '^{' | cut -c1-120
 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2962$n tools/cp_check.py --transport ce --heads 8 --kv-heads 8 2>&1 | grep '^{' | cut -c1-120
 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2963$n tools/cp_check.py --transport ce --groups 2 2>&1 | grep '^{' | cut -c1-120
done
RUNS="4:1 4:1 2:1" TRANSPORT=ce bash tools/multi_gpu_runs.sh gpurun_out/c4
