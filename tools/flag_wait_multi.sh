#!/bin/bash
# GPU suite on a 4-GPU box, then the CP forward's exposed K/V exchange per CTA
# (tools/cta_tail.py real ranks, -DBAM_CTA_CLOCK build) at N=2 and N=4.
#   gpurun --gpus 4 -- bash tools/flag_wait_multi.sh <tag>
cd $GRAFT_REPO_ROOT
out=gpurun_out/${1:-fw}
mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q > $out/pytest_gpu.log 2>&1; tail -2 $out/pytest_gpu.log
for n in 2 4; do for tr in ce nccl; do
  BAM_LIB_PATH=paper_2503_11367_b200/libbam_clk.so timeout 600 python -m torch.distributed.run \
    --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2977$n tools/cta_tail.py \
    --config 4 --transport $tr --out $out/cta_tail_real.jsonl > /dev/null 2> $out/ct_${n}_$tr.err || echo "FAIL $n $tr"
done; done
wc -l $out/cta_tail_real.jsonl
