#!/bin/bash
# N=2/4 A/B of the forward's class-major CTA order on one 4-GPU box (copy-engine
# transport with per-(rank, KV head) arrival flags, and NCCL), interleaved passes.
#   gpurun --gpus 4 -- bash tools/ab_class_order_multi.sh <tag>
cd $GRAFT_REPO_ROOT
out=gpurun_out/${1:-clsm}
mkdir -p $out
port=29600
for pass in 1 2; do for n in 4 2; do for tr in ce nccl; do for o in 1 0; do
  port=$((port+1))
  BAM_FWD_CLASS_ORDER=$o timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port $port bench.py --gpus $n --steps 5 --warmup 3 \
    --transport $tr --no-cpu-baseline --e2e-steps 2 > $out/b_${n}_${tr}_${o}_${pass}.json 2> $out/b_${n}_${tr}_${o}_${pass}.err
  python3 -c "
import json
d=json.loads([l for l in open('$out/b_${n}_${tr}_${o}_${pass}.json') if l.startswith('{')][-1])
print('pass $pass n $n $tr order $o', round(d['value'],1), 'fwd', round(d['fwd_kernel_ms'],3), 'bwd', round(d['bwd_main_ms'],3), 'imb', round(d['imbalance_measured'],4), 'clk', d['clocks']['sm_mhz'])" || echo "FAIL $n $tr $o"
done; done; done; done
