#!/bin/bash
# BASELINE configs 1-3 at their own CP degree (config 1: N=1, config 2: N=2,
# config 3: N=4) on one 4-GPU box, both transports.
#   gpurun --gpus 4 -- bash tools/configs_multi.sh <tag>
cd $GRAFT_REPO_ROOT
out=gpurun_out/${1:-cfgs}
mkdir -p $out
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --config 1 --steps 10 --warmup 3 > $out/bench_c1_n1.json 2> $out/c1.err; echo "c1 rc=$?"
for cn in "2 2" "3 4"; do set -- $cn
  for tr in auto nccl; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 \
      --master-port 2959$2 bench.py --config $1 --gpus $2 --steps 10 --warmup 3 --transport $tr \
      > $out/bench_c$1_n$2_$tr.json 2> $out/c$1_$tr.err; echo "c$1 n$2 $tr rc=$?"
  done
  CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --config $1 --steps 5 --warmup 3 --no-cpu-baseline \
    > $out/bench_c$1_n1.json 2> $out/c$1_n1.err; echo "c$1 n1 rc=$?"
done
for f in $out/bench_c*.json; do python3 -c "
import json
d=json.loads([l for l in open('$f') if l.startswith('{')][-1])
print('$f', round(d['value'],1), round(d.get('tflops_per_gpu',0),1), 'fwd', round(d['fwd_kernel_ms'],3), 'bwd', round(d['bwd_main_ms'],3), 'imb', round(d.get('imbalance_measured',1),4), 'e2e', round(d['e2e']['value'],1))" || echo "bad $f"; done
