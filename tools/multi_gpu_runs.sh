#!/bin/bash
# Multi-GPU bench lines (one box): N=2 and N=4 at the default KV-head groups,
# plus the head-group overlap ablation at N=4.
# usage: bash tools/multi_gpu_runs.sh <out_dir>
out=${1:-gpurun_out}
mkdir -p "$out"
TR=${TRANSPORT:-nccl}
run() {  # n groups
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 1000)) bench.py --gpus $1 --steps 5 --warmup 3 --groups $2 \
    --transport $TR > "$out/bench_n$1_g$2.json" 2> "$out/bench_n$1_g$2.err"
  echo "n=$1 groups=$2 transport=$TR rc=$? $(grep '^{' "$out/bench_n$1_g$2.json" | python3 -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['value'],1), round(d['tflops_per_gpu'],1), 'fwd', round(d['fwd_ms'],2), 'bwd', round(d['bwd_ms'],2), 'imb', round(d['imbalance_measured'],4), 'e2e', round(d['e2e']['value'],1), d['clocks'])" 2>&1 | tail -1)"
}
n=$(nvidia-smi -L | wc -l)
if [ -n "$RUNS" ]; then
  for r in $RUNS; do run ${r%:*} ${r#*:}; done
elif [ "$n" -ge 4 ]; then
  run 4 2; run 4 1; run 4 4; run 2 2
else
  run 2 2; run 2 1
fi
