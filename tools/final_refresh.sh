#!/bin/bash
# Round-end evidence on one 4-GPU box: GPU suite (incl. the N=2/4 multi-process
# parity tests) + smoke, bench lines at N=1 (with the CPU baseline) / 2 / 4 on
# both transports, the reference arm, the config-5 policy sweep and the exchange
# bandwidth at N=4, the ncu launch list of the N=1 bench and one --set full
# capture of the attention kernels.
#   gpurun --gpus 4 --timeout 3600 -- bash tools/final_refresh.sh <tag>
cd $GRAFT_REPO_ROOT
tag=${1:-final}
out=gpurun_out/$tag
mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; tail -2 $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $out/smoke.log 2>&1; tail -1 $out/smoke.log
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > $out/bench_n1.json 2> $out/bench_n1.err; echo "n1 rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $out/bench_ref_n1.json 2> $out/bench_ref_n1.err; echo "ref rc=$?"
for n in 2 4; do
  for tr in auto nccl; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port 2958$n bench.py --gpus $n --steps 5 --warmup 3 --transport $tr \
      > $out/bench_n${n}_$tr.json 2> $out/bench_n${n}_$tr.err
    echo "n$n $tr rc=$?"
  done
done
for f in $out/bench_n*.json; do python3 -c "
import json,sys
d=json.loads([l for l in open('$f') if l.startswith('{')][-1])
print('$f', round(d['value'],1), round(d.get('tflops_per_gpu',0),1), 'e2e', round(d['e2e']['value'],1), 'imb', d.get('imbalance_measured'), d['clocks'])"; done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29530 tools/sweep_policies.py > $out/sweep_policies_n4.jsonl 2> $out/sweep.err; echo "sweep rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29531 tools/exchange_bw.py > $out/exchange_bw_n4.jsonl 2> $out/xbw.err; echo "xbw rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 \
  > $out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"attn_(bwd|fwd_split)_kernel" -c 2 -o $out/prof python tools/run_attn.py --config 4 --iters 1 \
  > $out/ncu_full.log 2>&1; echo "ncu full rc=$?"
ls -la $out
