#!/bin/bash
# Round-end evidence on one 4-GPU box: GPU suite + smoke, bench lines at
# N=1 (with the CPU baseline) / 2 / 4, the reference arm, the ncu launch list of
# the N=1 bench and one --set full capture of the attention kernels.
#   gpurun --gpus 4 --timeout 3000 -- bash tools/final_refresh.sh <tag>
cd $GRAFT_REPO_ROOT
tag=${1:-final}
out=gpurun_out/$tag
mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; tail -2 $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $out/smoke.log 2>&1; tail -1 $out/smoke.log
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > $out/bench_n1.json 2> $out/bench_n1.err; echo "n1 rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $out/bench_ref_n1.json 2> $out/bench_ref_n1.err; echo "ref rc=$?"
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2958$n bench.py --gpus $n --steps 5 --warmup 3 > $out/bench_n$n.json 2> $out/bench_n$n.err
  echo "n$n rc=$?"
done
for f in $out/bench_n*.json; do python3 -c "
import json,sys
d=json.loads([l for l in open('$f') if l.startswith('{')][-1])
print('$f', round(d['value'],1), round(d.get('tflops_per_gpu',0),1), 'e2e', round(d['e2e']['value'],1), d['clocks'])"; done
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 \
  > $out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"attn_(bwd|fwd_split)_kernel" -c 2 -o $out/prof python tools/run_attn.py --config 4 --iters 1 \
  > $out/ncu_full.log 2>&1; echo "ncu full rc=$?"
ls -la $out
