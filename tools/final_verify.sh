#!/bin/bash
# Final verification on one 4-GPU box: the whole GPU suite, smoke, bench lines N=1/2/4.
cd $GRAFT_REPO_ROOT
out=gpurun_out/${1:-fv}
mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q > $out/pytest_gpu.log 2>&1; tail -2 $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $out/smoke.log 2>&1; tail -1 $out/smoke.log
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > $out/bench_n1.json 2> $out/bench_n1.err; echo "n1 rc=$?"
for n in 2 4; do for tr in auto nccl; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2970$n bench.py --gpus $n --steps 10 --warmup 3 --transport $tr > $out/bench_n${n}_$tr.json 2> $out/b_${n}_$tr.err
  echo "n$n $tr rc=$?"
done; done
for f in $out/bench_n*.json; do python3 -c "
import json
d=json.loads([l for l in open('$f') if l.startswith('{')][-1])
print('$f', round(d['value'],1), 'step', round(d['ms_per_step'],2), 'fwd', round(d['fwd_kernel_ms'],2), 'bwd', round(d['bwd_main_ms'],2), 'imb', round(d.get('imbalance_measured',1),4), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'], d['gpu_launches'])"; done
