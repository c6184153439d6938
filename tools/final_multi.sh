#!/bin/bash
# Multi-GPU tests and bench lines of the final code on one 4-GPU box.
cd $GRAFT_REPO_ROOT
out=gpurun_out/${1:-fm}
mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_cp.py -x -q > $out/pytest.log 2>&1; tail -2 $out/pytest.log
for pass in 1 2; do for n in 4 2; do for tr in auto nccl; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2968$n bench.py --gpus $n --steps 10 --warmup 3 --transport $tr > $out/bench_n${n}_${tr}_$pass.json 2> $out/b.err
  python3 -c "
import json
d=json.loads([l for l in open('$out/bench_n${n}_${tr}_$pass.json') if l.startswith('{')][-1])
print('pass $pass n$n $tr', round(d['value'],1), 'step', round(d['ms_per_step'],2), 'fwd', round(d['fwd_kernel_ms'],2), 'bwd', round(d['bwd_main_ms'],2), 'imb', round(d['imbalance_measured'],4), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'])" || echo "FAIL $n $tr"
done; done; done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29691 tools/exchange_bw.py > $out/xbw_n4.jsonl 2>/dev/null
grep kv_all_gather $out/xbw_n4.jsonl | cut -c1-200
