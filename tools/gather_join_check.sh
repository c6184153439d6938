#!/bin/bash
cd $GRAFT_REPO_ROOT
out=gpurun_out/${1:-gj}
mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_cp.py -x -q > $out/pytest.log 2>&1; tail -2 $out/pytest.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29692 tools/exchange_bw.py > $out/xbw_n4.jsonl 2>/dev/null
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29693 tools/exchange_bw.py > $out/xbw_n2.jsonl 2>/dev/null
python3 -c "
import json
for f in ('$out/xbw_n4.jsonl','$out/xbw_n2.jsonl'):
    for l in open(f):
        if l.startswith('{'):
            d=json.loads(l)
            if d['step']=='kv_all_gather': print(d['n_gpus'], d['transport'], round(d['nvlink_gbs_per_rank'],1))"
for pass in 1 2; do for n in 4 2; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2969$n bench.py --gpus $n --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $out/bench_n${n}_$pass.json 2> $out/b.err
  python3 -c "
import json
d=json.loads([l for l in open('$out/bench_n${n}_$pass.json') if l.startswith('{')][-1])
print('pass $pass n$n', round(d['value'],1), 'step', round(d['ms_per_step'],2), 'fwd', round(d['fwd_kernel_ms'],2), 'fwdwin-k', round(d['fwd_ms']-d['fwd_kernel_ms'],3), 'bwd', round(d['bwd_main_ms'],2), 'clk', d['clocks']['sm_mhz'])" || echo "FAIL $n"
done; done
