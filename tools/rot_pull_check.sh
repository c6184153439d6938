#!/bin/bash
# Rotation-order peer-by-peer K/V pulls: CP tests, exchange bandwidth, benches,
# and the forward's flag-wait share on real ranks.
cd $GRAFT_REPO_ROOT
out=gpurun_out/${1:-rot}
mkdir -p $out
timeout 1500 python -m pytest tests/test_gpu_cp.py tests/test_gpu_multi.py tests/test_gpu_attention.py -x -q > $out/pytest.log 2>&1; tail -2 $out/pytest.log
for n in 4 2; do timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2965$n tools/exchange_bw.py > $out/xbw_n$n.jsonl 2>/dev/null; done
for pass in 1 2; do for cn in "4 4" "3 4" "4 2"; do set -- $cn
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 \
    --master-port 2966$2 bench.py --config $1 --gpus $2 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 \
    > $out/b_c$1_n$2_$pass.json 2> $out/b.err
  python3 -c "
import json
d=json.loads([l for l in open('$out/b_c$1_n$2_$pass.json') if l.startswith('{')][-1])
print('pass $pass c$1 n$2', round(d['value'],1), 'step', round(d['ms_per_step'],3), 'fwd_k', round(d['fwd_kernel_ms'],3), 'fwd_win-k', round(d['fwd_ms']-d['fwd_kernel_ms'],3), 'bwd_k', round(d['bwd_main_ms'],3), 'k', [round(x,2) for x in d['per_rank_kernel_ms']])" || echo "FAIL c$1 n$2"
done; done
for n in 4 2; do
  BAM_LIB_PATH=paper_2503_11367_b200/libbam_clk.so timeout 600 python -m torch.distributed.run \
    --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2967$n tools/cta_tail.py \
    --config 4 --transport ce --out $out/cta_tail_real.jsonl > /dev/null 2> $out/ct.err || echo "FAIL ct $n"
done
python3 -c "
import json
for l in open('$out/xbw_n4.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print('xbw', d['n_gpus'], d['step'], d['transport'], round(d['nvlink_gbs_per_rank'],1))
for l in open('$out/xbw_n2.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print('xbw', d['n_gpus'], d['step'], d['transport'], round(d['nvlink_gbs_per_rank'],1))
for l in open('$out/cta_tail_real.jsonl'):
    d=json.loads(l)
    if d['kernel']=='fwd_split': print('flagwait', d['world'], d['rank'], round(d['flag_wait_frac']*100,3), round(d['span_ms'],3), round(d['busy_frac'],4))
"
