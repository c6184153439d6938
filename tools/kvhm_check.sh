#!/bin/bash
cd $GRAFT_REPO_ROOT
out=gpurun_out/${1:-kvhm}
mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_cp.py tests/test_gpu_multi.py -x -q > $out/pytest.log 2>&1; tail -2 $out/pytest.log
for pass in 1 2; do for cn in "4 4" "3 4" "4 2"; do set -- $cn
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 \
    --master-port 2963$2 bench.py --config $1 --gpus $2 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 \
    > $out/b_c$1_n$2_$pass.json 2> $out/b.err
  python3 -c "
import json
d=json.loads([l for l in open('$out/b_c$1_n$2_$pass.json') if l.startswith('{')][-1])
print('pass $pass c$1 n$2', round(d['value'],1), 'step', round(d['ms_per_step'],3), 'fwd_win-k', round(d['fwd_ms']-d['fwd_kernel_ms'],3), 'bwd_win-k', round(d['bwd_ms']-d['bwd_main_ms'],3), 'k', [round(x,2) for x in d['per_rank_kernel_ms']])" || echo "FAIL c$1 n$2"
done; done
