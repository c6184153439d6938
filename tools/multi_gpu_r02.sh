#!/bin/bash
# Round-2 multi-GPU evidence on one box with N GPUs (run under gpurun --gpus N).
N=${N:-4}
mkdir -p gpurun_out/r02_multi
python -m pytest tests/test_gpu_multi.py -q > gpurun_out/r02_multi/pytest_multi_n$N.log 2>&1; tail -2 gpurun_out/r02_multi/pytest_multi_n$N.log
for n in 2 $N; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2951$n \
    bench.py --gpus $n --steps 10 --warmup 3 > gpurun_out/r02_multi/bench_n$n.json 2> gpurun_out/r02_multi/bench_n$n.err
  tail -1 gpurun_out/r02_multi/bench_n$n.err
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2952$n \
    bench.py --gpus $n --steps 10 --warmup 3 --transport nccl > gpurun_out/r02_multi/bench_n${n}_nccl.json 2> gpurun_out/r02_multi/bench_n${n}_nccl.err
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29530 \
  tools/sweep_policies.py > gpurun_out/r02_multi/sweep_policies_n$N.jsonl 2> gpurun_out/r02_multi/sweep.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29531 \
  tools/exchange_bw.py > gpurun_out/r02_multi/exchange_bw_n$N.jsonl 2> gpurun_out/r02_multi/xbw.err
ls gpurun_out/r02_multi
