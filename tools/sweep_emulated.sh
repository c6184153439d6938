#!/bin/bash
# BASELINE.json config 5 at CP=8 (and 2, 4) with the ranks emulated on one GPU
# (tools/rank_time.py, ranks interleaved): per-rank kernel-only fwd+bwd time of
# every mask x policy; the exchange is not included (see bench.py / the N=2/4 runs)
out=${1:-gpurun_out/sweep_emulated.jsonl}
: > $out
for w in ${WORLDS:-8}; do
  for m in causal prefix_lm multimodal multi_image; do
    for pol in lpt zigzag contiguous; do
      python tools/rank_time.py --config $m --world $w --policy $pol --iters 2 | tail -1 >> $out
    done
  done
done
cat $out
