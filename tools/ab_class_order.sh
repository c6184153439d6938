#!/bin/bash
# A/B of the forward's class-major CTA order (BAM_FWD_CLASS_ORDER=1, default)
# against head-pair-major (0): emulated CP ranks (tools/rank_time.py), one GPU.
#   gpurun -- bash tools/ab_class_order.sh <tag>
cd $GRAFT_REPO_ROOT
out=gpurun_out/${1:-cls}
mkdir -p $out
for pass in 1 2 3; do for o in 0 1; do for w in 8 4; do
  echo "pass $pass order $o world $w"
  BAM_FWD_CLASS_ORDER=$o timeout 300 python tools/rank_time.py --config 4 --world $w --iters 2
done; done; done > $out/ab_rank_time.txt 2>&1
grep -c makespan $out/ab_rank_time.txt
