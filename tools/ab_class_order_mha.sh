#!/bin/bash
# MHA (configs 2, 3): query-block-pair class order A/B on emulated CP ranks + CTA tails.
cd $GRAFT_REPO_ROOT
out=gpurun_out/${1:-mha2}
mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_attention.py -x -q -k "class_order or pairs or config1 or split_kv" > $out/pytest.log 2>&1; tail -2 $out/pytest.log
for cw in "2 2" "3 4" "3 8"; do set -- $cw
  BAM_LIB_PATH=paper_2503_11367_b200/libbam_clk.so timeout 300 python tools/cta_tail.py --config $1 --world $2 --out $out/cta_tail.jsonl > /dev/null 2>&1 || echo FAIL $cw
done
for pass in 1 2; do for o in 0 1; do for cw in "2 2" "3 4"; do set -- $cw
  echo "pass $pass order $o config $1 world $2"
  BAM_FWD_CLASS_ORDER=$o timeout 300 python tools/rank_time.py --config $1 --world $2 --iters 2
done; done; done > $out/ab_rank_time.txt 2>&1
grep -c makespan $out/ab_rank_time.txt
