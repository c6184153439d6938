#!/bin/bash
# A/B timing of libbam variants (tools/time_attn.py), interleaved to cancel clock drift.
#   tools/ab_run.sh "4,2" libbam.so libbam_base.so ...   (from the repo root)
cfg=$1; shift
for pass in ${PASSES:-1 2}; do
  for lib in "$@"; do
    echo -n "pass $pass $lib "
    BAM_LIB_PATH=paper_2503_11367_b200/$lib python tools/time_attn.py --config "$cfg" --iters 5 | tr '\n' ' '
    echo
  done
done
