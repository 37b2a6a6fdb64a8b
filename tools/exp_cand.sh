#!/bin/bash
# candidate-mode K3 variants at cfg3 shape (256 query sets x 4096 random candidates of 1M sets)
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out
A="--sets 1000000 --qsets 256 --L 32 --C 7 --reps 5 --topk 100 --mode cand --cand 4096"
: > $O/exp_cand.txt
for v in base $VARIANTS; do
  if [ $v = base ]; then L=""; else L="paper_2210_15748_b200/csrc/variant_$v.so"; fi
  echo "== $v" >> $O/exp_cand.txt
  DSRT_LIB=$L python tools/prof_score.py $A >> $O/exp_cand.txt 2>&1
done
if [ -n "$NCU_CAND" ]; then
  ncu --set full --import-source on --clock-control none -k regex:score_cand_kernel -c 1 -f -o $O/prof_cand_r2 \
     python tools/prof_score.py --sets 1000000 --qsets 256 --L 32 --C 7 --reps 1 --topk 100 --mode cand --cand 4096 > $O/prof_cand_r2.log 2>&1
fi
