#!/bin/bash
# exhaustive K3 variants at cfg4 shape (200k sets x 1024 query sets, L=32 C=8) and cfg1 shape
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out
: > $O/exp_all.txt
for v in base $VARIANTS; do
  if [ $v = base ]; then L=""; else L="paper_2210_15748_b200/csrc/variant_$v.so"; fi
  echo "== $v" >> $O/exp_all.txt
  DSRT_LIB=$L python tools/prof_score.py --sets 200000 --qsets 1024 --L 32 --C 8 --reps 3 --topk 1000 --mode all >> $O/exp_all.txt 2>&1
  DSRT_LIB=$L python tools/prof_score.py --sets 100000 --qsets 1000 --L 64 --C 7 --reps 3 --topk 100 --mode all >> $O/exp_all.txt 2>&1
  DSRT_LIB=$L python tools/prof_score.py --sets 1000000 --qsets 256 --L 32 --C 7 --reps 5 --topk 100 --mode cand --cand 4096 >> $O/exp_all.txt 2>&1
done
