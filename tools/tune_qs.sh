for qs in 4 8; do
 DSRT_QS=$qs python tools/prof_score.py --sets 100000 --qsets 1024 --L 32 --C 8 --reps 3 --topk 100
 DSRT_QS=$qs python tools/prof_score.py --sets 100000 --qsets 1024 --L 32 --C 7 --reps 3 --topk 100
done
