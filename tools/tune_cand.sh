python tools/prof_score.py --sets 100000 --qsets 256 --L 32 --C 7 --reps 3 --topk 100 --mode cand
DSRT_LIB=paper_2210_15748_b200/csrc/variant_minb2.so python tools/prof_score.py --sets 100000 --qsets 256 --L 32 --C 7 --reps 3 --topk 100 --mode cand
