cd $GRAFT_REPO_ROOT
for i in 1 2; do
python tools/prof_score.py --sets 1000000 --qsets 256 --L 32 --C 7 --mode cand --cand 4096 --reps 5 >> gpurun_out/pc2.log 2>&1
DSRT_LIB=paper_2210_15748_b200/csrc/libdessert_U4.so python tools/prof_score.py --sets 1000000 --qsets 256 --L 32 --C 7 --mode cand --cand 4096 --reps 5 >> gpurun_out/pc2.log 2>&1
done
