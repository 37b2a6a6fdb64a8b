#!/bin/bash
# Final round-2 evidence: ncu --set full of the hash kernel, launch lists of a cfg3 and a cfg2 step,
# ncu --set full of the final candidate-scoring kernel.  Each command first runs plain.
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out
python tools/prof_hash.py --mode 3 --dtype bf16 --n 4000000 --reps 3 > $O/pf_hash.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:hash_tc_kernel -c 1 -f -o $O/prof_hash_tc_final \
    python tools/prof_hash.py --mode 3 --dtype bf16 --n 4000000 --reps 1 > /dev/null 2>&1
python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline > $O/pf_cfg3.log 2>&1 && \
DSRT_PROFILE_STEPS=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/c3_launches_steps.csv python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/prof_score.py --sets 1000000 --qsets 256 --L 32 --C 7 --reps 1 --topk 100 --mode cand --cand 4096 > $O/pf_cand.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:score_cand_kernel -c 1 -f -o $O/prof_cand_final \
    python tools/prof_score.py --sets 1000000 --qsets 256 --L 32 --C 7 --reps 1 --topk 100 --mode cand --cand 4096 > /dev/null 2>&1
echo done
