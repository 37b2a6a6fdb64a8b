#!/bin/bash
# ncu evidence for the dominant kernels (each command first runs plain, then under ncu).
set -x
python tools/prof_score.py --sets 20000 --qsets 1024 --L 64 --C 7 --reps 1 > gpurun_out/p1.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:score_all_kernel -c 1 -o gpurun_out/prof_score_all_l64c7 \
    python tools/prof_score.py --sets 20000 --qsets 1024 --L 64 --C 7 --reps 1 > /dev/null 2>&1
python tools/prof_score.py --sets 20000 --qsets 1024 --L 32 --C 8 --reps 1 > gpurun_out/p2.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:score_all_kernel -c 1 -o gpurun_out/prof_score_all_l32c8 \
    python tools/prof_score.py --sets 20000 --qsets 1024 --L 32 --C 8 --reps 1 > /dev/null 2>&1
python tools/prof_score.py --sets 100000 --qsets 256 --L 32 --C 7 --reps 1 --mode cand > gpurun_out/p3.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:score_cand_kernel -c 1 -o gpurun_out/prof_score_cand_l32c7 \
    python tools/prof_score.py --sets 100000 --qsets 256 --L 32 --C 7 --reps 1 --mode cand > /dev/null 2>&1
python bench.py --config 2 --vectors 2000000 --steps 2 --warmup 1 > gpurun_out/p4.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:hash_tc_kernel -c 1 -o gpurun_out/prof_hash_tc \
    python bench.py --config 2 --vectors 2000000 --steps 2 --warmup 1 > /dev/null 2>&1
python tools/prof_prefilter.py --reps 1 > gpurun_out/p5.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k "regex:pf_screen|select_kernel|topk_kernel" -c 3 -o gpurun_out/prof_prefilter \
    python tools/prof_prefilter.py --reps 1 > /dev/null 2>&1
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1
echo done
