#!/bin/bash
# ncu evidence for the bench lines: each command first runs plain (must exit 0),
# then once under ncu.  Outputs in gpurun_out/ (scratch); summaries go to profiles/.
set -x
O=gpurun_out
# cfg1: dominant kernel (full set) + launch list
python bench.py --steps 3 --warmup 3 > $O/n_cfg1.json 2> $O/n_cfg1.err && \
ncu --set full --import-source on --clock-control none -k regex:score_all_kernel -c 1 -o $O/ncu_cfg1 \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/n_cfg1_ncu.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg1.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/n_cfg1_launch.log 2>&1
# cfg2: tcgen05 hash
python bench.py --config 2 --steps 5 --warmup 3 > $O/n_cfg2.json 2> $O/n_cfg2.err && \
ncu --set full --import-source on --clock-control none -k regex:hash_tc_kernel -c 1 -o $O/ncu_cfg2 \
    python bench.py --config 2 --steps 1 --warmup 3 > $O/n_cfg2_ncu.log 2>&1
# cfg4 shape: one 1M-set launch (the per-launch size of the 8M-set run)
python bench.py --config 4 --sets 1000000 --steps 1 --warmup 3 --no-cpu-baseline > $O/n_cfg4.json 2> $O/n_cfg4.err && \
ncu --set full --import-source on --clock-control none -k regex:score_all_kernel -c 1 -o $O/ncu_cfg4 \
    python bench.py --config 4 --sets 1000000 --steps 1 --warmup 3 --no-cpu-baseline > $O/n_cfg4_ncu.log 2>&1
# cfg3: candidate scoring + prefilter screen of one batch
python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline > $O/n_cfg3.json 2> $O/n_cfg3.err && \
ncu --set full --import-source on --clock-control none -k "regex:score_cand_kernel|pf_screen" -c 3 -o $O/ncu_cfg3 \
    python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --latency-queries 0 > $O/n_cfg3_ncu.log 2>&1
ls -la $O
