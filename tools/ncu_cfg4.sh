#!/bin/bash
# ncu evidence for the cfg4 bench line (fused exhaustive search).  Each command
# first runs plain (must exit 0), then under ncu.  Scratch output in gpurun_out/.
#  1. launch list of the default bench (cold-cache, serialised per-launch times)
#  2. dram bytes of every scoring launch of one full cfg4 step (few metrics -> few replays)
#  3. one --set full capture of the largest scoring launch at 1M sets (pipe utilisation, stalls)
set -x
O=gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/c4_plain.json 2> $O/c4_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/c4_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/c4_launch.log 2>&1
DSRT_PROFILE_STEPS=1 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:score_all_kernel --csv --log-file $O/c4_traffic.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/c4_traffic.log 2>&1
python bench.py --sets 1000000 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/c4_1m.json 2> $O/c4_1m.err && \
ncu --set full --import-source on --clock-control none -k regex:score_all_kernel -s 2 -c 1 -o $O/ncu_c4_1m \
    python bench.py --sets 1000000 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/c4_1m_ncu.log 2>&1
ls -la $O
