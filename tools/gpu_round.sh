#!/bin/bash
# One GPU session: -m gpu tests, default bench, launch list + dram traffic of the timed step.
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo PYTEST_EXIT=$? >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
DSRT_PROFILE_STEPS=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/c4_launches_steps.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/c4_launch.log 2>&1
DSRT_PROFILE_STEPS=1 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:score_all_kernel --csv --log-file $O/c4_traffic2.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/c4_traffic2.log 2>&1
